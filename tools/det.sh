for env in "F2_X=1" "F2_NO_SPLIT_EARLY=1" "F2_NO_SPLIT_EARLY=1 F2_NO_PDL=1" "F2_NO_SPLIT_EARLY=1 F2_NO_GRAPH=1" "F2_NO_SPLIT_EARLY=1 F2_NO_EARLY_WIDE_TRSM=1" "F2_NO_EARLY_WIDE_TRSM=1"; do
  for i in 1 2 3; do echo "$env: $(env $env timeout 120 python tools/t3.py 65536 3 2>&1 | tail -1)"; done
done
