# side-stream CTA count / late threshold sweep of config 3 (python tools/t3.py)
for rep in 1 2; do
for sc in 12 16 20 24; do
  for lp in 30 38 46; do
    echo "SC=$sc LP=$lp: $(F2_SIDE_CTAS=$sc F2_LATE_PCT=$lp timeout 120 python tools/t3.py 65536 5 2>&1 | tail -1)"
  done
done
for sl in 32 64 96; do echo "SL=$sl: $(F2_SIDE_CTAS_LATE=$sl timeout 120 python tools/t3.py 65536 5 2>&1 | tail -1)"; done
done
