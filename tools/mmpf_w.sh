for w in 64 128 256 512 1024; do
  F2_MMPF_PANEL_BITS=$w timeout 120 python tools/mmpf_w.py 4096 4096 2>&1 | tail -1
  F2_MMPF_PANEL_BITS=$w timeout 120 python tools/mmpf_w.py 16384 16384 2>&1 | tail -1
  F2_MMPF_PANEL_BITS=$w timeout 120 python tools/mmpf_w.py 16384 131072 sparse 2>&1 | tail -1
done
