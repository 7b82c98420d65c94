#!/bin/bash
# MMPF table-apply over a 1 GiB C (tools/ta_bench.py): round-1 layouts vs the 1024-bit-tile kernel
echo "old: $(F2_MMPF_OLD64=1 python tools/ta_bench.py 1 8 16 24 32 33 64 2>&1 | tr '\n' ' ')"
for rb in 2048 8192 32768; do
  echo "rb=$rb: $(F2_MMPF_RBLOCK=$rb python tools/ta_bench.py 1 8 16 24 32 33 44 64 2>&1 | tr '\n' ' ')"
done
