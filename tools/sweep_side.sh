#!/bin/bash
# sweep of the look-ahead panel kernel's CTA counts and the early/late threshold (config 3 ms/step)
one() { python bench.py --no-cpu --no-configs --steps 8 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['check']['packed_matches_reference'])"; }
for rep in 1 2 3; do
for lp in 22 26 30 32 34 36 38; do for sl in 48 64; do
  echo -n "rep $rep LATE_PCT=$lp SIDE=24 SIDE_LATE=$sl: "
  F2_LATE_PCT=$lp F2_SIDE_CTAS=24 F2_SIDE_CTAS_LATE=$sl one
done; done; done
