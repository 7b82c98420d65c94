#!/bin/bash
# round-robin timing of several builds: tools/abn.sh "command" rounds libA.so libB.so ...
CMD=$1; R=$2; shift 2
for i in $(seq $R); do
  for L in "$@"; do echo "$L: $(F2_LIB=$L timeout 120 bash -c "$CMD" 2>&1 | tail -1)"; done
done
