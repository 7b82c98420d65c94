#!/bin/bash
# A/B timing of two builds: tools/ab.sh libA.so libB.so "command" [rounds]
A=$1; B=$2; CMD=$3; R=${4:-3}
for i in $(seq $R); do
  echo "A: $(F2_LIB=$A timeout 120 bash -c "$CMD" 2>&1 | tail -1)"
  echo "B: $(F2_LIB=$B timeout 120 bash -c "$CMD" 2>&1 | tail -1)"
done
