#!/bin/bash
# alternate env settings: abenv.sh "ENV_A" "ENV_B" "cmd" rounds
for i in $(seq $4); do
  echo "A: $(env $1 timeout 120 bash -c "$3" 2>&1 | tail -1)"
  echo "B: $(env $2 timeout 120 bash -c "$3" 2>&1 | tail -1)"
done
