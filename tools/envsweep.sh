#!/bin/bash
# round-robin timing of env settings: tools/envsweep.sh "command" rounds "ENV1" "ENV2" ...
CMD=$1; R=$2; shift 2
for i in $(seq $R); do
  for E in "$@"; do echo "$E: $(env $E timeout 120 bash -c "$CMD" 2>&1 | tail -1)"; done
done
