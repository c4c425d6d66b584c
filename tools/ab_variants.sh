#!/bin/bash
# Same-box A/B of library builds / runtime settings.  A variant is LIB[:VAR=VAL[,VAR=VAL...]]:
# OB_LIB_VARIANT=LIB selects libomega_b200.LIB.so, the assignments go into the environment.
# Usage (GPU box): VARIANTS="a b b:OB_RX_ONESWEEP=1" bash tools/ab_variants.sh out_dir config rounds
out=${1:-gpurun_out/ab}; cfg=${2:-cfg2}; rounds=${3:-2}
mkdir -p "$out"
for r in $(seq 1 $rounds); do
  for v in ${VARIANTS:-a b}; do
    lib=${v%%:*}; envs=""; [ "$v" != "$lib" ] && envs=$(echo "${v#*:}" | tr ',' ' ')
    tag=$(echo "$v" | tr ':=,' '___')
    env OB_LIB_VARIANT=$lib $envs python bench.py --config $cfg --no-cpu --no-e2e > "$out/${cfg}_${tag}_$r.json" 2> "$out/${cfg}_${tag}_$r.err"
    python -c "
import json
d=json.loads(open('$out/${cfg}_${tag}_$r.json').read().strip().splitlines()[-1])
print('$cfg', '$v', $r, d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])
"
  done
done
