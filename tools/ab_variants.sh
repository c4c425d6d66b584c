#!/bin/bash
# Same-box A/B of two library builds: OB_LIB_VARIANT=a / b select libomega_b200.{a,b}.so.
# Usage (GPU box): bash tools/ab_variants.sh out_dir config rounds
out=${1:-gpurun_out/ab}; cfg=${2:-cfg2}; rounds=${3:-2}
mkdir -p "$out"
for r in $(seq 1 $rounds); do
  for v in ${VARIANTS:-a b}; do
    OB_LIB_VARIANT=$v python bench.py --config $cfg --no-cpu --no-e2e > "$out/${cfg}_${v}_$r.json" 2> "$out/${cfg}_${v}_$r.err"
    python -c "
import json
d=json.loads(open('$out/${cfg}_${v}_$r.json').read().strip().splitlines()[-1])
print('$cfg', '$v', $r, d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])
"
  done
done
