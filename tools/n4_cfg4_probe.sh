out=${1:-gpurun_out/n4cfg4}; mkdir -p $out
port=29850
run() {
  local name=$1 n=$2; shift 2
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $n "$@" > "$out/$name.json" 2> "$out/$name.err" || echo "FAIL $name" >> "$out/failures.txt"
  python -c "
import json
d=json.loads(open('$out/$name.json').read().strip().splitlines()[-1])
print('$name', d['value'], d['value_one_request_at_a_time'], d['p50_ms'], d['p99_ms'])" >> "$out/summary.txt" 2>&1
}
run cfg4_cgp4_default 4 --config cfg4 --cgp-size 4 --no-e2e
OB_NO_PDL=1 run cfg4_cgp4_nopdl 4 --config cfg4 --cgp-size 4 --no-e2e
run cfg4_cgp4_lanes2 4 --config cfg4 --cgp-size 4 --no-e2e --lanes 2
run cfg4_cgp4_default_again 4 --config cfg4 --cgp-size 4 --no-e2e
touch "$out/failures.txt"
