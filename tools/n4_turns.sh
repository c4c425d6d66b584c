out=${1:-gpurun_out/n4turns}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_cgp.py -q -m gpu -k multi_process > $out/pytest_nccl.txt 2>&1
port=29880
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
run cfg4_cgp4_a 4 --config cfg4 --cgp-size 4 --no-e2e
run cfg4_cgp4_b 4 --config cfg4 --cgp-size 4 --no-e2e
run cfg4_cgp4_c 4 --config cfg4 --cgp-size 4 --no-e2e
run cfg4_cgp2x2 4 --config cfg4 --no-e2e
run cfg2_cgp4 4 --no-cpu --no-e2e --parallel cgp
run cfg2_cgp2x2 4 --no-cpu --no-e2e --parallel cgp --cgp-size 2
touch "$out/failures.txt"
