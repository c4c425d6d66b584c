set -x
mkdir -p gpurun_out/r2ai
python -m pytest tests/test_gpu_bench_parity.py tests/test_stored_transforms.py -x -q -m gpu > gpurun_out/r2ai/t.txt 2>&1
python bench.py > gpurun_out/r2ai/bench.json 2> gpurun_out/r2ai/bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:k_agg -c 40 --csv --log-file gpurun_out/r2ai/agg_warm.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --lanes 1 > gpurun_out/r2ai/ncu.log 2>&1
