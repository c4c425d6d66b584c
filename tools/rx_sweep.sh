set -x
mkdir -p gpurun_out
for mb in 1 2 3; do
  OB_NVCC_EXTRA="-DOB_RX_MINB=$mb" python -c "from paper_2501_08547_b200.build import build; build(force=True)" > gpurun_out/c2_build_$mb.log 2>&1
  timeout 300 python bench.py --no-cpu > gpurun_out/c2_bench_cfg2_mb$mb.json 2> gpurun_out/c2_bench_cfg2_mb$mb.err
  timeout 300 python bench.py --no-cpu --config cfg3 > gpurun_out/c2_bench_cfg3_mb$mb.json 2> gpurun_out/c2_bench_cfg3_mb$mb.err
done
OB_NVCC_EXTRA="-DOB_RX_MINB=2" python -c "from paper_2501_08547_b200.build import build; build(force=True)" > gpurun_out/c2_build_final.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/c2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c2_pytest.log
