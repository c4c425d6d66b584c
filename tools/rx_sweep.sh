# Tuning sweep for residency macros (-DOB_RX_MINB / -DOB_SCAN_MINB): rebuild, bench cfg1-3, then GPU tests.
# usage: bash tools/rx_sweep.sh TAG "FLAGS1" "FLAGS2" ...
set -x
tag=$1; shift
mkdir -p gpurun_out
i=0
for fl in "$@"; do
  i=$((i+1))
  OB_NVCC_EXTRA="$fl" python -c "from paper_2501_08547_b200.build import build; build(force=True)" > gpurun_out/${tag}_build_$i.log 2>&1
  echo "$fl" > gpurun_out/${tag}_flags_$i.txt
  for c in ${SWEEP_CONFIGS:-cfg2 cfg3 cfg1}; do
    timeout 300 python bench.py --no-cpu --config $c > gpurun_out/${tag}_bench_${c}_$i.json 2> gpurun_out/${tag}_bench_${c}_$i.err
  done
done
python -c "from paper_2501_08547_b200.build import build; build(force=True)" > gpurun_out/${tag}_build_final.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
