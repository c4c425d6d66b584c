# same-box A/B: parity of the shipped build, then VARIANTS over the given configs
set -x
out=${OUT:-gpurun_out/ab}
mkdir -p $out
python -m pytest ${TESTS:-tests/test_gpu_bench_parity.py tests/test_stored_transforms.py} -x -q -m gpu > $out/t.txt 2>&1
for c in ${CFGS:-cfg2}; do bash tools/ab_variants.sh $out $c ${ROUNDS:-2} >> $out/ab.txt 2>&1; done
