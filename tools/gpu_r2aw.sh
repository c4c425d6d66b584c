mkdir -p gpurun_out/r2aw
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2aw/t.txt 2>&1
REPS=2000 MODES="OB_LIB_VARIANT=g" bash tools/race_stress.sh gpurun_out/r2aw
VARIANTS="c g" bash tools/ab_variants.sh gpurun_out/r2aw cfg2 2 >> gpurun_out/r2aw/ab.txt 2>&1
VARIANTS="c g" bash tools/ab_variants.sh gpurun_out/r2aw cfg3 2 >> gpurun_out/r2aw/ab.txt 2>&1
