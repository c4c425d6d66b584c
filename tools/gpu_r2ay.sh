mkdir -p gpurun_out/r2ay
VARIANTS="c i h" bash tools/ab_variants.sh gpurun_out/r2ay cfg2 2 >> gpurun_out/r2ay/ab.txt 2>&1
VARIANTS="c i" bash tools/ab_variants.sh gpurun_out/r2ay cfg3 2 >> gpurun_out/r2ay/ab.txt 2>&1
REPS=2000 MODES="OB_LIB_VARIANT=i" bash tools/race_stress.sh gpurun_out/r2ay
OB_LIB_VARIANT=i timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2ay/t.txt 2>&1
