mkdir -p gpurun_out/r2ax
VARIANTS="c h" bash tools/ab_variants.sh gpurun_out/r2ax cfg2 2 >> gpurun_out/r2ax/ab.txt 2>&1
VARIANTS="c h" bash tools/ab_variants.sh gpurun_out/r2ax cfg3 2 >> gpurun_out/r2ax/ab.txt 2>&1
REPS=2000 MODES="OB_LIB_VARIANT=h" bash tools/race_stress.sh gpurun_out/r2ax
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2ax/t.txt 2>&1
