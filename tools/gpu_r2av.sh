mkdir -p gpurun_out/r2av
REPS=2500 MODES="OB_QROWS_SERIAL=1 X=1" bash tools/race_stress.sh gpurun_out/r2av
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2av/t.txt 2>&1
VARIANTS="a c f" bash tools/ab_variants.sh gpurun_out/r2av cfg2 2 >> gpurun_out/r2av/ab.txt 2>&1
VARIANTS="a c f" bash tools/ab_variants.sh gpurun_out/r2av cfg3 1 >> gpurun_out/r2av/ab.txt 2>&1
