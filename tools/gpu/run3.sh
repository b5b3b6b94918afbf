python -m pytest tests -m gpu -q -x --durations=15 -k "depth or configs" > gpurun_out/r2_gpu3.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2_gpu3.log
bash tools/gpu/prof_launch.sh d1
