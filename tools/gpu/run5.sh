python -m pytest tests -m gpu -q -x -k "depth or small_plan or config1 or large_synth or c3_frames or c4 or c5 or residency or edge" > gpurun_out/r2_gpu5.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_gpu5.log
bash tools/gpu/prof_launch.sh d3
