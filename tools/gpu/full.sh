# full GPU suite + default bench + launch list of the current build
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/gpu_full.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/gpu_full.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
python -c "__import__('__graft_entry__').smoke()"; echo "smoke rc=$?"
bash tools/gpu/prof_launch.sh full
