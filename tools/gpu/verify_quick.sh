# GPU suite + default bench of the current build
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/gpu_full.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_full.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/configs.py > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; cat gpurun_out/configs.log
