set -x
nproc
python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/r2_gpu1.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2_gpu1.log
python bench.py --steps 60 --warmup 5 --gather > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench1.json
tail -5 gpurun_out/r2_bench1.err
