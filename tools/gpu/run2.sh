python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r2_gpu2.log 2>&1; echo "pytest rc=$?"
tail -60 gpurun_out/r2_gpu2.log
python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r2_bench2.json'));print({k:d[k] for k in ['value','value_serial','ms_per_step','stages','e2e','value_exact_serial']})"
tail -3 gpurun_out/r2_bench2.err
