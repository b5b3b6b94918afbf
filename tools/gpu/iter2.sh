# quicker iteration: parity subset, bench, launch list, frames-in-flight sweep
python -m pytest tests -m gpu -q -x -k "${K:-small_cases or random_scenes or config1 or large_synth or c3_frames or fast_equals or depth or edge or overflow or plan or c5}" > gpurun_out/iter_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/iter_tests.log
python bench.py --steps 120 --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 120 > gpurun_out/iter_bench.json 2> gpurun_out/iter_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/iter_bench.json'));print('fps %.1f serial %.1f e2e %.1f' % (d['value'], d['value_serial'], d['e2e']['value']), {k: v['ms'] for k, v in d['stages'].items()})" || tail -5 gpurun_out/iter_bench.err
bash tools/gpu/prof_launch.sh iter
for dpt in ${DEPTHS:-}; do
python bench.py --steps 120 --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 1 --depth $dpt > /tmp/d.json 2>/dev/null && python -c "
import json;d=json.load(open('/tmp/d.json'));print('depth $dpt fps %.1f' % d['value'])"
done
