# bench C3 pipelined with the plan stages on a green-context partition of N SMs (args: N values; 0 = shared)
for n in "$@"; do
  python bench.py --steps ${STEPS:-120} --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 1 --partition $n ${EXTRA:-} > /tmp/p.json 2>/tmp/p.err
  python -c "
import json; d=json.load(open('/tmp/p.json'))
print('partition $n', 'fps %.1f serial %.1f' % (d['value'], d['value_serial']), {k: v['ms'] for k, v in d['stages'].items()})" || tail -5 /tmp/p.err
done
