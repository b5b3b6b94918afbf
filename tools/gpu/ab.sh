# A/B of library variants in tools/_libs/*.so (names as args): bench value + stage times
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_libs/$v.so"; fi
  SEELE_LIB=$lib python bench.py --steps 120 --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 1 > /tmp/ab_$v.json 2>/tmp/ab_$v.err
  python -c "
import json,sys; d=json.load(open('/tmp/ab_$v.json'))
print('$v', 'fps %.1f serial %.1f' % (d['value'], d['value_serial']), {k: v['ms'] for k, v in d['stages'].items()}, 'redecide', d['work']['alpha_redecide'], 't_amb', d['work']['t_ambiguous'])" || tail -3 /tmp/ab_$v.err
done
