for v in base clampE; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_libs/$v.so"; fi
  for c in "" "--n 6000000 --width 3840 --height 2160 --flat --depth 2 --steps 20"; do
  SEELE_LIB=$lib python bench.py --steps 60 --warmup 3 --no-cpu-baseline --no-exact --e2e-steps 1 $c > /tmp/ab.json 2>/tmp/ab.err
  python -c "
import json; d=json.load(open('/tmp/ab.json'))
print('$v', d['config']['workload'][:20], 'fps %.1f serial %.1f' % (d['value'], d['value_serial']), 'raster', d['stages']['raster']['ms'], 'redecide', d['work']['alpha_redecide'], 't_amb', d['work']['t_ambiguous'])" || tail -3 /tmp/ab.err
  done
done
