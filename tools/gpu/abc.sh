# A/B of library variants (tools/_libs/<name>.so; "base" = the in-tree build) on C3, and on C4 if C4=1
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_libs/$v.so"; fi
  cfgs=("")
  [ "${C4:-0}" = 1 ] && cfgs+=("--n 6000000 --width 3840 --height 2160 --flat --depth 2 --steps 20")
  for c in "${cfgs[@]}"; do
    SEELE_LIB=$lib python bench.py --steps ${STEPS:-120} --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 1 $c > /tmp/ab.json 2>/tmp/ab.err
    python -c "
import json; d=json.load(open('/tmp/ab.json'))
print('$v', d['config']['workload'][:3], 'fps %.1f serial %.1f' % (d['value'], d['value_serial']), {k: v['ms'] for k, v in d['stages'].items()}, 'redecide', d['work']['alpha_redecide'], 't_amb', d['work']['t_ambiguous'])" || tail -3 /tmp/ab.err
  done
done
