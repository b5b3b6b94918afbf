for flags in "" "--plan-first" "--raster-first" "--plan-first --depth 4" "--plan-first --depth 2"; do
python bench.py --steps 120 --warmup 5 --no-cpu-baseline --no-exact --e2e-steps 1 $flags > /tmp/d.json 2>/tmp/d.err && python -c "
import json;d=json.load(open('/tmp/d.json'));print('$flags', 'fps %.1f serial %.1f' % (d['value'], d['value_serial']))" || tail -3 /tmp/d.err
done
