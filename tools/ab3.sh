for i in 1 2 3; do for f in "" "--raster-first"; do
python bench.py --steps 600 --warmup 10 --no-cpu-baseline --e2e-steps 5 $f 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('flag[$f]', round(d['value'],1))"
done; done
