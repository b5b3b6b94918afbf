for i in 1 2; do for lib in tools/_libs/b1.so tools/_libs/b1s1.so; do
SEELE_LIB=$lib python bench.py --steps 600 --warmup 10 --no-cpu-baseline --e2e-steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['value_serial'],1))"
done; done
