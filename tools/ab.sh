#!/bin/bash
# A/B the C3 bench over library variants: tools/ab.sh default tools/_libs/x.so ...
cd "$(dirname "$0")/.."
for lib in "$@"; do
  if [ "$lib" = default ]; then unset SEELE_LIB; else export SEELE_LIB=$lib; fi
  python bench.py --steps 120 --warmup 5 --no-cpu-baseline --e2e-steps 10 "${AB_ARGS[@]}" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), round(d['value_serial'],1), {k: round(v['ms'],3) for k,v in d['stages'].items()}, {k: d['work'][k] for k in ('alpha_redecide','t_ambiguous','blends') if k in d['work']})"
done
