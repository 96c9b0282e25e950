# bench ms/step for an environment toggle: bash tools/dbg/env_ab.sh VAR v1 v2 ...
VAR=$1; shift
for v in "$@"; do
  for r in 1 2; do
    env $VAR=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); c = d['config']
print('$VAR=$v', round(d['ms_per_step'], 4), 'e2e', round(d['e2e']['value'], 1), 'sel', round(c.get('selector_overhead', 0), 3), 'static', c.get('static_ms_per_step'))
"
  done
done
