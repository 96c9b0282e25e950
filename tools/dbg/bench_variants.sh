# bench ms/step + stage stamps (dynamic) for each prebuilt library variant: bash tools/dbg/bench_variants.sh TAG v1 v2 ...
TAG=$1; shift
cp paper_2508_06041_b200/libdpq_b200.so /tmp/base.so
for v in "$@"; do
  cp paper_2508_06041_b200/libdpq_b200_$v.so paper_2508_06041_b200/libdpq_b200.so
  touch paper_2508_06041_b200/libdpq_b200.so
  for r in 1 2; do
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); c = d['config']
print('$v', round(d['ms_per_step'], 4), 'e2e', round(d['e2e']['value'], 1), 'sel', round(c.get('selector_overhead', 0), 3), 'static', c.get('static_ms_per_step'))
"
  done
  timeout 200 python tools/stage_stamps.py > gpurun_out/stamps_${TAG}_$v.log 2>&1
  sed -n 1,7p gpurun_out/stamps_${TAG}_$v.log
done
cp /tmp/base.so paper_2508_06041_b200/libdpq_b200.so
