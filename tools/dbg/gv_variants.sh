# quick GEMV sweep for each prebuilt library variant: bash tools/dbg/gv_variants.sh TAG v1 v2 ...
TAG=$1; shift
cp paper_2508_06041_b200/libdpq_b200.so /tmp/base.so
for v in "$@"; do
  cp paper_2508_06041_b200/libdpq_b200_$v.so paper_2508_06041_b200/libdpq_b200.so
  touch paper_2508_06041_b200/libdpq_b200.so
  echo "== $v"
  timeout 120 python tools/gemv_sweep.py --quick --reps 10 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(d['shape'], d['mode'], d.get('bits', d.get('pair')), round(d['us'], 2), round(d['GBps']))
"
done
cp /tmp/base.so paper_2508_06041_b200/libdpq_b200.so
