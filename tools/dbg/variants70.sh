# bench the 70B-width slice for each prebuilt library variant: bash tools/dbg/variants70.sh TAG v1 v2 ...
TAG=$1; shift
cp paper_2508_06041_b200/libdpq_b200.so /tmp/base.so
for v in "$@"; do
  cp paper_2508_06041_b200/libdpq_b200_$v.so paper_2508_06041_b200/libdpq_b200.so
  touch paper_2508_06041_b200/libdpq_b200.so
  timeout 300 python bench.py --config llama2_70b_slice --target 4.0 --steps 10 --warmup 3 --no-cpu-baseline --skip-static > gpurun_out/b70_${TAG}_$v.log 2>&1
  timeout 200 python tools/stage_stamps.py > gpurun_out/stamps_${TAG}_$v.log 2>&1
  echo "== $v"; python -c "
import json; d=json.loads(open('gpurun_out/b70_${TAG}_$v.log').read().strip().splitlines()[-1]); print('70b slice', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; head -1 gpurun_out/stamps_${TAG}_$v.log
done
cp /tmp/base.so paper_2508_06041_b200/libdpq_b200.so
