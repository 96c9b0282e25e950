# run stage stamps + bench for each prebuilt library variant: bash tools/dbg/variants.sh TAG v1 v2 ...
TAG=$1; shift
cp paper_2508_06041_b200/libdpq_b200.so /tmp/base.so
for v in "$@"; do
  cp paper_2508_06041_b200/libdpq_b200_$v.so paper_2508_06041_b200/libdpq_b200.so
  touch paper_2508_06041_b200/libdpq_b200.so
  timeout 200 python tools/stage_stamps.py > gpurun_out/stamps_${TAG}_$v.log 2>&1
  timeout 200 python tools/stage_stamps.py --static 3 > gpurun_out/stamps_${TAG}_${v}_s3.log 2>&1
  echo "== $v"; head -1 gpurun_out/stamps_${TAG}_$v.log; head -1 gpurun_out/stamps_${TAG}_${v}_s3.log
done
cp /tmp/base.so paper_2508_06041_b200/libdpq_b200.so
