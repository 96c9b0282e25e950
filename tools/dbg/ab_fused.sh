timeout 900 python -m pytest tests/test_gpu_parity_widths.py tests/test_gpu_runtime.py tests/test_tp.py -x -q 2>&1 | tail -4
for f in 1 0; do
  DPQ_FUSED_IN=$f timeout 200 python tools/stage_stamps.py > gpurun_out/stamps_fused$f.log 2>&1
  DPQ_FUSED_IN=$f timeout 200 python tools/stage_stamps.py --static 3 > gpurun_out/stamps_fused${f}_s3.log 2>&1
  echo "== fused=$f"; head -7 gpurun_out/stamps_fused$f.log; head -1 gpurun_out/stamps_fused${f}_s3.log
done
