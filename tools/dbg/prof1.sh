set -x
timeout 200 python tools/stage_stamps.py --static 3 > gpurun_out/stamps_s3.log 2>&1
timeout 200 python tools/stage_stamps.py --static 4 > gpurun_out/stamps_s4.log 2>&1
timeout 300 python tools/selector_split.py > gpurun_out/split.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:engine_kernel --profile-from-start off -c 1 -o gpurun_out/eng_v3 python tools/ncu_engine.py > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
