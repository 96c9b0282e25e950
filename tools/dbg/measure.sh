# one GPU measurement pass: gpu tests (optional), bench, selector split, stage stamps
# usage: bash tools/dbg/measure.sh TAG [tests]
TAG=${1:-x}
if [ "$2" = "tests" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputest_$TAG.log; tail -3 gpurun_out/gputest_$TAG.log; fi
if [ "$2" = "parity" ]; then timeout 900 python -m pytest tests/test_gpu_parity_widths.py tests/test_gpu_runtime.py tests/test_gpu_api.py -x -q 2>&1 | tail -15 > gpurun_out/gputest_$TAG.log; tail -3 gpurun_out/gputest_$TAG.log; fi
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
timeout 300 python tools/selector_split.py > gpurun_out/split_$TAG.log 2>&1
timeout 200 python tools/stage_stamps.py > gpurun_out/stamps_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log | cut -c1-400
tail -2 gpurun_out/split_$TAG.log
head -7 gpurun_out/stamps_$TAG.log
