# round-end bench lines for profiles/: bash tools/dbg/final_bench.sh
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fb_8b.log 2>&1; tail -1 gpurun_out/fb_8b.log > gpurun_out/r2_bench_8b.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --config llama2_7b --target 3.5 --no-cpu-baseline > gpurun_out/fb_7b35.log 2>&1; tail -1 gpurun_out/fb_7b35.log > gpurun_out/r2_bench_llama2_7b_t3.5.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --config llama2_7b --target 4.5 --no-cpu-baseline > gpurun_out/fb_7b45.log 2>&1; tail -1 gpurun_out/fb_7b45.log > gpurun_out/r2_bench_llama2_7b_t4.5.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --config cfg1 --no-cpu-baseline > gpurun_out/fb_cfg1.log 2>&1; tail -1 gpurun_out/fb_cfg1.log > gpurun_out/r2_bench_cfg1_refplan.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --async-estimators --no-cpu-baseline > gpurun_out/fb_async.log 2>&1; tail -1 gpurun_out/fb_async.log > gpurun_out/r2_bench_8b_async_estimators.jsonl
timeout 1500 python bench.py --steps 10 --warmup 3 --config llama2_70b --target 4.0 --no-cpu-baseline > gpurun_out/fb_70b.log 2>&1; tail -1 gpurun_out/fb_70b.log > gpurun_out/r2_bench_llama2_70b_full_t4.0.jsonl
for f in gpurun_out/r2_bench_*.jsonl; do echo $f; cut -c1-200 $f; done
