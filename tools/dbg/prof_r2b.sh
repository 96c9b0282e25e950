# ncu pass of the round-end engine: full capture of one decode launch + the bench launch list
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel --profile-from-start off -c 1 -o gpurun_out/eng_r2b python tools/ncu_engine.py > gpurun_out/ncu_r2b.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:engine_kernel --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 4 --warmup 3 --skip-static --no-cpu-baseline > gpurun_out/ncu_bench_r2b.log 2>&1
tail -3 gpurun_out/ncu_r2b.log
