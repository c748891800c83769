# Round profiling: plain bench, launch list, one full capture of the top kernel.
set -x
python paper_2604_26256_b200/build.py > /dev/null
python bench.py --steps 2 --warmup 1 > gpurun_out/prof_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_plain_bench2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rowwise_kernel|fused_cluster|stream_kernel" -s 8 -c 1 -o gpurun_out/prof_bench_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
