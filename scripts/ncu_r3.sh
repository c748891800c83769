P='{"kernel":1}'
python scripts/sweep.py --rows 16384 --reps 0 --plans "$P" > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_cluster" -c 1 -o gpurun_out/prof_r3 python scripts/sweep.py --rows 16384 --reps 0 --plans "$P" > gpurun_out/ncu_r3.log 2>&1
echo rc=$? >> gpurun_out/ncu_r3.log
