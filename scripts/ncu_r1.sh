P='{"kernel":1};{"kernel":2}'
python scripts/sweep.py --rows 16384 --reps 1 --plans "$P" > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_cluster|rowwise" -c 2 -o gpurun_out/prof_r1 python scripts/sweep.py --rows 16384 --reps 1 --plans "$P" > gpurun_out/ncu_r1.log 2>&1
echo rc=$? >> gpurun_out/ncu_r1.log
