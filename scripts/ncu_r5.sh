P='{"kernel":2,"ctas_per_sm":2,"stages":4,"row_cache":0}'
python scripts/sweep.py --rows 32768 --reps 0 --plans "$P" > gpurun_out/plain5.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rowwise" -c 1 -o gpurun_out/prof_r5 python scripts/sweep.py --rows 32768 --reps 0 --plans "$P" > gpurun_out/ncu_r5.log 2>&1
echo rc=$? >> gpurun_out/ncu_r5.log
