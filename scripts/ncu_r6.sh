P='{"kernel":2}'
python scripts/sweep.py --rows 32768 --reps 0 --plans "$P" > gpurun_out/plain6.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rowwise" -c 1 -o gpurun_out/prof_r6 python scripts/sweep.py --rows 32768 --reps 0 --plans "$P" > gpurun_out/ncu_r6.log 2>&1
echo rc=$? >> gpurun_out/ncu_r6.log
