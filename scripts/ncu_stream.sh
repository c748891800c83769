#!/bin/bash
# ncu --set full of the K3c stream kernel on a 65536-row prod chunk
PLAN=${1:-'{"kernel":3}'}
python paper_2604_26256_b200/build.py >/dev/null
timeout 200 python scripts/sweep.py --rows 65536 --reps 1 --plans "$PLAN" > gpurun_out/stream_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 \
  -o gpurun_out/stream_full -f python scripts/sweep.py --rows 65536 --reps 0 --plans "$PLAN" > gpurun_out/stream_ncu.log 2>&1
tail -2 gpurun_out/stream_ncu.log
