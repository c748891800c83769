#!/bin/bash
# one ncu --set full capture of the tcgen05 forward kernel (first launch after warm-up)
python paper_2604_26256_b200/build.py >/dev/null
timeout 300 python scripts/bench_lmhead.py --skip-unfused --steps 2 --warmup 1 > gpurun_out/lm_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmhead_kernel -s 2 -c 2 \
  -o gpurun_out/lmhead_full -f python scripts/bench_lmhead.py --skip-unfused --steps 1 --warmup 1 \
  > gpurun_out/lm_ncu.log 2>&1
tail -3 gpurun_out/lm_ncu.log
