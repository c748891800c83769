set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t20
python scripts/bench_lmhead.py --steps 1 --warmup 1 --skip-unfused > gpurun_out/t20/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 2 \
    -o gpurun_out/t20/gemm python scripts/bench_lmhead.py --steps 1 --warmup 1 --skip-unfused > gpurun_out/t20/ncu_gemm.log 2>&1 && \
ncu --set full --clock-control none -k regex:lmhead_kernel -c 2 \
    -o gpurun_out/t20/lmhead python scripts/bench_lmhead.py --steps 1 --warmup 1 --skip-unfused > gpurun_out/t20/ncu_lmhead.log 2>&1
