set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t15
for V in 152064 180000 200000 230000 262144; do
  python scripts/sweep.py --config large --vocab $V --rows 65536 --reps 3 --plans '{"kernel":3,"chunk_kb":32,"stages":6,"lag":3};{"kernel":3,"chunk_kb":32,"stages":6,"lag":1};{"kernel":3,"chunk_kb":32,"stages":6,"lag":3,"cluster_size":2}' >> gpurun_out/t15/split_sweep.jsonl 2>> gpurun_out/t15/split_sweep.err
done
timeout 1500 python -m pytest tests/test_gpu_golden.py -q --timeout 1200 > gpurun_out/t15/golden.log 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/t15/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 2 -c 1 \
    -o gpurun_out/t15/k3c python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/t15/ncu.log 2>&1
