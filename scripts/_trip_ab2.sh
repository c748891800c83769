set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t21
for v in cur2 cur3 cur2 cur3; do
  cp abtmp/$v.so paper_2604_26256_b200/libgrpo_async.so
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/t21/bench_$v.json 2>>gpurun_out/t21/bench.err
done
cp abtmp/cur3.so paper_2604_26256_b200/libgrpo_async.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vocab_parallel.py tests/test_gpu_guard_bands.py -q --timeout 900 > gpurun_out/t21/tests.log 2>&1
