set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t17
for v in prev cur2 prev cur2; do
  cp abtmp/$v.so paper_2604_26256_b200/libgrpo_async.so
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/t17/bench_$v.json 2>>gpurun_out/t17/bench.err
done
cp abtmp/cur2.so paper_2604_26256_b200/libgrpo_async.so
timeout 900 python scripts/precision_fuzz.py 200 0 > gpurun_out/t17/prec.jsonl 2> gpurun_out/t17/prec.err
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_closed_forms.py tests/test_gpu_multigpu_step.py -q --timeout 900 > gpurun_out/t17/tests.log 2>&1
