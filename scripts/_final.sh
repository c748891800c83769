# end-of-round evidence run (one GPU): smoke, the -m gpu suite, bench lines, precision fuzz,
# launch list + full ncu capture of the dominant kernel, full capture of the LM-head GEMMs
set -x
cd $GRAFT_REPO_ROOT
D=gpurun_out/final; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1
echo smoke_exit $? >> $D/status.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 > $D/gpu_tests.log 2>&1
echo tests_exit $? >> $D/status.txt
python bench.py > $D/bench_prod.json 2> $D/bench_prod.err
echo bench_prod_exit $? >> $D/status.txt
python bench.py --config large --no-cpu-baseline > $D/bench_large.json 2> $D/bench_large.err
echo bench_large_exit $? >> $D/status.txt
python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref.json 2> $D/bench_ref.err
echo bench_ref_exit $? >> $D/status.txt
timeout 900 python scripts/precision_fuzz.py 200 0 > $D/prec.jsonl 2> $D/prec.err
echo prec_exit $? >> $D/status.txt
timeout 1200 bash scripts/profile_round.sh > $D/profile_round.log 2>&1
echo profile_exit $? >> $D/status.txt
timeout 300 python scripts/bench_lmhead.py --skip-unfused --steps 2 --warmup 1 > $D/lm_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lmhead_kernel|gemm_kernel" -s 2 -c 4 \
  -o gpurun_out/lmhead_gemms_full -f python scripts/bench_lmhead.py --skip-unfused --steps 1 --warmup 1 > $D/lm_ncu.log 2>&1
echo lm_ncu_exit $? >> $D/status.txt
