set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t16
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29513"
cp paper_2604_26256_b200/libgrpo_async.so abtmp/cur.so
for v in v1 v2; do
  cp abtmp/vp_$v.so paper_2604_26256_b200/libgrpo_async.so
  timeout 600 $TR --nproc-per-node 4 scripts/vp_multi_gpu.py > gpurun_out/t16/vp4_$v.log 2>&1
done
cp abtmp/cur.so paper_2604_26256_b200/libgrpo_async.so
timeout 600 $TR --nproc-per-node 4 scripts/vp_multi_gpu.py > gpurun_out/t16/vp4_cur.log 2>&1
