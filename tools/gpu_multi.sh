# multi-rank bench path on ONE GPU (ranks share cuda:0, gather over gloo): N = 2, 4
export SHB_BENCH_SHARE_GPU=1
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 --json-out gpurun_out/bench_share$N.json > gpurun_out/bench_share$N.log 2>&1; echo "N=$N rc=$?"; tail -1 gpurun_out/bench_share$N.log | cut -c1-400
done
unset SHB_BENCH_SHARE_GPU
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tr1.log 2>&1; echo "torchrun N=1 rc=$?"; tail -1 gpurun_out/bench_tr1.log | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref2.log 2>&1; echo "ref N=2 rc=$?"; tail -1 gpurun_out/bench_ref2.log | cut -c1-300
