#!/bin/bash
# cfg5 at N=2/4: per-rank K7 / pull times (why K7 is slower than at N=1)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-c5m}
for N in 2 4; do
  LL_BENCH_RANK_STATS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2951$N bench.py --gpus $N --workload cfg5 --steps 624 --no-e2e > gpurun_out/bench_${TAG}_n$N.log 2> gpurun_out/bench_${TAG}_n$N.err
  echo "N=$N rc=$?"; grep kernel_ms gpurun_out/bench_${TAG}_n$N.err | cut -c1-300
  tail -1 gpurun_out/bench_${TAG}_n$N.log | cut -c1-200
done
N=4
LL_BENCH_RANK_STATS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port 29519 bench.py --gpus $N --steps 624 --no-e2e > gpurun_out/bench_${TAG}_n4_cfg2.log 2> gpurun_out/bench_${TAG}_n4_cfg2.err
echo "N=4 cfg2 rc=$?"; grep kernel_ms gpurun_out/bench_${TAG}_n4_cfg2.err | cut -c1-300
tail -1 gpurun_out/bench_${TAG}_n4_cfg2.log | cut -c1-200
