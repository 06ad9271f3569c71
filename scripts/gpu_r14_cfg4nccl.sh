#!/bin/bash
# final build: the regular scheme at full volume over NCCL (crop-window messages), N=2 and N=4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2969$N bench.py --gpus $N --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r14_n${N}_cfg4_nccl.log 2>&1
  echo "cfg4 nccl n$N rc=$?"; tail -1 gpurun_out/bench_r14_n${N}_cfg4_nccl.log | cut -c1-200
done
