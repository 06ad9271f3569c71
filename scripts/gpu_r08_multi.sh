#!/bin/bash
# 4-GPU box: TMA-for-peer-samples A/B and NCCL host-stall probe, then the r08 multi-GPU evidence
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash scripts/gpu_tmafar.sh
for N in 2 4; do
  N=$N TAG=r08 STEPS=624 bash scripts/gpu_multi.sh
done
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2956$N bench.py --gpus $N --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r08_n${N}_cfg4_nccl.log 2>&1
  echo "cfg4 nccl n$N rc=$?"
done
