#!/bin/bash
# r06 multi-GPU evidence (4-GPU box): every workload at N=2 and N=4, plus the multi-GPU tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for N in 2 4; do
  N=$N TAG=r06 STEPS=624 bash scripts/gpu_multi.sh
done
N=2; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29561 bench.py --gpus 2 --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r06_n2_cfg4_nccl.log 2>&1
echo "cfg4 nccl n2 rc=$?"
N=4; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
   --master-port 29562 bench.py --gpus 4 --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r06_n4_cfg4_nccl.log 2>&1
echo "cfg4 nccl n4 rc=$?"
