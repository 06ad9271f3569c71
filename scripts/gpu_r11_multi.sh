#!/bin/bash
# final multi-GPU evidence (4-GPU box): every workload at N=2 and N=4, NCCL regular scheme, multi tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for N in 2 4; do
  N=$N TAG=r11 STEPS=624 bash scripts/gpu_multi.sh
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2963$N bench.py --gpus $N --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r11_n${N}_cfg4_nccl.log 2>&1
  echo "cfg4 nccl n$N rc=$?"
done
