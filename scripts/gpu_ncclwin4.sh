#!/bin/bash
# cfg2 NCCL at N=4 with logs kept (window slots)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
   --master-port 2964$i bench.py --gpus 4 --exchange nccl --steps 312 > gpurun_out/ncclwin4_$i.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncclwin4_$i.log | cut -c1-300
done
