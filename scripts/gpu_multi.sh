#!/bin/bash
# multi-GPU: exchange tests + bench at N=2 (p2p and nccl)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${N:-2}
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 600 -rf > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?"; tail -5 gpurun_out/pytest_multi.log
for X in p2p nccl; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port 29511 bench.py --gpus $N --steps 312 --warmup 5 --exchange $X > gpurun_out/bench_n${N}_${X}.log 2>&1
echo "bench $X rc=$?"; tail -2 gpurun_out/bench_n${N}_${X}.log | cut -c1-600
done
