#!/bin/bash
# r05 multi-GPU evidence on a 4-GPU box: 1/2/4-GPU cfg2 lines, every workload at N=4,
# the 2/4-GPU exchange tests, and cfg3's storage-tier roofline at N=1.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg3 --steps 312 --no-cpu-baseline > gpurun_out/bench_r05_n1_cfg3.log 2>&1
echo "cfg3 n1 rc=$?"; tail -1 gpurun_out/bench_r05_n1_cfg3.log | cut -c1-300
timeout 600 python bench.py --steps 624 --no-cpu-baseline > gpurun_out/bench_r05_n1_cfg2.log 2>&1; echo "cfg2 n1 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 624 > gpurun_out/bench_r05_n2_cfg2_p2p.log 2>&1
echo "cfg2 n2 rc=$?"; tail -1 gpurun_out/bench_r05_n2_cfg2_p2p.log | cut -c1-200
N=4 TAG=r05 bash scripts/gpu_multi.sh
