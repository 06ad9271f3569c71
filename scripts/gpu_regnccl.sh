#!/bin/bash
# regular scheme over NCCL: 2-GPU parity tests, cfg4 P2P vs NCCL at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 600 -rf > gpurun_out/pytest_regnccl.log 2>&1
echo "pytest multi rc=$?"; tail -3 gpurun_out/pytest_regnccl.log
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items()})"; }
for X in p2p nccl; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 29541 bench.py --gpus 2 --workload cfg4 --exchange $X --steps 312 2>&1 | show "cfg4 n2 $X"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29542 bench.py --gpus 2 --exchange nccl --steps 624 2>&1 | show "cfg2 n2 nccl"
