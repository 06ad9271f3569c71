#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 600 -rf > gpurun_out/pytest_multi.log 2>&1; echo "multi rc=$?"; tail -2 gpurun_out/pytest_multi.log
for X in nccl p2p; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 624 --exchange $X 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$X', round(l['value']), round(l['ms_per_step'],4), 'e2e', round(l['e2e']['value']), l['kernel_ms'])"
done
