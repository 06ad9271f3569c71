#!/bin/bash
# NCCL messages as crop windows: 2-GPU tests, cfg2 / cfg4 NCCL at N=2 and N=4 (4-GPU box)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 600 -rf > gpurun_out/pytest_ncclwin.log 2>&1
echo "pytest multi rc=$? $(tail -1 gpurun_out/pytest_ncclwin.log)"
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'host', round(l['host_enqueue_ms_per_step'],3), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items() if v})"; }
for N in 2 4; do
  for W in cfg2 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2962$N bench.py --gpus $N --workload $W --exchange nccl --steps 312 2>&1 | show "$W nccl n$N"
  done
done
