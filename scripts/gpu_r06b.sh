#!/bin/bash
# 2-GPU box: all GPU tests, cfg5 N=1 (pitched generator), cfg2 NCCL N=2 twice (spread)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r06b.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r06b.log)"
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'host', round(l['host_enqueue_ms_per_step'],3), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items()})"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | show "cfg5 n1"
for i in 1 2 3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 2957$i bench.py --gpus 2 --exchange nccl --steps 624 2>&1 | show "cfg2 n2 nccl #$i"
done
nproc; cat /proc/cpuinfo | grep "model name" | head -1
