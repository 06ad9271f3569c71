#!/bin/bash
# resize prologue prefetched on the side stream + grid-stride pull: tests, cfg5 N=1/2/4 (4-GPU box)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r05d.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r05d.log)"
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'frac', round(l['roofline']['frac'],4), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items()})"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | show "cfg5 n1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline 2>&1 | show "cfg2 n1"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2952$N bench.py --gpus $N --workload cfg5 --steps 624 2>&1 | show "cfg5 n$N"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2953$N bench.py --gpus $N --steps 624 2>&1 | show "cfg2 n$N"
done
