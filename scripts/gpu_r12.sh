#!/bin/bash
# e2e with the epoch order D2H into pinned memory: N=1 and N=2/4, cfg2 / cfg5
cd "$GRAFT_REPO_ROOT" || exit 1
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']))"; }
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline 2>&1 | show "cfg2 n1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | show "cfg5 n1"
for N in 2 4; do
  for W in cfg2 cfg5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2965$N bench.py --gpus $N --workload $W --steps 624 2>&1 | show "$W n$N"
  done
done
