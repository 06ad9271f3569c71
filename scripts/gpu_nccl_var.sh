#!/bin/bash
# NCCL-exchange host stalls: cfg2 nccl N=2 with and without the NVML clock sampler
cd "$GRAFT_REPO_ROOT" || exit 1
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'host', round(l['host_enqueue_ms_per_step'],3), 'e2e', l['e2e'] and round(l['e2e']['value']))"; }
for i in 1 2 3; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 2958$i bench.py --gpus 2 --exchange nccl --steps 624 --no-cpu-baseline 2>&1 | show "clocks #$i"
  LL_BENCH_NO_CLOCKS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 2959$i bench.py --gpus 2 --exchange nccl --steps 624 --no-cpu-baseline 2>&1 | show "noclk  #$i"
done
