#!/bin/bash
# A/B of the next-epoch plan prefetch mode (LL_PLAN_PREFETCH) at N GPUs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${N:-4}
for rep in 1 2; do
for mode in stream inline off; do
for ex in p2p nccl; do
  f=gpurun_out/planab_n${N}_${mode}_${ex}_${rep}.log
  LL_PLAN_PREFETCH=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
     --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 1560 --exchange $ex \
     --no-cpu-baseline --no-e2e > $f 2>&1
  echo "$mode $ex rep$rep rc=$? $(tail -1 $f | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(round(l['value']), round(l['ms_per_step'],4), l['kernel_ms'])" 2>&1)"
done; done; done
