#!/bin/bash
# N=2 quick checks: resize/loader parity tests, then cfg5 and cfg2 NCCL/P2P bench lines
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-n2ab}
timeout 900 python -m pytest tests -q -m gpu -k "resize or variable or storage or loader" --timeout 400 > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}.log)"
run() {
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 29513 bench.py --gpus 2 --no-e2e "$@" > gpurun_out/bench_${TAG}_${name}.log 2>&1
  echo "bench $name rc=$? $(tail -1 gpurun_out/bench_${TAG}_${name}.log | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(round(l['value']), round(l['ms_per_step'],4), l['kernel_ms'])" 2>&1)"
}
run cfg5 --workload cfg5 --steps 312
run cfg2_nccl --exchange nccl --steps 624
run cfg2_p2p --steps 624
run cfg2_nccl2 --exchange nccl --steps 624
