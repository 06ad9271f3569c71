#!/bin/bash
# host-path NCCL exchange on the side stream (double-buffered): every GPU test (1/2/4 GPUs), smoke, NCCL bench lines at N=2/4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r17.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r17.log)"
grep -E "^FAILED" gpurun_out/pytest_r17.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r17.log 2>&1; echo "smoke rc=$?"
for N in 2 4; do
  for w in cfg2 cfg4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
       --master-port 2999$N bench.py --gpus $N --workload $w --exchange nccl --steps 312 > gpurun_out/bench_r17_n${N}_${w}_nccl.log 2>&1
    echo "$w nccl n$N rc=$?"; tail -1 gpurun_out/bench_r17_n${N}_${w}_nccl.log | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(round(l['value']), 'e2e', round(l['e2e']['value']))"
  done
done
