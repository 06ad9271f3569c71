#!/bin/bash
# final build on a 4-GPU box: every GPU test (1/2/4-GPU), N=1 lines, N=2/4 multi evidence
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -rf > gpurun_out/pytest_r14.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r14.log)"
grep -E "^FAILED" gpurun_out/pytest_r14.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r14.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bench_r14_cfg2.log 2>&1; echo "n1 cfg2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_r14_cfg5.log 2>&1; echo "n1 cfg5 rc=$?"
for N in 2 4; do
  N=$N TAG=r14 STEPS=624 bash scripts/gpu_multi.sh
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 2969$N bench.py --gpus $N --workload cfg4 --exchange nccl --steps 312 > gpurun_out/bench_r14_n${N}_cfg4_nccl.log 2>&1
  echo "cfg4 nccl n$N rc=$?"
done
