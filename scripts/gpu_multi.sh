#!/bin/bash
# multi-GPU: exchange tests + bench lines at N GPUs for every workload
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${N:-2}
TAG=${TAG:-r01}
nvidia-smi topo -m > gpurun_out/topo_n${N}.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q --timeout 600 -rf > gpurun_out/pytest_multi_n${N}.log 2>&1
echo "pytest multi rc=$?"; tail -2 gpurun_out/pytest_multi_n${N}.log
run() {
  local name=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 29511 bench.py --gpus $N "$@" > gpurun_out/bench_${TAG}_n${N}_${name}.log 2>&1
  echo "bench $name rc=$?"; tail -1 gpurun_out/bench_${TAG}_n${N}_${name}.log | python -c "
import json,sys
try:
    l=json.loads(sys.stdin.read()); x=l.get('exchange') or {}; print(round(l['value']), round(l['ms_per_step'],4), 'e2e', round(l['e2e']['value']) if l.get('e2e') else None, 'roof', round(l['roofline']['frac'],3), 'nvlink', x.get('nvlink_gbs'))
except Exception as e: print('parse fail', e)"
}
run cfg2_p2p --steps ${STEPS:-624}
run cfg2_nccl --steps ${STEPS:-624} --exchange nccl
run cfg3 --workload cfg3 --steps ${STEPS:-312}
run cfg4 --workload cfg4 --steps ${STEPS:-312}
run cfg4_nccl --workload cfg4 --exchange nccl --steps ${STEPS:-312}
run cfg4_bf16 --workload cfg4 --dtype bf16 --steps ${STEPS:-312}
run cfg4_nccl_bf16 --workload cfg4 --dtype bf16 --exchange nccl --steps ${STEPS:-312}
run cfg5 --workload cfg5 --steps ${STEPS:-312}
run cfg5_nccl --workload cfg5 --exchange nccl --steps ${STEPS:-312}
