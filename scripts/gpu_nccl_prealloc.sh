#!/bin/bash
# NCCL exchange buffers preallocated at comm_init: 4-learner tests and cfg2/cfg4 NCCL at N=4,
# default build and the crop-window variant (variants/lib_win2.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'host', round(l['host_enqueue_ms_per_step'],3))" 2>/dev/null || echo "$1 FAILED"; }
for V in default win2; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 500 python -m pytest tests/test_gpu_multi.py -q --timeout 240 -rf -k "nccl" > gpurun_out/prealloc_pytest_$V.log 2>&1
  echo "$V pytest rc=$? $(tail -1 gpurun_out/prealloc_pytest_$V.log)"
  for W in cfg2 cfg4; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
       --master-port 2968$i bench.py --gpus 4 --workload $W --exchange nccl --steps 312 --no-cpu-baseline > gpurun_out/prealloc_${V}_$W.log 2>&1
    cat gpurun_out/prealloc_${V}_$W.log | show "$V $W nccl n4"
  done
done
