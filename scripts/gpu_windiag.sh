#!/bin/bash
# diagnose the crop-window NCCL variant at 4 learners (variants/lib_win.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_LIB=$PWD/variants/lib_win.so
timeout 600 python -m pytest tests/test_gpu_multi.py -q --timeout 240 -rf -k "four and nccl" > gpurun_out/windiag_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/windiag_pytest.log)"
NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
   --master-port 29671 bench.py --gpus 4 --exchange nccl --steps 312 --no-e2e --no-cpu-baseline > gpurun_out/windiag_bench_noe2e.log 2>&1
echo "bench no-e2e rc=$?"; tail -2 gpurun_out/windiag_bench_noe2e.log | cut -c1-200
