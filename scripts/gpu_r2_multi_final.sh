#!/bin/bash
# Round-2 multi-GPU evidence of the final build on one 4-GPU box: the
# multi-GPU suite (2- and 4-learner cases), then every workload at N = 2 and
# N = 4 (scripts/gpu_multi.sh), including NCCL variants of cfg2 / cfg4 / cfg5.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for b in tests/cxx/_bin/test_*; do echo "$(basename $b): $($b 2>/dev/null | tail -1)"; done > gpurun_out/cxx_suites_${TAG:-r2x}.txt; cat gpurun_out/cxx_suites_${TAG:-r2x}.txt
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rf > gpurun_out/pytest_multi_${TAG:-r2x}_n4.log 2>&1; echo "multi pytest rc=$?"; tail -2 gpurun_out/pytest_multi_${TAG:-r2x}_n4.log
N=2 TAG=${TAG:-r2x} STEPS=624 bash scripts/gpu_multi.sh
N=4 TAG=${TAG:-r2x} STEPS=624 bash scripts/gpu_multi.sh
