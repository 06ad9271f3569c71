#!/bin/bash
# final build, 4-GPU box: multi-GPU tests and bench lines at N=2 and N=4 for every workload
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for N in 2 4; do
  N=$N TAG=r14 STEPS=624 bash scripts/gpu_multi.sh
done
