#!/bin/bash
# 4-GPU box: every GPU test (multi-GPU ones included), then per-rank cfg5 / cfg2 stats at N=2/4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r05c.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r05c.log)"
bash scripts/gpu_cfg5_multi.sh
