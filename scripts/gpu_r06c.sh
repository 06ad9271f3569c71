#!/bin/bash
# per-loader scratch names: all GPU tests (1 GPU) + cfg5 bench, then the K7 L2-prefetch A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r06c.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r06c.log)"
grep -E "FAILED|Error" gpurun_out/pytest_r06c.log | head -5
bash scripts/gpu_k7var.sh
