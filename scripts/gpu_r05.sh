#!/bin/bash
# Round evidence pass at HEAD: GPU tests, smoke, then the 1-GPU bench/ncu pass.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r05}
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 -rf > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
TAG=$TAG bash scripts/gpu_round.sh
