#!/bin/bash
# Round-2 1-GPU evidence of the final build: the GPU suite, smoke, the bench
# lines (cfg2 fp32 / bf16, cfg3, cfg5, reference arms) and the ncu launch
# lists + full captures of K6 and K7 (scripts/gpu_round.sh).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r2x}
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
TAG=$TAG bash scripts/gpu_round.sh
