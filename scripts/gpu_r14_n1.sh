#!/bin/bash
# final build, 1 GPU: every 1-GPU test + smoke, then the full bench/ncu evidence pass
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r14.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r14.log)"
grep -E "^FAILED" gpurun_out/pytest_r14.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r14.log 2>&1; echo "smoke rc=$?"
TAG=r14 bash scripts/gpu_round.sh
