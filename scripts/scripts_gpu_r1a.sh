#!/bin/bash
# first GPU pass: parity tests, smoke, short bench (no profiler)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py --steps 312 --warmup 5 --cpu-seconds 10 > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -5 gpurun_out/pytest_gpu.log
tail -3 gpurun_out/smoke.log
tail -2 gpurun_out/bench.log
