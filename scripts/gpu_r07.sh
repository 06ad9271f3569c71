#!/bin/bash
# host-path K7 prologue on the side stream + per-loader tags: GPU tests, cfg5/cfg2 bench (e2e), ncu of K7
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r07.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r07.log)"
grep -E "^FAILED" gpurun_out/pytest_r07.log | head
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'frac', round(l['roofline']['frac'],4), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items()})"; }
timeout 600 python bench.py --workload cfg5 --no-cpu-baseline 2>&1 | show "cfg5"
timeout 600 python bench.py --no-cpu-baseline 2>&1 | show "cfg2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_rows' -s 3 -c 1 \
    -o gpurun_out/prof_r07_k7 python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r07_k7.log 2>&1
echo "ncu rc=$?"
bash scripts/gpu_k7var.sh
LL_LIB=$PWD/variants/lib_ws.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_ws' -s 3 -c 1 \
    -o gpurun_out/prof_r07_ws python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_r07_ws.log 2>&1
echo "ncu ws rc=$?"
