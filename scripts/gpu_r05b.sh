#!/bin/bash
# K7 word-aligned rows + plan priming: GPU tests, K7 A/B vs the r05 binary,
# short-run cfg2 lines (priming), e2e prefetch depth 2 vs 4, K7 ncu.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r05b}
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 -rf > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}.log)"
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'frac', round(l['roofline']['frac'],4), l['kernel_ms'])"; }
for V in default rows default rows; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 1560 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | show "cfg5 $V"
done
unset LL_LIB
for S in 50 624 1560; do
  timeout 600 python bench.py --steps $S --warmup 3 --no-cpu-baseline 2>&1 | show "cfg2 steps=$S"
done
timeout 600 python bench.py --steps 624 --warmup 3 --no-cpu-baseline --prefetch-depth 4 2>&1 | show "cfg2 depth4"
timeout 600 python bench.py --workload cfg5 --steps 624 --warmup 3 --no-cpu-baseline --prefetch-depth 4 2>&1 | show "cfg5 depth4"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_rows' -s 3 -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"
