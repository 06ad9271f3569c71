#!/bin/bash
# K7 variants A/B (cfg5, 1 GPU): LL_LIB=variants/lib_<v>.so; parity of each variant first
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for V in ${VARIANTS:-default}; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python -m pytest tests -q -m gpu -k "resize or variable" --timeout 300 > gpurun_out/pytest_var_$V.log 2>&1
  echo "$V pytest rc=$? $(tail -1 gpurun_out/pytest_var_$V.log)"
done
for V in ${VARIANTS:-default} ${VARIANTS:-default}; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 1560 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V', round(l['value']), round(l['roofline']['frac'],4), round(l['kernel_ms']['augment_resize']*1000,1))"
done
