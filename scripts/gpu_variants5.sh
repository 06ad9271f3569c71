#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for V in default ${VARIANTS}; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 312 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V', round(l['value']), round(l['roofline']['frac'],4), l['kernel_ms'])"
done
