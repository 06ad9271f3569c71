#!/bin/bash
# K6 / K7 prefetch variants (1 GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for V in default k6pf nol1pf; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python -m pytest tests -q -m gpu -k "augment or loader" --timeout 300 > gpurun_out/pytest_var_$V.log 2>&1
  echo "$V pytest rc=$? $(tail -1 gpurun_out/pytest_var_$V.log)"
done
for R in 1 2; do
for V in default k6pf; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  for D in fp32 bf16; do
  timeout 600 python bench.py --dtype $D --steps 1560 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V $D', round(l['value']), round(l['roofline']['frac'],4), round(l['kernel_ms']['augment_crop']*1000,1))"
  done
done
for V in default nol1pf; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 1560 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V cfg5', round(l['value']), round(l['roofline']['frac'],4), round(l['kernel_ms']['augment_resize']*1000,1))"
done
done
