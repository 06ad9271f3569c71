#!/bin/bash
# K6 storage-tier samples via TMA bulk copies: parity, cfg3 A/B (1 GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for V in default tmast; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python -m pytest tests -q -m gpu -k "storage or augment or loader" --timeout 300 > gpurun_out/pytest_var_$V.log 2>&1
  echo "$V pytest rc=$? $(tail -1 gpurun_out/pytest_var_$V.log)"
done
for R in 1 2; do
for V in default tmast; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 600 python bench.py --workload cfg3 --steps 312 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V cfg3', round(l['value']), round(l['storage_roofline']['achieved'],1), round(l['storage_roofline']['frac'],3), round(l['kernel_ms']['augment_crop']*1000,1))"
done
done
unset LL_LIB
timeout 600 python bench.py --steps 624 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('default cfg2', round(l['value']), round(l['roofline']['frac'],4))"
