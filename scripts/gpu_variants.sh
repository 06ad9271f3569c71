#!/bin/bash
# A/B of library build variants (variants/*.so) on the cfg2 / cfg2-bf16 bench
cd "$GRAFT_REPO_ROOT" || exit 1
for V in default ${VARIANTS}; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  for DT in fp32 bf16; do
    timeout 600 python bench.py --steps 624 --warmup 5 --no-cpu-baseline --no-e2e --dtype $DT 2>&1 | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$V $DT', round(l['value']), round(l['roofline']['frac'],4), round(l['kernel_ms']['augment_crop']*1000,2),'us')"
  done
done
