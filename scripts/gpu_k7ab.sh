#!/bin/bash
# K7 variant A/B (LL_K7: 0 = staged smem band kernel, 8/16/32 = global-gather rows kernel)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-k7ab}
for rb in ${RBS:-0 8 16 32}; do
  LL_K7=$rb timeout 600 python -m pytest tests -q -m gpu -k "resize or variable" --timeout 300 > gpurun_out/pytest_${TAG}_$rb.log 2>&1
  echo "rb=$rb pytest rc=$? $(tail -1 gpurun_out/pytest_${TAG}_$rb.log)"
  LL_K7=$rb timeout 600 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 312 > gpurun_out/bench_${TAG}_$rb.log 2>&1
  echo "rb=$rb bench rc=$? $(tail -1 gpurun_out/bench_${TAG}_$rb.log | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print(round(l['value']), round(l['ms_per_step'],4), round(l['roofline']['frac'],3), round(l['roofline']['avg_launch_ms']*1000,1),'us')")"
done
for rb in ${NCU_RBS:-16 32}; do
  LL_K7=$rb timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_(band|rows)' -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_$rb python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_$rb.log 2>&1
  echo "ncu rb=$rb rc=$?"
done
