#!/bin/bash
# K7 next-band L2 prefetch variant + ncu of the current K7
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash scripts/gpu_k7var.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_rows' -s 3 -c 1 \
    -o gpurun_out/prof_k7l2 python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k7l2.log 2>&1
echo "ncu rc=$?"
