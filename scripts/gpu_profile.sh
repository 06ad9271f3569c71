#!/bin/bash
# launch list + full ncu capture of the top kernels (1 GPU)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r01}
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_${TAG}.log; exit 1; }
echo "plain ok"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'augment_crop|k_permute|k_assign' -s 3 -c 4 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full_${TAG}.log
ls -la gpurun_out
