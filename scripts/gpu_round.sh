#!/bin/bash
# Full 1-GPU evidence pass: bench lines (cfg2 headline, cfg5, reference arm),
# then the ncu launch list + full capture for the dominant kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${TAG}.csv 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}_cfg2.log 2>&1; echo "bench cfg2 rc=$?"
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg5.log 2>&1; echo "bench cfg5 rc=$?"
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline --steps 312 > gpurun_out/bench_${TAG}_cfg3.log 2>&1; echo "bench cfg3 rc=$?"
timeout 900 python bench.py --dtype bf16 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg2bf16.log 2>&1; echo "bench cfg2 bf16 rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_${TAG}_ref.log 2>&1; echo "bench ref rc=$?"
timeout 900 python bench.py --impl reference --workload cfg5 --steps 4 --warmup 1 > gpurun_out/bench_${TAG}_ref5.log 2>&1; echo "bench ref5 rc=$?"
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
CMD5="python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 && timeout 600 $CMD5 > gpurun_out/plain5_${TAG}.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'augment_crop|k_permute|k_assign' -s 3 -c 4 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches5_${TAG}.csv $CMD5 > /dev/null 2>&1; echo "launches5 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:'augment_resize|resize_prep' -s 3 -c 2 -o gpurun_out/prof5_${TAG} $CMD5 > gpurun_out/ncu_full5_${TAG}.log 2>&1; echo "full5 rc=$?"
for f in gpurun_out/bench_${TAG}_*.log; do echo $f; tail -1 $f | cut -c1-400; done
