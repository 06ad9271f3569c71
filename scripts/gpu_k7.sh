#!/bin/bash
# K7 iteration: resize parity tests, cfg5 bench (fp32/bf16), one ncu capture of the band kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${TAG:-k7}
timeout 600 python -m pytest tests -q -m gpu -k "resize or variable" --timeout 300 > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/bench_${TAG}_cfg5.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench_${TAG}_cfg5.log | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print(round(l['value']), l['ms_per_step'], l['roofline'], l.get('e2e',{}).get('value'))"
CMD="python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'resize_band' -s 3 -c 1 \
    -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full_${TAG}.log
