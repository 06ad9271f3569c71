#!/bin/bash
# A/B of augment implementations (parity first)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
IMPLS=${IMPLS:-"0 1 2 3"}
for IMPL in $IMPLS; do
LL_AUG_IMPL=$IMPL timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 400 -k "augment or loader" > gpurun_out/pytest_impl$IMPL.log 2>&1
echo "pytest impl$IMPL rc=$?"; tail -1 gpurun_out/pytest_impl$IMPL.log
done
for IMPL in $IMPLS; do for DT in fp32 bf16; do
LL_AUG_IMPL=$IMPL timeout 600 python bench.py --steps 624 --warmup 5 --no-cpu-baseline --no-e2e --dtype $DT > gpurun_out/ab_${IMPL}_${DT}.log 2>&1
echo "impl $IMPL $DT rc=$?"; tail -1 gpurun_out/ab_${IMPL}_${DT}.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(round(l['value']), round(l['ms_per_step'],5), round(l['roofline']['achieved']), round(l['roofline']['frac'],4), l['kernel_ms']['augment_crop'])"
done; done
