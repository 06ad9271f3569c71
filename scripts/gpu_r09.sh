#!/bin/bash
# TMA for all far samples + 20 ms clock sampler: GPU tests; K7 two-columns A/B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/pytest_r09.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_r09.log)"
grep -E "^FAILED" gpurun_out/pytest_r09.log | head
bash scripts/gpu_k7var.sh
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), 'e2e', l['e2e'] and round(l['e2e']['value']), 'host', round(l['host_enqueue_ms_per_step'],3), l['clocks'].get('samples'))"; }
timeout 600 python bench.py --no-cpu-baseline 2>&1 | show "cfg2"
