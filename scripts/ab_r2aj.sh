# r2aj: K6 peer windows pulled ahead on the side stream (LL_CROP_PULL=1, new
# default) vs fused TMA reads of peer shards inside K6 (LL_CROP_PULL=0); 2 GPUs
# (the side-stream pull build measured here was removed afterwards; LL_CROP_PULL no longer exists)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2aj_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2aj_pytest.log
tail -2 gpurun_out/r2aj_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}; e=l.get('e2e') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), round(l['roofline']['frac'],3), x.get('nvlink_gbs'), 'e2e', round(e.get('value',0)/1e6,3), l['clocks']['sm_mhz'], l.get('kernel_ms'))
" >> gpurun_out/r2aj_ab.txt 2>&1; }
for i in 1 2; do
  for v in 1 0; do
    for w in "cfg4" "cfg4 --dtype bf16" "cfg2"; do
      LL_CROP_PULL=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 bench.py --gpus 2 --workload $w --steps 312 --no-cpu-baseline > /tmp/o.json 2>>gpurun_out/r2aj.err
      line "n2-${w// /}-pull$v"
    done
  done
done
cat gpurun_out/r2aj_ab.txt
