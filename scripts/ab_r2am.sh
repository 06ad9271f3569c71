# r2am: NCCL_P2P_NVL_CHUNKSIZE sweep with registered exchange buffers, every workload over NCCL at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'nvl', round(x.get('nvlink_gbs') or 0,1), 'wire', round(x.get('wire_ms_per_step') or 0,4))
" >> gpurun_out/r2am_ab.txt 2>&1; }
for cs in 524288 262144 131072 65536 32768; do
  for w in "cfg4" "cfg4 --dtype bf16" "cfg2" "cfg5"; do
    NCCL_P2P_NVL_CHUNKSIZE=$cs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus 2 --workload $w --exchange nccl --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2am.err
    line "chunk=$cs ${w// /}"
  done
done
cat gpurun_out/r2am_ab.txt
