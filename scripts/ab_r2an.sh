# r2an: N=4 NCCL regression hunt: registration x chunk size for cfg2/cfg5 over NCCL
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'nvl', round(x.get('nvlink_gbs') or 0,1), 'wire', round(x.get('wire_ms_per_step') or 0,4))
" >> gpurun_out/r2an_ab.txt 2>&1; }
for v in "LL_NCCL_REGISTER=1 NCCL_P2P_NVL_CHUNKSIZE=131072" "LL_NCCL_REGISTER=1 NCCL_P2P_NVL_CHUNKSIZE=524288" "LL_NCCL_REGISTER=0 NCCL_P2P_NVL_CHUNKSIZE=131072" "LL_NCCL_REGISTER=0 NCCL_P2P_NVL_CHUNKSIZE=524288"; do
  for w in cfg2 cfg5 cfg4; do
    env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus 4 --workload $w --exchange nccl --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2an.err
    line "n4 $w $v"
  done
done
cat gpurun_out/r2an_ab.txt
