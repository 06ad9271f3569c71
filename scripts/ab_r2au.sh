# r2au: NCCL P2P channel counts with registered buffers (regular scheme), cfg4 over NCCL at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'nvl', round(x.get('nvlink_gbs') or 0,1), 'wire', round(x.get('wire_ms_per_step') or 0,4))
" >> gpurun_out/r2au_ab.txt 2>&1; }
for i in 1 2; do
for knob in "X=1" "NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64" "NCCL_MAX_P2P_NCHANNELS=16" "NCCL_NTHREADS=256" "NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64 NCCL_MIN_NCHANNELS=64 NCCL_MAX_NCHANNELS=64"; do
  for w in "cfg4" "cfg4 --dtype bf16"; do
    env $knob timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus 2 --workload $w --exchange nccl --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2au.err
    line "${w// /} $knob"
  done
done
done
cat gpurun_out/r2au_ab.txt
