# r2al: NCCL knobs with registered exchange buffers, cfg4 over NCCL at N=2 (+ standalone probe at each)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'nvl', round(x.get('nvlink_gbs') or 0,1), 'wire', round(x.get('wire_ms_per_step') or 0,4))
" >> gpurun_out/r2al_ab.txt 2>&1; }
for knob in "" "NCCL_P2P_NVL_CHUNKSIZE=2097152" "NCCL_P2P_NVL_CHUNKSIZE=131072" "NCCL_MIN_NCHANNELS=32" "NCCL_MAX_NCHANNELS=16" "NCCL_MAX_NCHANNELS=8" "NCCL_NTHREADS=512" "NCCL_PROTO=Simple"; do
  echo "== $knob" >> gpurun_out/r2al_probe.txt
  env $knob timeout 120 ./scripts/nccl_reg_probe.bin 2>&1 | grep -E "registered|Register" | grep -E " 80 MB|160 MB" >> gpurun_out/r2al_probe.txt
  env $knob timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus 2 --workload cfg4 --exchange nccl --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2al.err
  line "cfg4-nccl ${knob:-default}"
done
cat gpurun_out/r2al_probe.txt gpurun_out/r2al_ab.txt
