# r2ao: NCCL exchange defaults after r2an (registration + 128 KB chunks for the regular
# scheme only; balanced schemes on cudaMalloc buffers and NCCL's default chunks): every
# NCCL workload at N=4 and N=2 on one 4-GPU box, plus the multi-GPU suite at N=4
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}; e=l.get('e2e') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), 'nvl', round(x.get('nvlink_gbs') or 0,1), 'wire', round(x.get('wire_ms_per_step') or 0,4), 'e2e', round(e.get('value',0)/1e6,3))
" >> gpurun_out/r2ao_ab.txt 2>&1; }
for N in 4 2; do
  for w in "cfg2" "cfg5" "cfg4" "cfg4 --dtype bf16"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29531 bench.py --gpus $N --workload $w --exchange nccl --steps 312 --no-cpu-baseline > /tmp/o.json 2>>gpurun_out/r2ao.err
    line "n$N ${w// /}"
  done
done
cat gpurun_out/r2ao_ab.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2ao_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ao_pytest.log; tail -2 gpurun_out/r2ao_pytest.log
