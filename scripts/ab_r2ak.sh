# r2ak: NCCL exchange buffers from ncclMemAlloc + ncclCommRegister (LL_NCCL_REGISTER=1,
# new default) vs cudaMalloc (=0); standalone send/recv probe first; 2 GPUs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
(timeout 120 ./scripts/nccl_reg_probe.bin; echo "--- torch-bundled nccl";
 LD_LIBRARY_PATH=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib timeout 120 ./scripts/nccl_reg_probe.bin) > gpurun_out/r2ak_probe.txt 2>&1
cat gpurun_out/r2ak_probe.txt
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2ak_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ak_pytest.log
tail -2 gpurun_out/r2ak_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}; e=l.get('e2e') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), round(l['roofline']['frac'],3), 'nvl', x.get('nvlink_gbs'), x.get('wire_ms_per_step'), 'e2e', round(e.get('value',0)/1e6,3), l['clocks']['sm_mhz'])
" >> gpurun_out/r2ak_ab.txt 2>&1; }
for i in 1 2; do
  for v in 1 0; do
    for w in "cfg4" "cfg4 --dtype bf16" "cfg2" "cfg5"; do
      LL_NCCL_REGISTER=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 bench.py --gpus 2 --workload $w --exchange nccl --steps 312 --no-cpu-baseline > /tmp/o.json 2>>gpurun_out/r2ak.err
      line "n2-nccl-${w// /}-reg$v"
    done
  done
done
cat gpurun_out/r2ak_ab.txt
