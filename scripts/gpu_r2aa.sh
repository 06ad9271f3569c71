# r2aa (2 GPUs): host steps over NCCL issued once their tables land (submit
# never blocks): multi suite + host-path parity, e2e of cfg2 / cfg4 / cfg5 over NCCL at N = 2
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2aa_multi.log 2>&1; echo rc=$? >> gpurun_out/r2aa_multi.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/r2aa_parity.log 2>&1; echo rc=$? >> gpurun_out/r2aa_parity.log
for w in cfg2 cfg4 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --workload $w --exchange nccl --steps 624 --warmup 20 > /tmp/o.json 2>> gpurun_out/r2aa_bench.err
  python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]
print('$w', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3))
" >> gpurun_out/r2aa_ab.txt
done
tail -2 gpurun_out/r2aa_multi.log; tail -2 gpurun_out/r2aa_parity.log; cat gpurun_out/r2aa_ab.txt
