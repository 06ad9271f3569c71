# r2n (2 GPUs): NCCL send/recv on their own stream (host-driven prologues no
# longer queue behind them): multi-GPU suite, cfg4 / cfg2 over NCCL at N = 2
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2n_multi.log 2>&1; echo rc=$? >> gpurun_out/r2n_multi.log
for w in cfg4 cfg2 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload $w --exchange nccl --steps 624 --warmup 20 > /tmp/o.json 2>> gpurun_out/r2n_bench.err
  grep '^{' /tmp/o.json >> gpurun_out/r2n_bench.jsonl
  python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]; x=d['exchange']
print('$w', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(x['wire_ms_per_step'],4), round(x['pack_ms_per_step'],4), round(x['nvlink_gbs'],1), round(x['frac'],3), 'e2e', d['e2e'] and round(d['e2e']['value']/1e6,3))
" >> gpurun_out/r2n_ab.txt
done
tail -2 gpurun_out/r2n_multi.log; cat gpurun_out/r2n_ab.txt
