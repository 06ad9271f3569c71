# r2ah (2 GPUs): P2P exchange NVLink GB/s in the bench line (cfg4 / cfg2 at N = 2) + parity of the touched paths
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "p2p" > gpurun_out/r2ah_multi.log 2>&1; echo rc=$? >> gpurun_out/r2ah_multi.log
for w in cfg4 cfg2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --workload $w --steps 624 --warmup 20 --no-e2e > /tmp/o.json 2>> gpurun_out/r2ah_bench.err
  python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]; x=d['exchange']
print('$w', round(d['value']/1e6,3), round(d['ms_per_step'],4), x and round(x['nvlink_gbs'],1), x and round(x['frac'],3), x and x['recv_bytes_per_step'])
" >> gpurun_out/r2ah_ab.txt
done
tail -2 gpurun_out/r2ah_multi.log; cat gpurun_out/r2ah_ab.txt
