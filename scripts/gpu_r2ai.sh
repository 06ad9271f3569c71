# r2ai (2 GPUs): host-path K7 prologue on the side stream (NCCL / unbalanced host steps)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "host_path or variable" > gpurun_out/r2ai_multi.log 2>&1; echo rc=$? >> gpurun_out/r2ai_multi.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host or resize or variable" > gpurun_out/r2ai_parity.log 2>&1; echo rc=$? >> gpurun_out/r2ai_parity.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --workload cfg5 --exchange nccl --steps 624 --warmup 20 > /tmp/o.json 2>> gpurun_out/r2ai_bench.err
python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]
print('cfg5-nccl', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3))
" >> gpurun_out/r2ai_ab.txt
tail -2 gpurun_out/r2ai_multi.log; tail -2 gpurun_out/r2ai_parity.log; cat gpurun_out/r2ai_ab.txt
