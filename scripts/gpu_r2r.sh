# r2r (2 GPUs): K7 prologue prefetched in NCCL mode too (cfg5 over NCCL), and
# K6 bf16 at 5 CTAs / SM: parity + multi suite + cfg5 NCCL / P2P at N = 2
python -m pytest tests -m gpu -x -q -k "crop or unaligned or resize or variable or cfg5" > gpurun_out/r2r_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2r_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "variable or storage or exchange" > gpurun_out/r2r_multi.log 2>&1; echo rc=$? >> gpurun_out/r2r_multi.log
for ex in nccl p2p; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --workload cfg5 --exchange $ex --steps 624 --warmup 20 > /tmp/o.json 2>> gpurun_out/r2r_bench.err
  python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]
print('cfg5-$ex', round(d['value']/1e6,3), round(d['ms_per_step'],4), 'e2e', d['e2e'] and round(d['e2e']['value']/1e6,3))
" >> gpurun_out/r2r_ab.txt
done
tail -2 gpurun_out/r2r_pytest.log; tail -2 gpurun_out/r2r_multi.log; cat gpurun_out/r2r_ab.txt
