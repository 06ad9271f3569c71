# r2g (2 GPUs): distributed trainer tests (1 and 2 GPUs), then cfg4 over NCCL
# at N = 2 under NCCL tuning variants, with the exchange's NVLink GB/s.
python -m pytest tests/test_gpu_train.py tests/test_gpu_multi.py -x -q -k "trainer" > gpurun_out/r2g_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2g_pytest.log
run() {
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --workload cfg4 --exchange nccl --steps 624 --warmup 20 --no-e2e > /tmp/o.json 2>> gpurun_out/r2g_bench.err
  python -c "
import json; d=[json.loads(l) for l in open('/tmp/o.json') if l.startswith('{')][0]; x=d['exchange']
print('$*', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(x['wire_ms_per_step'],4), round(x['pack_ms_per_step'],4), round(x['nvlink_gbs'],1), round(x['frac'],3))
" >> gpurun_out/r2g_ab.txt
}
run X=0
run NCCL_P2P_NVL_CHUNKSIZE=2097152
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
run NCCL_NCHANNELS_PER_NET_PEER=32 NCCL_MIN_NCHANNELS=32
run NCCL_P2P_USE_CUDA_MEMCPY=1
run NCCL_PROTO=Simple NCCL_P2P_NVL_CHUNKSIZE=1048576 NCCL_MIN_P2P_NCHANNELS=16
run X=0
cat gpurun_out/r2g_ab.txt; tail -3 gpurun_out/r2g_pytest.log
