# NCCL send/recv knob sweep for the exchange (probe alone, 80 MB per peer)
p=29520
for v in "X=0" "NCCL_BUFFSIZE=16777216" "NCCL_BUFFSIZE=33554432 NCCL_P2P_NVL_CHUNKSIZE=2097152" \
         "NCCL_P2P_READ_ENABLE=1" "NCCL_P2P_READ_ENABLE=0" "NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=64" \
         "NCCL_BUFFSIZE=33554432 NCCL_P2P_NVL_CHUNKSIZE=4194304 NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=64" \
         "NCCL_CTA_POLICY=1" "NCCL_P2P_LL_THRESHOLD=0"; do
  p=$((p+1))
  echo "== $v" >> gpurun_out/r2i_sweep.txt
  env $v timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p scripts/nccl_probe.py 80 2>/dev/null | grep '^{' >> gpurun_out/r2i_sweep.txt
done
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,P2P timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29599 scripts/nccl_probe.py 80 > gpurun_out/r2i_debug.log 2>&1
cat gpurun_out/r2i_sweep.txt
