# NCCL send/recv knobs II: copy-engine P2P (NCCL_P2P_USE_CUDA_MEMCPY) with and
# without cuMem, 80 MB per peer, probe alone (each run bounded by timeout 90)
p=29600
for v in "X=0" "NCCL_CUMEM_ENABLE=0" "NCCL_P2P_USE_CUDA_MEMCPY=1 NCCL_CUMEM_ENABLE=0" \
         "NCCL_P2P_USE_CUDA_MEMCPY=1" "NCCL_P2P_DIRECT_DISABLE=1" "NCCL_BUFFSIZE=67108864 NCCL_P2P_NVL_CHUNKSIZE=4194304"; do
  p=$((p+1))
  echo "== $v" >> gpurun_out/r2ag_sweep.txt
  env $v timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p scripts/nccl_probe.py 80 2>/dev/null | grep '^{' >> gpurun_out/r2ag_sweep.txt
  echo "rc=$?" >> gpurun_out/r2ag_sweep.txt
done
cat gpurun_out/r2ag_sweep.txt
