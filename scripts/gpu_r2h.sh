timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 scripts/nccl_probe.py 10 40 80 160 > gpurun_out/r2h_nccl_probe.jsonl 2> gpurun_out/r2h.err
NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 scripts/nccl_probe.py 80 >> gpurun_out/r2h_nccl_probe.jsonl 2>> gpurun_out/r2h.err
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 scripts/nccl_probe.py 80 > /dev/null 2> gpurun_out/r2h_nccl_debug.log
cat gpurun_out/r2h_nccl_probe.jsonl
