# r2f (2 GPUs): multi-GPU parity incl. storage tier / cfg5 / small sources over
# NCCL, then cfg2 / cfg4 / cfg5 over NCCL at N = 2 with the exchange's NVLink GB/s.
python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2f_multi.log 2>&1; echo rc=$? >> gpurun_out/r2f_multi.log
for w in cfg2 cfg4 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $w --exchange nccl --steps 624 --warmup 20 >> gpurun_out/r2f_bench.jsonl 2>> gpurun_out/r2f_bench.err
done
tail -3 gpurun_out/r2f_multi.log
