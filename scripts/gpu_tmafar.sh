#!/bin/bash
# K6 peer-shard (NVLink) samples via TMA bulk copies: 2-GPU parity, cfg2/cfg4 at N=2 and N=4 (4-GPU box)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for V in default tmafar; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  timeout 900 python -m pytest tests -q -m gpu -k "multi or exchange or regular or p2p or peer" --timeout 600 > gpurun_out/pytest_var_$V.log 2>&1
  echo "$V pytest rc=$? $(tail -1 gpurun_out/pytest_var_$V.log)"
done
show() { python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(l['value']), round(l['ms_per_step'],4), {k: v and round(v*1000,1) for k, v in l['kernel_ms'].items() if v})"; }
for N in 2 4; do
for V in default tmafar; do
  if [ "$V" = default ]; then unset LL_LIB; else export LL_LIB=$PWD/variants/lib_$V.so; fi
  for W in cfg2 cfg4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
       --master-port 2960$N bench.py --gpus $N --workload $W --steps 312 --no-e2e 2>&1 | show "$V $W n$N"
  done
done
done
unset LL_LIB
bash scripts/gpu_nccl_var.sh
