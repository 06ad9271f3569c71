# The driver's round-end bench commands on the final build (N = 1 and N = 2, both arms)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_n1.out 2> gpurun_out/drv_n1.err; echo "n1 rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref1.out 2> gpurun_out/drv_ref1.err; echo "ref1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/drv_n2.out 2> gpurun_out/drv_n2.err; echo "n2 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 \
  bench.py --impl reference --gpus 2 --steps 20 --warmup 5 > gpurun_out/drv_ref2.out 2> gpurun_out/drv_ref2.err; echo "ref2 rc=$?"
for f in n1 ref1 n2 ref2; do echo "== $f"; tail -1 gpurun_out/drv_$f.out | cut -c1-300; done
