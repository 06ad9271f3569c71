# r2ar: K6 far samples interleaved over the grid (variants/k6_far_interleave.so) vs first,
# with the span-request build; cfg4 bf16 / fp32 over P2P at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,3), round(l['ms_per_step'],4), round(l['roofline']['frac'],3), x.get('nvlink_gbs'), l['clocks']['sm_mhz'])
" >> gpurun_out/r2ar_ab.txt 2>&1; }
for i in 1 2; do
  for v in default k6_far_interleave; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    for w in "cfg4 --dtype bf16" "cfg4" "cfg5"; do
      LL_LIB=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 bench.py --gpus 2 --workload $w --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2ar.err
      line "n2-${w// /}-$v"
    done
  done
done
cat gpurun_out/r2ar_ab.txt
