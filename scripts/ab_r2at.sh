# r2at: K6 far-band bulk requests of G rows: storage tier G = 2 / 4 (vs row requests) on cfg3
# at N=1; peers G = 8 / 4 (vs the whole 32-row band) on cfg4 at N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
LL_LIB=variants/k6_g32_h2.so timeout 600 python -m pytest tests -m gpu -x -q -k "storage" > gpurun_out/r2at_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2at_pytest.log
LL_LIB=variants/k6_g4_h0.so timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "p2p" >> gpurun_out/r2at_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2at_pytest.log
grep -E "passed|rc=" gpurun_out/r2at_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); r=l.get('storage_roofline') or {}; x=l.get('exchange') or {}
print('$1', round(l['value']/1e6,4), round(l['ms_per_step'],4), 'pcie', r.get('frac'), 'nvl', x.get('nvlink_gbs'), l['clocks']['sm_mhz'])
" >> gpurun_out/r2at_ab.txt 2>&1; }
for i in 1 2; do
  for v in default k6_g32_h2 k6_g32_h4; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    LL_LIB=$L timeout 600 python bench.py --workload cfg3 --steps 156 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2at.err; line cfg3-$v
  done
  for v in default k6_g8_h0 k6_g4_h0; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    for w in "cfg4 --dtype bf16" "cfg4"; do
      LL_LIB=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29531 bench.py --gpus 2 --workload $w --steps 312 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2at.err
      line "n2-${w// /}-$v"
    done
  done
done
cat gpurun_out/r2at_ab.txt
