# r2ap: K6 staging loads with an L2 evict-first cache policy (variants/k6_evict_first.so) vs none; 1 GPU
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
LL_LIB=variants/k6_evict_first.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "crop or unaligned or augment" > gpurun_out/r2ap_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ap_pytest.log; tail -2 gpurun_out/r2ap_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); r=l['roofline']
print('$1', round(l['value']/1e6,3), round(r['avg_launch_ms']*1e3,2), round(r['frac'],4), l['clocks']['sm_mhz'])
" >> gpurun_out/r2ap_ab.txt 2>&1; }
for i in 1 2; do
  for v in default k6_evict_first; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    LL_LIB=$L timeout 600 python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ap.err; line bf16-$v
    LL_LIB=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ap.err; line fp32-$v
  done
done
cat gpurun_out/r2ap_ab.txt
