# r2ae: K6 local-sample staging with 256-bit loads (LDG.256, sm_100) vs 128-bit
LL_LIB=variants/k6_v8.so python -m pytest tests -m gpu -x -q -k "crop or unaligned or loader or storage" > gpurun_out/r2ae_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ae_pytest.log
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,2), round(r['frac'],4))
" >> gpurun_out/r2ae_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
for i in 1 2; do
  for v in default v8; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v = v8 ] && L=variants/k6_v8.so
    LL_LIB=$L python bench.py --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ae.err; line fp32-$v
    LL_LIB=$L python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ae.err; line bf16-$v
  done
done
cat gpurun_out/r2ae_ab.txt; tail -2 gpurun_out/r2ae_pytest.log
