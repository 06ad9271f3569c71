# r2q: K6 occupancy (min blocks per SM 1 = 4 resident at 66 regs, 5, 6) for bf16 and fp32
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,2), round(r['frac'],4), d['clocks']['sm_mhz'])
" >> gpurun_out/r2q_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
LL_LIB=variants/k6_mb6.so python -m pytest tests -m gpu -x -q -k "crop or unaligned" > gpurun_out/r2q_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2q_pytest.log
for i in 1 2; do
  for v in default k6_mb5 k6_mb6; do
    L=""; [ $v != default ] && L=variants/$v.so
    LL_LIB=${L:-paper_1910_01196_b200/liblocload_b200.so} python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2q.err; line bf16-$v
    LL_LIB=${L:-paper_1910_01196_b200/liblocload_b200.so} python bench.py --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2q.err; line fp32-$v
  done
done
cat gpurun_out/r2q_ab.txt; tail -2 gpurun_out/r2q_pytest.log
