# r2ad: K7 L2 prefetch of the band's distinct row range (each row once) vs lo/hi rows per output row
LL_LIB=variants/k7_pfrange.so python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5" > gpurun_out/r2ad_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2ad_pytest.log
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), d['clocks']['reasons'])
" >> gpurun_out/r2ad_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
for i in 1 2 3; do
  python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ad.err; line default
  LL_LIB=variants/k7_pfrange.so python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2ad.err; line pfrange
done
LL_LIB=variants/k7_pfrange.so ncu --set full --clock-control none -k regex:augment_resize -c 1 -s 30 -o gpurun_out/r2ad_k7_pfrange python bench.py --workload cfg5 --steps 10 --warmup 30 --no-cpu-baseline --no-e2e > /dev/null 2>&1
cat gpurun_out/r2ad_ab.txt; tail -2 gpurun_out/r2ad_pytest.log
