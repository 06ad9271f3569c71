# r2o: K7 tap loads with L1 eviction hints (evict_last / evict_first) vs default
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), d['clocks']['sm_mhz'])
" >> gpurun_out/r2o_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
for i in 1 2; do
  python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2o.err; line default
  LL_LIB=variants/k7_evict_last.so python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2o.err; line evict_last
  LL_LIB=variants/k7_evict_first.so python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2o.err; line evict_first
done
cat gpurun_out/r2o_ab.txt
