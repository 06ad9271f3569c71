# r2t: host-path prefetch depth for e2e (4 = default vs 6 / 8), cfg2 fp32 and bf16
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json'))
print('$1', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), d['clocks']['sm_mhz'])
" >> gpurun_out/r2t_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
for i in 1 2; do
  for dp in 4 6 8; do
    python bench.py --no-cpu-baseline --steps 624 --prefetch-depth $dp > /tmp/o.json 2>>gpurun_out/r2t.err; line fp32-depth$dp
  done
  python bench.py --no-cpu-baseline --steps 624 --dtype bf16 --prefetch-depth 8 > /tmp/o.json 2>>gpurun_out/r2t.err; line bf16-depth8
  python bench.py --no-cpu-baseline --steps 624 --dtype bf16 > /tmp/o.json 2>>gpurun_out/r2t.err; line bf16-depth4
done
cat gpurun_out/r2t_ab.txt
