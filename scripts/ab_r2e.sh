# r2e: K7 micro-opts (prefetch shifts, magic accumulator, unroll 2) and the
# L2 fetch-granularity knob for K6 bf16.  Measurement aid.
python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5 or augment or crop" > gpurun_out/r2e_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2e_pytest.log
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), round(r['kernel_only']['avg_launch_ms']*1e3,1) if r['kernel_only'] else None, d['clocks']['sm_mhz'])
" >> gpurun_out/r2e_ab.txt; }
for i in 1 2; do
  LL_K7=rows LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2e_bench.err; line cfg5-rows
  LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2e_bench.err; line cfg2bf16-default
  for g in 32 64 128; do
    LL_L2_FETCH=$g LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2e_bench.err; line cfg2bf16-l2fetch$g
  done
done
for g in 0 32; do
  LL_L2_FETCH=$g ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:augment_crop -c 3 --csv python bench.py --dtype bf16 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2e_ncu_l2fetch$g.csv 2>/dev/null
done
cat gpurun_out/r2e_ab.txt; tail -2 gpurun_out/r2e_pytest.log
