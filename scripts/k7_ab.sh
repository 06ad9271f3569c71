python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5 or storage" > gpurun_out/r2d_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2d_pytest.log
for v in rows staged8 staged16 rows staged8 staged16; do
  LL_K7=$v LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2d_bench.err
  python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$v', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), round(r['kernel_only']['avg_launch_ms']*1e3,1) if r['kernel_only'] else None, d['clocks']['sm_mhz'])
" >> gpurun_out/r2d_k7ab.txt
done
cat gpurun_out/r2d_k7ab.txt; tail -2 gpurun_out/r2d_pytest.log
