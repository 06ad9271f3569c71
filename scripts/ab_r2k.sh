# r2k: K7 software-pipelined tap loads (pair i+1's words in flight under
# pair i) and K6 with per-row staging for unaligned rows (the 16-B-aligned
# instantiation must not lose); variants/k7_nopipe.so = the previous build.
python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5 or crop or unaligned or storage" > gpurun_out/r2k_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2k_pytest.log
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), round(r['kernel_only']['avg_launch_ms']*1e3,1) if r['kernel_only'] else None, d['clocks']['sm_mhz'])
" >> gpurun_out/r2k_ab.txt; }
export LL_BENCH_NO_HEADLINE_PLAN=1
for i in 1 2; do
  python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg5-pipe-38reg
  LL_LIB=variants/k7_nopipe.so python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg5-prev
  LL_LIB=variants/k7_pipe_r32.so python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg5-pipe-32reg
  python bench.py --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg2-fp32-new
  LL_LIB=variants/k7_nopipe.so python bench.py --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg2-fp32-prev
  python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg2-bf16-new
  LL_LIB=variants/k7_nopipe.so python bench.py --dtype bf16 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2k_bench.err; line cfg2-bf16-prev
done
cat gpurun_out/r2k_ab.txt; grep -h "passed\|rc=" gpurun_out/r2k_pytest.log
