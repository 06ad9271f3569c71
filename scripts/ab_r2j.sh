# r2j: K7 row reuse (distinct source rows tapped once per row pair), 35 vs 32 registers
python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5" > gpurun_out/r2j_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2j_pytest.log
line() { python -c "
import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']
print('$1', round(d['value']/1e6,3), round(r['avg_launch_ms']*1e3,1), round(r['frac'],3), round(r['kernel_only']['avg_launch_ms']*1e3,1) if r['kernel_only'] else None, d['clocks']['sm_mhz'])
" >> gpurun_out/r2j_ab.txt; }
for i in 1 2; do
  LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2j_bench.err; line reuse-35reg
  LL_LIB=paper_1910_01196_b200/variants_k7r32.so LL_BENCH_NO_HEADLINE_PLAN=1 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2j_bench.err; line reuse-32reg
done
F=$(ls paper_1910_01196_b200/liblocload_b200.so)
ncu --set full --clock-control none --import-source on -k regex:augment_resize -c 1 -s 30 -o gpurun_out/r2j_k7 python bench.py --workload cfg5 --steps 10 --warmup 30 --no-cpu-baseline --no-e2e > gpurun_out/r2j_ncu.log 2>&1
cat gpurun_out/r2j_ab.txt; tail -2 gpurun_out/r2j_pytest.log
