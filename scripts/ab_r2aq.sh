# r2aq: K7 two adjacent columns per thread (variants/k7_two_cols.so, one 32-bit bf16x2 store
# per row and channel) vs the one-column kernel; cfg5 at N=1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
LL_LIB=variants/k7_two_cols.so timeout 900 python -m pytest tests -m gpu -x -q -k "resize or variable or cfg5" > gpurun_out/r2aq_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2aq_pytest.log; tail -2 gpurun_out/r2aq_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); r=l['roofline']
print('$1', round(l['value']/1e6,3), round(r['avg_launch_ms']*1e3,2), round(r['frac'],4), l['clocks']['sm_mhz'], l['clocks']['reasons'])
" >> gpurun_out/r2aq_ab.txt 2>&1; }
for i in 1 2; do
  for v in default k7_two_cols; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    LL_LIB=$L timeout 600 python bench.py --workload cfg5 --no-cpu-baseline --no-e2e --steps 624 > /tmp/o.json 2>>gpurun_out/r2aq.err; line cfg5-$v
  done
done
cat gpurun_out/r2aq_ab.txt
LL_LIB=variants/k7_two_cols.so timeout 600 ncu --set full --clock-control none -k regex:augment_resize -s 3 -c 1 -o gpurun_out/prof_r2aq python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu rc=$?
