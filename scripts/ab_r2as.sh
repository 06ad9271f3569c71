# r2as: K6 storage-tier (pinned host, PCIe) bands as one span request (variants/k6_host_span.so)
# vs 32 row requests; cfg3 at N=1 (alpha = 0.25: 75 % of samples from the storage tier)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export LL_BENCH_NO_HEADLINE_PLAN=1
LL_LIB=variants/k6_host_span.so timeout 600 python -m pytest tests -m gpu -x -q -k "storage" > gpurun_out/r2as_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2as_pytest.log; tail -2 gpurun_out/r2as_pytest.log
line() { python -c "
import json,sys
l=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); r=l.get('storage_roofline') or {}
print('$1', round(l['value']/1e6,4), round(l['ms_per_step'],4), r.get('frac'), r.get('achieved'), l['clocks']['sm_mhz'])
" >> gpurun_out/r2as_ab.txt 2>&1; }
for i in 1 2; do
  for v in default k6_host_span; do
    L=paper_1910_01196_b200/liblocload_b200.so; [ $v != default ] && L=variants/$v.so
    LL_LIB=$L timeout 600 python bench.py --workload cfg3 --steps 156 --no-cpu-baseline --no-e2e > /tmp/o.json 2>>gpurun_out/r2as.err; line cfg3-$v
  done
done
cat gpurun_out/r2as_ab.txt
