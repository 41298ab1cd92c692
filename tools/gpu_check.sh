# tests + both bench arms (no profilers)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
tail -1 gpurun_out/bench.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'clocks', d['clocks'])
print('e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'])
for k in ('config3','config4','config5','langevin','persistence'): print(k, d.get(k))"
tail -1 gpurun_out/bench_ref.log | cut -c1-300
