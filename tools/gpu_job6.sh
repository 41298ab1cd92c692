mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu --steps 100 > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['config3']['ms'], d['config4']['ms'], d['config5']['ms'])"
for c in c2 c3; do timeout 300 python tools/profile_case.py $c > gpurun_out/plain_$c.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/profile_case.py $c > gpurun_out/ncu_l_$c.log 2>&1; echo launches_$c=$?; done
