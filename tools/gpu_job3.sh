mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu --steps 50 > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config3'], d['config4'], d['config5'])"
timeout 300 python tools/profile_case.py c3 > gpurun_out/plain_c3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_case.py c3 > gpurun_out/ncu_l3.log 2>&1; echo ncu_l_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk -s 2 -c 1 -o gpurun_out/prof_bulk_c3_v2 python tools/profile_case.py c3 > gpurun_out/ncu_full_bulk.log 2>&1; echo ncu_bulk=$?
