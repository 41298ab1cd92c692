mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "consume or config4 or host_buffer or bad_state" > gpurun_out/pytest_c4.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_c4.log
timeout 600 python bench.py --no-e2e --no-cpu --steps 20 > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config4'])"
timeout 300 python tools/profile_case.py c4 > gpurun_out/plain_c4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:consume -s 2 -c 1 -o gpurun_out/full_consume2 python tools/profile_case.py c4 > gpurun_out/ncu_f_c4.log 2>&1; echo full_c4=$?
