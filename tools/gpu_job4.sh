mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gaussian" > gpurun_out/pytest_gauss.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gauss.log
timeout 600 python bench.py --no-e2e --no-cpu --steps 20 > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config5'])"
timeout 300 python tools/profile_case.py c5 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/prof_gauss_c5_v2 python tools/profile_case.py c5 > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5=$?
