mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "consume or config4 or gaussian" > gpurun_out/pytest_consume.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_consume.log
timeout 300 python tools/profile_case.py c4 > gpurun_out/plain_c4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:consume -s 2 -c 1 -o gpurun_out/prof_consume_c4 python tools/profile_case.py c4 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4=$?
timeout 300 python tools/profile_case.py c5 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/prof_gauss_c5 python tools/profile_case.py c5 > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5=$?
