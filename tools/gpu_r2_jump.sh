mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "jump or make_streams or config3" > gpurun_out/jump_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/jump_tests.log
timeout 300 python tools/time_jump.py --compare 2>&1 | tail -3
if [ -n "$J_FULL" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_tc -s 2 -c 1 -o gpurun_out/apply_tc python tools/profile_case.py jump > /dev/null 2>&1; echo full=$?; fi
