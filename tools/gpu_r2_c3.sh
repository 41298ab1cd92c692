# Config 3 after a K3 change: parity (make_streams / jump / tensor-core tests),
# timing vs the IMAD bulk, and the launch list of one config-3 call.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -m gpu -q -x -k "make_streams or config3 or tensor or jump or golden or smoke" > gpurun_out/c3_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/c3_tests.log
timeout 300 python tools/time_c3.py --compare 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_case.py c3 > /dev/null 2>&1; echo ncu=$?
if [ -n "$C3_FULL" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_tc -s 2 -c 1 -o gpurun_out/bulk_tc python tools/profile_case.py c3 > /dev/null 2>&1; echo full=$?; fi
