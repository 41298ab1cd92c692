mkdir -p gpurun_out
for n in 1 127 128 129 1000 100000; do timeout 120 python tools/time_c3.py --n $n --reps 2 --compare 2>&1 | tail -1; done
timeout 300 python tools/time_c3.py --compare > gpurun_out/tc_full3.log 2>&1; echo full=$?; tail -3 gpurun_out/tc_full3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_graph.py tests/test_gpu_text.py -m gpu -q -x > gpurun_out/tc_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/tc_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bulk_tc -s 3 -c 1 -o gpurun_out/bulk_tc2 python tools/time_c3.py --reps 1 > gpurun_out/tcncu.log 2>&1; echo ncu=$?
