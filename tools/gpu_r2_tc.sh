# tensor-core bulk kernel: equality with the IMAD kernel, parity tests, timing
mkdir -p gpurun_out
timeout 300 python tools/time_c3.py --n 1000 --compare > gpurun_out/tc_small.log 2>&1; echo small=$?; tail -2 gpurun_out/tc_small.log
timeout 300 python tools/time_c3.py --compare > gpurun_out/tc_full.log 2>&1; echo full=$?; tail -3 gpurun_out/tc_full.log
RANMAR_BULK=imad timeout 300 python tools/time_c3.py > gpurun_out/tc_imad.log 2>&1; tail -1 gpurun_out/tc_imad.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py tests/test_gpu_graph.py -m gpu -q -x > gpurun_out/tc_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/tc_pytest.log
