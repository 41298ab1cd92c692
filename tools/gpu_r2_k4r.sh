# K4r vs K4: gaussian parity (K4r, the default) and config-5 timing of both.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranmars.py tests/test_gpu_langevin.py tests/test_gpu_fullsize.py -m gpu -q -x -k "gaussian or config5" > gpurun_out/k4r_test.log 2>&1; echo "tests=$? $(tail -1 gpurun_out/k4r_test.log)"
timeout 300 python tools/time_k4.py 2>&1 | tail -1
RANMAR_K4OLD=1 timeout 300 python tools/time_k4.py 2>&1 | tail -1
