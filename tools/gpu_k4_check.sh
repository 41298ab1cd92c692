# K4 parity (gaussian tests) and config-5 timing at the current build.
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranmars.py tests/test_gpu_langevin.py tests/test_gpu_fullsize.py -m gpu -q -x -k "gaussian or config5" 2>&1 | tail -1
timeout 300 python tools/time_k4.py 2>&1 | tail -1
