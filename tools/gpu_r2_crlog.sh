# Round 2: correctly rounded log for gaussian(): GPU parity, the exhaustive
# domain sweep and the K4 config-5 time after the change.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_langevin.py tests/test_gpu_ranmars.py -m gpu -q -x -k "gauss or crlog or fp64 or langevin or ranmars or RanMars" > gpurun_out/pytest_crlog.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_crlog.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -s -k "config5" > gpurun_out/pytest_c5full.log 2>&1; echo fullsize=$?; tail -3 gpurun_out/pytest_c5full.log
timeout 300 python tools/time_k4.py > gpurun_out/time_k4.log 2>&1; echo k4=$?; cat gpurun_out/time_k4.log
timeout 1200 python tools/crlog_sweep.py > gpurun_out/crlog_sweep.log 2>&1; echo sweep=$?; tail -2 gpurun_out/crlog_sweep.log
