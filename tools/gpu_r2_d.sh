# Round 2 (d): re-baseline at HEAD after the container rebuild.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rs -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 400 gpurun_out/bench.log
timeout 300 python tools/time_k4.py > gpurun_out/k4.log 2>&1; echo k4=$?; cat gpurun_out/k4.log
