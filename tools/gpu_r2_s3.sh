# Session-3 check: whole GPU suite, smoke, our bench arm.
mkdir -p gpurun_out/s3
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/s3/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/s3/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/s3/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/s3/bench.log 2>&1; echo bench=$?
