# Round 2 (e): whole GPU suite, smoke, both bench arms at HEAD.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
