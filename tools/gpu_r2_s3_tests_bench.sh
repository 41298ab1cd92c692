# GPU suite, smoke and both bench arms at HEAD (outputs under gpurun_out/final3/).
mkdir -p gpurun_out/final3
O=gpurun_out/final3
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > $O/bench.log 2>&1; echo bench=$?
timeout 1200 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo bench_ref=$?
