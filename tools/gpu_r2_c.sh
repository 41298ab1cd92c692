# Round 2 (c): whole GPU suite (incl. the reference demos / acceptance suite on
# the drop-in), the crlog sweep with the exception table, both bench arms.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_facade.py -m gpu -q -s -k "acceptance or demo" > gpurun_out/dropin.log 2>&1; echo dropin=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 600 gpurun_out/bench.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
timeout 1200 python tools/crlog_sweep.py > gpurun_out/crlog_sweep.log 2>&1; echo sweep=$?
