# Round 2 (b): the whole GPU suite after the _dev-contract refactor, smoke, and
# the crlog sweep recording the accurate phase's undecided inputs (mode 2).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python tools/crlog_sweep.py > gpurun_out/crlog_sweep.log 2>&1; echo sweep=$?; tail -c 1500 gpurun_out/crlog_sweep.log
