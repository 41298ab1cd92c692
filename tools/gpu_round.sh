# Full round-end style run: tests, smoke, both bench arms, launch lists and one
# ncu --set full capture per hot kernel. Outputs under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|Socket|Core|Thread" >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
for c in c2 c3 c4 c5 lang; do
  timeout 300 python tools/profile_case.py $c > gpurun_out/plain_$c.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/profile_case.py $c > gpurun_out/ncu_l_$c.log 2>&1; echo launches_$c=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_store -s 2 -c 1 -o gpurun_out/full_gen_store python tools/profile_case.py c2 > gpurun_out/ncu_f_c2.log 2>&1; echo full_c2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk -s 2 -c 1 -o gpurun_out/full_bulk python tools/profile_case.py c3 > gpurun_out/ncu_f_c3.log 2>&1; echo full_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:consume -s 2 -c 1 -o gpurun_out/full_consume python tools/profile_case.py c4 > gpurun_out/ncu_f_c4.log 2>&1; echo full_c4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/full_gaussian python tools/profile_case.py c5 > gpurun_out/ncu_f_c5.log 2>&1; echo full_c5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:langevin -s 2 -c 1 -o gpurun_out/full_langevin python tools/profile_case.py lang > gpurun_out/ncu_f_lang.log 2>&1; echo full_lang=$?
