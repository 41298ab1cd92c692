set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
grep -E "max ulp" gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log
timeout 300 python tools/profile_case.py c2 > gpurun_out/plain_c2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_case.py c2 > gpurun_out/ncu_l2.log 2>&1; echo ncu_l_c2=$?
timeout 300 python tools/profile_case.py c3 > gpurun_out/plain_c3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_case.py c3 > gpurun_out/ncu_l3.log 2>&1; echo ncu_l_c3=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_store -s 2 -c 1 -o gpurun_out/prof_gen_c2 python tools/profile_case.py c2 > gpurun_out/ncu_full_gen.log 2>&1; echo ncu_gen=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk -s 2 -c 1 -o gpurun_out/prof_bulk_c3 python tools/profile_case.py c3 > gpurun_out/ncu_full_bulk.log 2>&1; echo ncu_bulk=$?
ls -la gpurun_out
