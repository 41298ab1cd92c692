mkdir -p gpurun_out
timeout 300 python tools/profile_case.py c3 > gpurun_out/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk -s 2 -c 1 -o gpurun_out/full_bulk2 python tools/profile_case.py c3 > gpurun_out/ncu_f_c3.log 2>&1; echo full_c3=$?
