mkdir -p gpurun_out
timeout 300 python tools/profile_case.py c5 > gpurun_out/plain_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/prof_gauss_c5_v3 python tools/profile_case.py c5 > gpurun_out/ncu_c5.log 2>&1; echo ncu_c5=$?
