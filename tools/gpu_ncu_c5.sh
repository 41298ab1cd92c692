mkdir -p gpurun_out
export RANMAR_GAUSS_Q=1
timeout 300 python tools/profile_case.py c5 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/full_gaussian_q python tools/profile_case.py c5 > gpurun_out/ncu_f_c5.log 2>&1; echo full_c5=$?
