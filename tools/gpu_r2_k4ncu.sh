# K4 gaussian_kernel: one ncu --set full capture (2^20 atoms x 300 deviates) for the
# instruction mix / stall breakdown.
mkdir -p gpurun_out
timeout 300 python tools/profile_case.py c5 > gpurun_out/plain_c5.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gaussian_kernel -s 2 -c 1 -o gpurun_out/k4_full python tools/profile_case.py c5 > gpurun_out/ncu_k4.log 2>&1; echo ncu=$?
