mkdir -p gpurun_out
for v in 0 1; do
RANMAR_K4=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/k4_v$v python tools/profile_case.py c5 > gpurun_out/ncu_k4_v$v.log 2>&1; echo ncu$v=$?
done
