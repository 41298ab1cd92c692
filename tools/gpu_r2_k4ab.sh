# K4 A/B: parity (gaussian tests) and config-5 timing per RANMAR_K4 variant.
mkdir -p gpurun_out
for v in ${K4_VARIANTS:-0 5}; do
  RANMAR_K4=$v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_ranmars.py tests/test_gpu_langevin.py -m gpu -q -x -k "gaussian or config5" > gpurun_out/k4ab_test_$v.log 2>&1; echo "v=$v tests=$? $(tail -1 gpurun_out/k4ab_test_$v.log)"
  RANMAR_K4=$v timeout 300 python tools/time_k4.py 2>&1 | tail -1
done
if [ -n "$K4_NCU" ]; then
  RANMAR_K4=$K4_NCU timeout 900 ncu --set full --clock-control none --import-source on -k regex:gaussian -s 2 -c 1 -o gpurun_out/k4_v$K4_NCU python tools/profile_case.py c5 > gpurun_out/ncu_k4_v$K4_NCU.log 2>&1; echo ncu=$?
fi
