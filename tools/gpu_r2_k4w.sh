# K4w A/B: gaussian parity per RANMAR_K4 variant, then config-5 timing.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for v in ${K4_VARIANTS:-1 3 2 0}; do
  RANMAR_K4=$v timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranmars.py tests/test_gpu_langevin.py -m gpu -q -x -k "gaussian" > gpurun_out/k4w_test_$v.log 2>&1; echo "v=$v tests=$? $(tail -1 gpurun_out/k4w_test_$v.log)"
  RANMAR_K4=$v timeout 300 python tools/time_k4.py 2>&1 | tail -1
done
