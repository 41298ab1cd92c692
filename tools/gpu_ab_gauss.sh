# A/B of gauss_kernel.cu variants (K4x2 via RB_K4X2=1): each variant file is copied in,
# rebuilt, checked (gaussian parity) and timed against K4.
# (the original source is restored and rebuilt at the end)
ORIG=$(mktemp); cp paper_2512_00093_b200/csrc/gauss_kernel.cu $ORIG
for v in "$@"; do
  cp $v paper_2512_00093_b200/csrc/gauss_kernel.cu && make lib > /dev/null 2>&1 && echo "variant $v" && \
  RB_K4X2=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranmars.py tests/test_gpu_langevin.py -m gpu -q -x -k "gaussian" 2>&1 | tail -1 && \
  RB_K4X2=1 python tools/time_k4.py | tail -1
done
python tools/time_k4.py | tail -1
cp $ORIG paper_2512_00093_b200/csrc/gauss_kernel.cu && rm -f $ORIG && make lib > /dev/null 2>&1
