# A/B of jump_kernels.cu variants: each variant file is copied in, rebuilt, checked and timed.
# (the original source is restored and rebuilt at the end)
ORIG=$(mktemp); cp paper_2512_00093_b200/csrc/jump_kernels.cu $ORIG
for v in "$@"; do
  cp $v paper_2512_00093_b200/csrc/jump_kernels.cu && make lib > /dev/null 2>&1 && echo "variant $v" && \
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "make_streams or three_level or config3 or jump" 2>&1 | tail -1 && \
  python tools/time_c3.py --reps 50 | tail -1; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:level_kernel --csv python tools/time_c3.py --reps 2 2>/dev/null | grep level_kernel | tail -2 | cut -c1-200
done
cp $ORIG paper_2512_00093_b200/csrc/jump_kernels.cu && rm -f $ORIG && make lib > /dev/null 2>&1
