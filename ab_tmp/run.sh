ORIG=$(mktemp); cp paper_2512_00093_b200/csrc/jump_kernels.cu $ORIG
for v in ab_tmp/keep.cu ab_tmp/conc.cu ab_tmp/keep.cu ab_tmp/conc.cu; do
  cp $v paper_2512_00093_b200/csrc/jump_kernels.cu && make lib > /dev/null 2>&1 && echo "variant $v" && \
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -m gpu -q -x -k "jump" 2>&1 | tail -1 && \
  python tools/time_jump.py --compare | tail -3 | head -1; python tools/time_jump.py | tail -1
done
cp $ORIG paper_2512_00093_b200/csrc/jump_kernels.cu; make lib > /dev/null 2>&1
