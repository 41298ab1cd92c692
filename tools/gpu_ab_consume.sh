# A/B of consume_kernel variants: each variant file is copied in, rebuilt, timed.
# (the original source is restored and rebuilt at the end)
ORIG=$(mktemp); cp paper_2512_00093_b200/csrc/consume_kernel.cu $ORIG
for v in "$@"; do
  cp $v paper_2512_00093_b200/csrc/consume_kernel.cu && make lib > /dev/null 2>&1 && echo "variant $v" && python tools/time_c4.py --reps 3 | tail -1
done
cp $ORIG paper_2512_00093_b200/csrc/consume_kernel.cu && rm -f $ORIG && make lib > /dev/null 2>&1
