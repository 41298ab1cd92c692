# A/B of consume_kernel variants: each /tmp-free variant file is copied in, rebuilt, timed.
for v in "$@"; do
  cp $v paper_2512_00093_b200/csrc/consume_kernel.cu && make lib > /dev/null 2>&1 && echo "variant $v" && python tools/time_c4.py --reps 3 | tail -1
done
