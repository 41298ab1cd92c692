# A/B of text_kernels.cu variants made by sed expressions ("label|sed-expr" arguments):
# each is built, checked (text parity) and timed; the original is restored and rebuilt.
F=paper_2512_00093_b200/csrc/text_kernels.cu
ORIG=$(mktemp); cp $F $ORIG
for v in "$@"; do
  label=${v%%|*}; expr=${v#*|}
  cp $ORIG $F; [ -n "$expr" ] && sed -i "$expr" $F
  make lib > /dev/null 2>&1 || { echo "variant $label: build failed"; continue; }
  echo "variant $label: $(timeout 600 python -m pytest tests/test_gpu_text.py -q -x 2>&1 | tail -1)"
  for r in 1 2; do python tools/time_text.py | tail -1; done
done
cp $ORIG $F && rm -f $ORIG && make lib > /dev/null 2>&1
