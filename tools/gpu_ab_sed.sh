# A/B of one source file's variants made by sed expressions:
#   bash tools/gpu_ab_sed.sh FILE "CHECK-AND-TIME COMMAND" "label|sed-expr" ...
# each variant is built and the command run; the original is restored and rebuilt.
F=$1; CMD=$2; shift 2
ORIG=$(mktemp); cp $F $ORIG
for v in "$@"; do
  label=${v%%|*}; expr=${v#*|}
  cp $ORIG $F; [ -n "$expr" ] && sed -i "$expr" $F
  make lib > /dev/null 2>&1 || { echo "variant $label: build failed"; continue; }
  echo "variant $label:"; bash -c "$CMD"
done
cp $ORIG $F && rm -f $ORIG && make lib > /dev/null 2>&1
