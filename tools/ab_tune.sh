# A/B library builds on the tune tool: bash tools/ab_tune.sh "<tune args>" lib1.so lib2.so ...
ARGS=$1; shift
for r in 1 2; do for L in "$@"; do
  echo "== $L rep $r"; PP_LIB_PATH=$L timeout 300 python tools/tune.py $ARGS
done; done
