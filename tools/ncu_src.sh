# full ncu captures (source-level) of quicksort kernels:
#   bash tools/ncu_src.sh OUT "k=v,..." regex:skip:count [regex:skip:count ...]
OUT=gpurun_out/$1; mkdir -p $OUT; P=$2; shift 2
i=0
for spec in "$@"; do
  IFS=: read -r rx sk ct <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $sk -c $ct -o $OUT/full_$i -f \
    python tools/profile_quicksort.py --reps 1 --kind uniform --params "$P" > $OUT/full_$i.log 2>&1
  echo "full_$i ($spec) exit $?" >> $OUT/status.txt
  i=$((i+1))
done
