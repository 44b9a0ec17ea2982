# full ncu captures of the quicksort kernels (one launch each)
OUT=gpurun_out/${1:-ncuqs}
mkdir -p $OUT
for k in qs_leaf_merge qs_small_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 0 -c 1 -o $OUT/$k -f python tools/profile_quicksort.py --reps 1 --kind uniform > $OUT/$k.log 2>&1
echo "$k exit $?" >> $OUT/status.txt
done
cat $OUT/status.txt
