# ncu --set full of one quicksort kernel: bash tools/ncu_one.sh OUT regex [extra env]
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-0} -c 1 -o $OUT/$2 -f python tools/profile_quicksort.py --reps 1 --kind ${4:-uniform} > $OUT/$2.log 2>&1
echo "exit $?"
