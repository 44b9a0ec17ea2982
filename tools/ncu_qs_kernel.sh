# launch list + one full capture of a quicksort kernel under given params:
#   bash tools/ncu_qs_kernel.sh OUT kernel_regex "k=v,..." [kind]
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv \
  python tools/profile_quicksort.py --reps 1 --kind ${4:-uniform} --params "$3" > $OUT/launches.log 2>&1
echo "launches exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 0 -c 1 -o $OUT/full -f \
  python tools/profile_quicksort.py --reps 1 --kind ${4:-uniform} --params "$3" > $OUT/full.log 2>&1
echo "full exit $?"
