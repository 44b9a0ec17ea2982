#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, launch list, one full ncu capture.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tag] [what]'
# what: any of tests,smoke,bench,launches,qs,ncu (comma separated; default all)
set -u
TAG=${1:-r01}
WHAT=${2:-tests,smoke,bench,launches,qs,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
nproc > "$OUT/host.txt"; lscpu | grep -i 'model name' >> "$OUT/host.txt"; free -g >> "$OUT/host.txt"
has() { [[ ",$WHAT," == *",$1,"* ]]; }
if has tests; then
  timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest_gpu exit $?" >> "$OUT/status.txt"
fi
if has smoke; then
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/status.txt"
fi
if has bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/status.txt"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
  echo "bench_ref exit $?" >> "$OUT/status.txt"
fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    -k regex:"ss_group|reduce_count|scan_swap|tile_scan|locate_kernel|swap_kernel|small_partition|count_kernel" \
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-e2e \
    > "$OUT/ncu_launches.log" 2>&1
  echo "launches exit $?" >> "$OUT/status.txt"
fi
if has qs; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file "$OUT/launches_qs_uniform.csv" python tools/profile_quicksort.py --reps 1 --kind uniform \
    > "$OUT/ncu_qs.log" 2>&1
  echo "launches_qs exit $?" >> "$OUT/status.txt"
  PP_QS_PROF=1 timeout 300 python tools/profile_quicksort.py --reps 2 --kind uniform > "$OUT/qs_levels_uniform.log" 2>&1
  PP_QS_PROF=1 timeout 300 python tools/profile_quicksort.py --reps 2 --kind dup1000 > "$OUT/qs_levels_dup1000.log" 2>&1
  echo "qs_levels exit $?" >> "$OUT/status.txt"
fi
if has ncu; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ss_group -s 1 -c 1 \
    -o "$OUT/group_full" -f python tools/profile_partition.py > "$OUT/ncu_full.log" 2>&1
  echo "ncu_full exit $?" >> "$OUT/status.txt"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ss_group -s 1 -c 1 \
    -o "$OUT/group_full_u32" -f python tools/profile_partition.py --dtype u32 > "$OUT/ncu_full_u32.log" 2>&1
  echo "ncu_full_u32 exit $?" >> "$OUT/status.txt"
  # the headline launch (2^33 u64): one-pass DRAM metrics, no replay of the 64 GiB kernel
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:ss_group -c 1 --csv --log-file "$OUT/c3_traffic.csv" python tools/size_sweep.py --exps 33 --reps 1 \
    > "$OUT/ncu_c3.log" 2>&1
  echo "ncu_c3_traffic exit $?" >> "$OUT/status.txt"
fi
cat "$OUT/status.txt"
