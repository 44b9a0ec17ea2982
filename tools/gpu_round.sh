#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, launch list, one full ncu capture.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [tag] [what]'
# what: any of tests,smoke,bench,launches,ncu (comma separated; default all)
set -u
TAG=${1:-r01}
WHAT=${2:-tests,smoke,bench,launches,ncu}
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
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline --no-e2e \
    > "$OUT/ncu_launches.log" 2>&1
  echo "launches exit $?" >> "$OUT/status.txt"
fi
if has ncu; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ss_group -s 1 -c 1 \
    -o "$OUT/group_full" -f python tools/profile_partition.py > "$OUT/ncu_full.log" 2>&1
  echo "ncu_full exit $?" >> "$OUT/status.txt"
fi
cat "$OUT/status.txt"
