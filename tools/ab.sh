# A/B the c2 partition bench across library builds: bash tools/ab.sh lib1.so lib2.so ...
for r in 1 2; do for L in "$@"; do
  PP_LIB_PATH=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/ab_$(basename $L)_$r.json 2>&1
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$(basename $L)_$r.json')); print('$L', $r, round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4), d['clocks']['sm_mhz'])"
done; done
