# A/B the c2 partition bench across param settings: bash tools/ab_params.sh "cleanup_chain=0" "cleanup_chain=1"
for r in 1 2; do for spec in "$@"; do
  PP_BENCH_PARAMS="$spec" timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-e2e > gpurun_out/abp.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/abp.json')); print('$spec', $r, round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4), d['clocks']['sm_mhz'], d['split_ok'] if 'split_ok' in d else '')"
done; done
