# quicksort: parity tests + phase profile (debug) + small-segment threshold sweep
OUT=gpurun_out/${1:-qs3}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_quicksort.py -q -x > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/status.txt
for cfg in 0 1; do
PP_QS_PROF=1 timeout 300 python - > $OUT/prof_cfg$cfg.log 2>&1 <<PY
import sys; sys.path.insert(0,'.')
import torch, paper_2004_12532_b200 as pp, synth
pp.load(build_if_missing=False); pp.pp_set_param("qs_small_cfg", $cfg)
n=1<<28
q0=synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda"); q=torch.empty_like(q0)
for r in range(2):
    q.copy_(q0); torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record(); pp.pp_quicksort_u64(q); e.record(); torch.cuda.synchronize(); print("ms", s.elapsed_time(e), flush=True)
PY
done
timeout 900 python tools/tune_qs.py --grid "leaf=2048,4096,8192;qs_small=32768,65536,131072" > $OUT/tune1.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches_uniform.csv python tools/profile_quicksort.py --reps 1 --kind uniform > $OUT/ncu_u.log 2>&1
cat $OUT/status.txt
