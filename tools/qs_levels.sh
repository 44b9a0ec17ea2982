OUT=gpurun_out/${1:-qsl}
mkdir -p $OUT
for w in 2; do
PP_QS_PROF=1 timeout 300 python - > $OUT/levels_w$w.log 2>&1 <<PY
import sys; sys.path.insert(0,'.')
import torch, paper_2004_12532_b200 as pp, synth
pp.load(build_if_missing=False); pp.pp_set_param("qs_waves", $w)
n=1<<28
q0=synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda"); q=torch.empty_like(q0)
for r in range(2):
    q.copy_(q0); torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record(); pp.pp_quicksort_u64(q); e.record(); torch.cuda.synchronize(); print("ms", s.elapsed_time(e), flush=True)
PY
done
