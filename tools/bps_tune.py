import sys; sys.path.insert(0,'.')
import torch, paper_2004_12532_b200 as pp, synth
pp.load(build_if_missing=False)
n=1<<27; src=synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda"); w=torch.empty_like(src); d=torch.zeros(1,dtype=torch.int64,device="cuda")
for nt in (256,128,256,128):
    pp.pp_set_param("bps_nt", nt); ts=[]
    for i in range(4):
        w.copy_(src); torch.cuda.synchronize()
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); pp.pp_partition_bps_async_u64(w, 1<<63, d); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    print(nt, min(ts[1:]), flush=True)
