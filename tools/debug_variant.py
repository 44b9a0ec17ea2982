import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_12532_b200 as pp, synth, oracle
v = int(sys.argv[1]); n = int(sys.argv[2])
pp.load(build_if_missing=False)
pp.pp_set_param("variant", v)
a = synth.uniform_u64_np(n, 5)
t = torch.from_numpy(a.view(np.int64).copy()).cuda()
s = pp.pp_partition_u64(t, 1 << 63)
print(pp.pp_last_stats())
oracle.check_partition(a, t.cpu().numpy().view(np.uint64), 1 << 63, s)
print("ok", v, n)
