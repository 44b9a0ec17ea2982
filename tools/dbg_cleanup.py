import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, paper_2004_12532_b200 as pp, oracle
from gpu_util import to_dev, to_host
pp.load(build_if_missing=False)
rng = np.random.default_rng(5)
for n in (70001, 300007, 1<<20):
  a = rng.integers(0, 4, size=n).astype(np.uint64)
  for p in (1,2,3):
    for path in (2,3):
      for chain in (0,1):
        pp.reset_params(); pp.pp_set_param("path",path); pp.pp_set_param("small_n",0); pp.pp_set_param("min_lines_per_group",2); pp.pp_set_param("cleanup_chain",chain)
        t=to_dev(a); s=pp.pp_partition(t,p); o=to_host(t,np.uint64); st=pp.pp_last_stats()
        K=oracle.count(a,p); ok = s==K and oracle.is_partitioned(o,p,s)
        bad = int(np.sum(o[:K]>=p)) + int(np.sum(o[K:]<p))
        print(n,p,path,chain,"ok" if ok else "BAD", bad, {k:st[k] for k in ("W","M","nTasks")}, flush=True)
