#!/usr/bin/env python
"""Sanity check beyond the test sizes: quicksort of 2^k u64 keys (default
2^30 = 8 GiB) uniform and [0,1000); compares with torch.sort (library) on the
order-preserving int64 image; prints time and verdict."""
import sys
import os
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402
from gpu_util import order_key  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << k
pp.load(build_if_missing=False)
for kind in ("uniform", "dup1000"):
    t = (synth.uniform_u64_torch(n, 77, "cuda") if kind == "uniform"
         else synth.mod_range_u64_torch(n, 77, 1000, "cuda"))
    ref = torch.sort(order_key(t)).values
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pp.pp_quicksort(t)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t0)
    ok = torch.equal(order_key(t), ref)
    print(f"quicksort 2^{k} {kind}: {ms:.1f} ms, equals library sort: {ok}", flush=True)
    del t, ref
    torch.cuda.empty_cache()
