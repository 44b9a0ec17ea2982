#!/usr/bin/env python
"""Config 1 (2^20 u64, L2-resident) back-to-back partition calls: GPU time and
host time per call, per cleanup-tail setting, in repeated rounds (shows the
warm-up of the first calls).  Every call gets a fresh copy of the input.

    python tools/c1_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402

pp.load(build_if_missing=False)
n1 = 1 << 20
src = synth.uniform_u64_torch(n1, synth.SEEDS["c1"], "cuda")
bufs = [src.clone() for _ in range(200)]
d1 = torch.zeros(1, dtype=torch.int64, device="cuda")
for rnd in range(3):
    for spec in ["", "cleanup_chain=0", "cleanup_chain=1"]:
        pp.reset_params()
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            pp.pp_set_param(k, int(v))
        for b in bufs:
            b.copy_(src)
        torch.cuda.synchronize()
        for b in bufs[:10]:
            pp.pp_partition_async_u64(b, 1 << 63, d1)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        s.record()
        for b in bufs[10:]:
            pp.pp_partition_async_u64(b, 1 << 63, d1)
        e.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(rnd, spec or "default", "gpu ms/call %.4f" % (s.elapsed_time(e) / 190),
              "host us/call %.1f" % ((t1 - t0) / 190 * 1e6), flush=True)
