#!/usr/bin/env python
"""Step time of back-to-back c2 partitions with the library's inner timing
events on vs off (does an event between the group kernel and its PDL
dependent cost time?)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402

pp.load(build_if_missing=False)
n = 1 << 27
src = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
bufs = [src.clone() for _ in range(20)]
d = torch.zeros(1, dtype=torch.int64, device="cuda")
for rep in range(3):
    for timing in (False, True):
        for b in bufs:
            b.copy_(src)
        torch.cuda.synchronize()
        pp.pp_timing(timing)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for b in bufs:
            pp.pp_partition_async_u64(b, 1 << 63, d)
        e.record()
        torch.cuda.synchronize()
        if timing:
            pp.pp_timing_read()
        pp.pp_timing(False)
        print(f"rep {rep} inner_timing={timing}: {s.elapsed_time(e) / len(bufs):.4f} ms/step", flush=True)
