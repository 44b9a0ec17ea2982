#!/usr/bin/env python
"""BASELINE config 1 (2^20 u64, L2-resident, launch-bound): per-call GPU time
(events around back-to-back calls) and host time per call, under parameter
settings.   python tools/c1_probe.py "" "fused=1" "g=64" ...
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    specs = sys.argv[1:] or [""]
    pp.load(build_if_missing=False)
    n = int(os.environ.get("C1_N", 1 << 20))
    src = synth.uniform_u64_torch(n, synth.SEEDS["c1"], "cuda")
    bufs = [src.clone() for _ in range(60)]
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for spec in specs:
        pp.reset_params()
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            pp.pp_set_param(k, int(v))
        for b in bufs:
            b.copy_(src)
        for b in bufs[:5]:
            pp.pp_partition_async_u64(b, 1 << 63, d)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        t0 = time.perf_counter()
        for b in bufs[5:]:
            pp.pp_partition_async_u64(b, 1 << 63, d)
        t1 = time.perf_counter()
        e.record()
        torch.cuda.synchronize()
        gpu_ms = s.elapsed_time(e) / 55
        # GPU-only: one call at a time, synchronized
        single = []
        for b in bufs[5:25]:
            b.copy_(src)
            torch.cuda.synchronize()
            s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s2.record()
            pp.pp_partition_async_u64(b, 1 << 63, d)
            e2.record()
            torch.cuda.synchronize()
            single.append(s2.elapsed_time(e2))
        single.sort()
        print(json.dumps({"n": n, "spec": spec, "b2b_ms": round(gpu_ms, 4), "host_ms_per_call": round((t1 - t0) * 1e3 / 55, 4),
                          "single_ms": round(single[len(single) // 2], 4)}), flush=True)
    pp.reset_params()


if __name__ == "__main__":
    main()
