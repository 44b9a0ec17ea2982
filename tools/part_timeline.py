#!/usr/bin/env python
"""Kernel timeline (CUPTI via torch.profiler) of single partitions: every
kernel's start / duration relative to the first kernel of the call, and the
GPU-idle gaps -- where the time of a call goes beyond the group kernel.

    python tools/part_timeline.py [--exp 27] [--dtype u64] [--reps 3] [--params k=v,...]
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exp", type=int, default=27)
    ap.add_argument("--dtype", default="u64")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--params", default="")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    n = 1 << args.exp
    u64 = args.dtype == "u64"
    src = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda") if u64 else synth.uniform_u32_torch(n, 7, "cuda")
    pivot = (1 << 63) if u64 else (1 << 31)
    part = pp.pp_partition_async_u64 if u64 else pp.pp_partition_async_u32
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    work = torch.empty_like(src)
    for _ in range(3):
        work.copy_(src)
        part(work, pivot, d)
    torch.cuda.synchronize()
    for r in range(args.reps):
        work.copy_(src)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            part(work, pivot, d)
            torch.cuda.synchronize()
        path = os.path.join(tempfile.mkdtemp(), "t.json")
        prof.export_chrome_trace(path)
        ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
        ev.sort(key=lambda e: e["ts"])
        t0 = ev[0]["ts"]
        end = t0
        print(f"rep {r}: n=2^{args.exp} {args.dtype}")
        for e in ev:
            gap = e["ts"] - end
            print(f"  start {e['ts'] - t0:9.2f} us  dur {e['dur']:8.2f} us  gap {gap:7.2f}  {e['name'][:70]}")
            end = max(end, e["ts"] + e["dur"])
        print(f"  span {end - t0:.2f} us")


if __name__ == "__main__":
    main()
