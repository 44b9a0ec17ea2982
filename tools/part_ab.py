#!/usr/bin/env python
"""Partition timings for A/B runs (CUDA events, median of reps, fresh copy of
the input before every rep): c2 uniform u64 2^27 and the c4 u32 patterns.

    PP_LIB_PATH=... python tools/part_ab.py [--c4 partitioned,all_false,reverse]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def timed(fn, src, reps):
    work = torch.empty_like(src)
    ts = []
    for r in range(reps + 2):
        work.copy_(src)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(work)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return round(ts[len(ts) // 2], 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", default="partitioned,all_false,all_true,reverse")
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--params", default="", help="k=v,k=v library params")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    res = {"lib": os.environ.get("PP_LIB_PATH", "default"), "params": args.params}
    c2 = synth.uniform_u64_torch(1 << 27, synth.SEEDS["c2"], "cuda")
    res["c2"] = timed(lambda w: pp.pp_partition_async_u64(w, 1 << 63, d), c2, args.reps)
    del c2
    for pat in filter(None, args.c4.split(",")):
        a = synth.adversarial_u32_torch(1_000_000_007, pat, synth.SEEDS["c4"], "cuda")
        res["c4_" + pat] = timed(lambda w: pp.pp_partition_async_u32(w, synth.ADV_PIVOT_U32, d), a, args.reps)
        del a
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
