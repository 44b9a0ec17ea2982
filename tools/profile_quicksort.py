#!/usr/bin/env python
"""Driver for quicksort profiling: sorts n = 2^k u64 keys (uniform or [0,1000)).

    python tools/profile_quicksort.py [--n 28] [--kind uniform|dup1000] [--reps 2] [--params k=v,...]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--kind", default="uniform")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--params", default="", help="k=v,k=v library params")
    ap.add_argument("--dtype", default="u64")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    n = 1 << args.n
    if args.kind == "uniform":
        q0 = (synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda") if args.dtype == "u64"
              else synth.uniform_u32_torch(n, synth.SEEDS["c5"], "cuda"))
    else:
        q0 = synth.mod_range_u64_torch(n, synth.SEEDS["c5"], 1000, "cuda")
        if args.dtype == "u32":
            q0 = q0.to(torch.int32)
    sort = pp.pp_quicksort_u64 if args.dtype == "u64" else pp.pp_quicksort_u32
    q = torch.empty_like(q0)
    for r in range(args.reps):
        q.copy_(q0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sort(q)
        torch.cuda.synchronize()
        print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.2f} ms")


if __name__ == "__main__":
    main()
