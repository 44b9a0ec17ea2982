#!/usr/bin/env python
"""Sweep group-kernel variants / group counts on the c2 workload and print a
table (group-kernel ms, whole-partition ms, effective GB/s, window).  GPU only.

    python tools/tune.py [--n 27] [--variants 0,1,2] [--mlpg 16] [--reps 10]
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


def run(n, pivot, variant, reps, dtype="u64", **params):
    pp.reset_params()
    pp.pp_set_param("variant", variant)
    for k, v in params.items():
        pp.pp_set_param(k, v)
    dev = torch.device("cuda")
    if dtype == "u64":
        pristine = synth.uniform_u64_torch(n, synth.SEEDS["c2"], dev)
    else:
        pristine = synth.uniform_u32_torch(n, synth.SEEDS["c2"], dev)
    buf = torch.empty_like(pristine)
    flush = torch.empty(64 << 20, dtype=torch.int64, device=dev)
    d = torch.zeros(1, dtype=torch.int64, device=dev)
    f = pp.pp_partition_async_u64 if dtype == "u64" else pp.pp_partition_async_u32
    for i in range(3):
        buf.copy_(pristine)
        f(buf, pivot, d)
    torch.cuda.synchronize()
    pp.pp_timing(True)
    for i in range(reps):
        buf.copy_(pristine)
        flush.fill_(i)
        f(buf, pivot, d)
    torch.cuda.synchronize()
    t = pp.pp_timing_read()
    pp.pp_timing(False)
    st = pp.pp_last_stats()
    w = 8 if dtype == "u64" else 4
    tot = t["total_ms"] / t["calls"]
    grp = t["group_ms"] / t["calls"]
    res = {"variant": variant, **params, "g": st["g"], "LK": st["line_keys"], "grp_ms": round(grp, 4),
           "rest_ms": round(t["rest_ms"] / t["calls"], 4), "total_ms": round(tot, 4),
           "grp_GBs": round(2 * w * st["n_lines"] * st["line_keys"] / grp / 1e6, 1),
           "eff_GBs": round(2 * w * n / tot / 1e6, 1), "window_frac": round(st["W"] / n, 5), "M": st["M"],
           "nTasks": st["nTasks"]}
    pp.reset_params()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=27)
    ap.add_argument("--variants", default="0,1,2,3,4,5,6")
    ap.add_argument("--mlpg", default="16")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dtype", default="u64")
    ap.add_argument("--mu", type=float, default=0.5)
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    n = 1 << args.n
    pivot = synth.PIVOT_MU[args.mu] if args.dtype == "u64" else int(args.mu * (1 << 32))
    for v in [int(x) for x in args.variants.split(",")]:
        for m in [int(x) for x in args.mlpg.split(",")]:
            print(json.dumps(run(n, pivot, v, args.reps, args.dtype, min_lines_per_group=m)), flush=True)


if __name__ == "__main__":
    main()
