#!/usr/bin/env python
"""A/B quicksort parameter settings on the GPU (CUDA-event timing, median of
reps), each result checked against the library sort.

    python tools/qs_ab.py "" "leaf=8192" "qs_early=0" [--n 28] [--kinds uniform,dup1000] [--dtype u64]
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


def lib_sorted(x):
    """Ascending unsigned order via the library sort (sign-flipped signed view)."""
    if x.dtype == torch.int64:
        flip = torch.tensor(-(1 << 63), dtype=torch.int64, device=x.device)
    else:
        flip = torch.tensor(-(1 << 31), dtype=torch.int32, device=x.device)
    return torch.sort(x ^ flip).values ^ flip


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="*", default=[""])
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--kinds", default="uniform,dup1000")
    ap.add_argument("--dtype", default="u64")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--seed", type=int, default=None, help="input seed (default: config 5's)")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    n = 1 << args.n
    seed = synth.SEEDS["c5"] if args.seed is None else args.seed
    inputs = {}
    for kind in args.kinds.split(","):
        if kind == "uniform":
            q0 = (synth.uniform_u64_torch(n, seed, "cuda") if args.dtype == "u64"
                  else synth.uniform_u32_torch(n, seed, "cuda"))
        else:  # dup1000, dup10000, ...: keys uniform in [0, m)
            m = int(kind[3:]) if kind.startswith("dup") and kind[3:].isdigit() else 1000
            q0 = synth.mod_range_u64_torch(n, seed, m, "cuda")
            if args.dtype == "u32":
                q0 = q0.to(torch.int32)
        inputs[kind] = (q0, lib_sorted(q0))
    sort = pp.pp_quicksort_u64 if args.dtype == "u64" else pp.pp_quicksort_u32
    for rnd in range(args.rounds):
        for spec in args.specs:
            pp.reset_params()
            for kv in filter(None, spec.split(",")):
                k, v = kv.split("=")
                pp.pp_set_param(k, int(v))
            res = {"spec": spec, "round": rnd}
            for kind, (q0, ref) in inputs.items():
                q = torch.empty_like(q0)
                times = []
                for r in range(args.reps + 1):
                    q.copy_(q0)
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    sort(q)
                    b.record()
                    torch.cuda.synchronize()
                    if r > 0:
                        times.append(a.elapsed_time(b))
                ok = bool(torch.equal(q, ref))
                times.sort()
                res[kind] = round(times[len(times) // 2], 3)
                res[kind + "_ok"] = ok
            print(json.dumps(res), flush=True)
    pp.reset_params()


if __name__ == "__main__":
    main()
