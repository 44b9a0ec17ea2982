#!/usr/bin/env python
"""Sweep quicksort parameters on BASELINE config 5 (2^28 u64, uniform and
[0,1000)); prints one JSON line per setting.  GPU only.

    python tools/tune_qs.py [--n 28] [--grid "leaf_algo=0,1;qs_waves=2,4"]
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--grid", default="leaf_algo=0,1")
    ap.add_argument("--kinds", default="uniform,dup1000")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    n = 1 << args.n
    axes = []
    for part in args.grid.split(";"):
        k, vs = part.split("=")
        axes.append([(k, int(v)) for v in vs.split(",")])
    for kind in args.kinds.split(","):
        if kind == "uniform":
            q0 = synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda")
        else:
            q0 = synth.mod_range_u64_torch(n, synth.SEEDS["c5"], 1000, "cuda")
        q = torch.empty_like(q0)
        for combo in itertools.product(*axes):
            pp.reset_params()
            for k, v in combo:
                pp.pp_set_param(k, v)
            ts = []
            for r in range(args.reps + 1):
                q.copy_(q0)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                pp.pp_quicksort_u64(q)
                e.record()
                torch.cuda.synchronize()
                if r > 0:
                    ts.append(s.elapsed_time(e))
            ok = bool((q[1:] ^ (-(1 << 63)) >= q[:-1] ^ (-(1 << 63))).all())
            print(json.dumps({"kind": kind, **dict(combo), "ms": round(min(ts), 3),
                              "keys_per_s": n / (min(ts) / 1e3), "sorted": ok}), flush=True)
        del q0, q
    pp.reset_params()


if __name__ == "__main__":
    main()
