#!/usr/bin/env python
"""Time the distributed quicksort through the loopback transport (P emulated
ranks on ONE GPU: local sorts run one after another, exchanges are D2D
copies) -- a proxy for the number and size of distributed rounds, NOT a
multi-GPU number.

    python tools/qs_dist_loopback_time.py [--n 28] [--P 8] [--kinds uniform,dup1000]
"""
import argparse
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
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--kinds", default="uniform,dup1000")
    ap.add_argument("--reps", type=int, default=3)  # (>= 1)
    ap.add_argument("--params", default="", help="k=v,k=v library params")
    a = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, a.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    n = 1 << a.n
    for kind in a.kinds.split(","):
        q0 = (synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda") if kind == "uniform"
              else synth.mod_range_u64_torch(n, synth.SEEDS["c5"], 1000, "cuda"))
        q = torch.empty_like(q0)
        ts = []
        for _ in range(a.reps + 1):
            q.copy_(q0)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            pp.pp_quicksort_dist_loopback(q, [n // a.P] * a.P)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        print({"kind": kind, "P": a.P, "params": a.params, "ms": sorted(ts[1:])[len(ts[1:]) // 2],
               "lib": os.path.basename(pp.LIB_PATH)})


if __name__ == "__main__":
    main()
