#!/usr/bin/env python
"""Config 1 (2^20 u64): time per call and window fraction vs the group count g
(param g; 0 = auto) -- back-to-back calls on fresh copies.

    python tools/c1_groups_probe.py [--exp 20] [--gs 0,16,32,64,96,148]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exp", type=int, default=20)
    ap.add_argument("--gs", default="0,16,32,48,64,96,148")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    n = 1 << args.exp
    src = synth.uniform_u64_torch(n, synth.SEEDS["c1"], "cuda")
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    reps = 150
    bufs = [src.clone() for _ in range(reps + 10)]
    for rnd in range(2):
        for g in map(int, args.gs.split(",")):
            pp.reset_params()
            pp.pp_set_param("g", g)
            for b in bufs:
                b.copy_(src)
            for b in bufs[:10]:
                pp.pp_partition_async_u64(b, 1 << 63, d)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for b in bufs[10:]:
                pp.pp_partition_async_u64(b, 1 << 63, d)
            e.record()
            torch.cuda.synchronize()
            st = pp.pp_last_stats()
            print(rnd, f"g={g:4d} (used {st['g']:4d})  {s.elapsed_time(e) / reps * 1e3:7.1f} us/call  window {st['W'] / n:.4f}",
                  flush=True)


if __name__ == "__main__":
    main()
