#!/usr/bin/env python
"""Short driver for ncu captures: a few c2 partitions (n=2^27 u64, mu=0.5).

    python tools/profile_partition.py [--reps 3] [--n 27]
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n", type=int, default=27)
    ap.add_argument("--dtype", default="u64")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    pp.reset_params()
    n = 1 << args.n
    dev = torch.device("cuda")
    if args.dtype == "u64":
        pristine, piv = synth.uniform_u64_torch(n, synth.SEEDS["c2"], dev), 1 << 63
    else:
        pristine, piv = synth.uniform_u32_torch(n, synth.SEEDS["c2"], dev), 1 << 31
    buf = torch.empty_like(pristine)
    for _ in range(args.reps):
        buf.copy_(pristine)
        split = pp.pp_partition(buf, piv)
    torch.cuda.synchronize()
    print("split", split, pp.pp_last_stats())


if __name__ == "__main__":
    main()
