#!/usr/bin/env python
"""Extended quicksort stress (GPU): random sizes, key distributions, widths
and tuning parameters (incl. the two-lane level loop and the early per-CTA
recursion), each result checked against numpy's sort.  Seeded from argv.

    python tools/fuzz_qs.py [iterations] [seed]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402

PARAMS = [{}, {"qs_lanes": 1}, {"qs_early": 0}, {"qs_lanes": 1, "qs_early": 1}, {"qs_early_min": 1},
          {"qs_small": 1 << 17}, {"qs_cta_max": 1 << 18}, {"qs_heavy": 1 << 17}, {"leaf": 5000},
          {"leaf_algo": 5}, {"qs_minl": 4}, {"qs_early_min": 1, "qs_small": 1 << 15, "qs_cta_max": 1 << 20}]


def keys(rng, n, dt):
    mx = np.iinfo(dt).max
    k = int(rng.integers(0, 6))
    if k == 0:
        return rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
    if k == 1:
        return rng.integers(0, int(rng.integers(1, 3000)), size=n).astype(dt)
    if k == 2:
        c = rng.integers(0, 40, size=n).astype(np.uint64) << np.uint64(40 if dt == np.uint64 else 26)
        return (c + rng.integers(0, 5000, size=n).astype(np.uint64)).astype(dt)
    if k == 3:
        return np.sort(rng.integers(0, mx, size=n, dtype=dt, endpoint=True))[::-1].copy()
    if k == 4:  # zipf-like
        z = rng.zipf(1.2, size=n)  # int64; clip to the key range (and to int64 for u64)
        return np.minimum(z, min(int(mx), np.iinfo(np.int64).max)).astype(dt)
    return np.full(n, rng.integers(0, mx, dtype=dt, endpoint=True), dtype=dt)


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 7
    rng = np.random.default_rng(seed)
    pp.load(build_if_missing=False)
    bad = 0
    for it in range(iters):
        dt = np.uint64 if rng.integers(0, 2) else np.uint32
        n = int(rng.choice([rng.integers(0, 5000), rng.integers(5000, 400000), rng.integers(400000, 6000000)]))
        a = keys(rng, n, dt)
        prm = PARAMS[int(rng.integers(0, len(PARAMS)))]
        pp.reset_params()
        for k, v in prm.items():
            pp.pp_set_param(k, v)
        t = torch.from_numpy(a.view(np.int64 if dt == np.uint64 else np.int32).copy()).cuda()
        pp.pp_quicksort(t) if dt == np.uint64 else pp.pp_quicksort_u32(t)
        out = t.cpu().numpy().view(dt)
        if not np.array_equal(out, np.sort(a)):
            bad += 1
            print("MISMATCH", it, n, dt.__name__, prm, flush=True)
    pp.reset_params()
    print(f"fuzz_qs: {iters} sorts, {bad} mismatches (seed {seed})", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
