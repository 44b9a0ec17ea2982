"""Small-n workloads for compute-sanitizer --
test infrastructure (it imports oracle/).  compute-sanitizer is closed on this
GPU pool; tools/sanitize.sh keeps the recipe for others.

Every kernel family of libpp.so runs once per case at sizes the sanitizer
finishes quickly, each result checked against the oracle (so a tool run is
also a parity run).  Usage (on the GPU box):

    compute-sanitizer --tool racecheck python tests/sanitize_run.py [--only NAME]

tools/sanitize.sh runs memcheck / racecheck / synccheck / initcheck over it
and keeps the logs under profiles/.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402
from gpu_util import to_dev, to_host  # noqa: E402


def part(a, p, **params):
    pp.reset_params()
    for k, v in params.items():
        pp.pp_set_param(k, v)
    t = to_dev(a)
    K = pp.pp_partition(t, p)
    oracle.check_partition(a, to_host(t, a.dtype), p, K)


def qsort(a, **params):
    pp.reset_params()
    for k, v in params.items():
        pp.pp_set_param(k, v)
    t = to_dev(a)
    pp.pp_quicksort(t)
    ref = a.copy()
    oracle.quicksort(ref)
    assert np.array_equal(to_host(t, a.dtype), ref)


def case_partition():
    u64 = synth.uniform_u64_np(300_007, 11)
    u32 = synth.uniform_u32_np(500_003, 12)
    part(u64[:5000], 1 << 63)                                   # single CTA
    part(u64, 1 << 63, small_n=1 << 12, cleanup_chain=1)        # group + 3-kernel cleanup chain
    part(u64, 1 << 62, small_n=1 << 12, cleanup_chain=0)        # group + fused tail (bitmap)
    part(u64, 1 << 63, small_n=1 << 12, cleanup_chain=0, cleanup_bitmap=0)  # fused tail, grid barrier
    part(u64, 1 << 63, small_n=1 << 12, path=3)                 # cleanup only
    part(u32, 1 << 31, small_n=1 << 12)
    part(u32, 1 << 30, small_n=1 << 12, cleanup_chain=0)


def case_quicksort():
    qsort(synth.uniform_u64_np(1 << 19, 21), qs_heavy=1 << 17)
    qsort(synth.mod_range_u64_np(1 << 19, 22, 1000))
    qsort(synth.uniform_u32_np(1 << 19, 23))


def case_bps_stable():
    a = synth.uniform_u64_np(200_003, 31)
    pp.reset_params()
    t = to_dev(a)
    K = pp.pp_partition_bps(t, 1 << 63)
    ref = a.copy()
    Kr = oracle.partition_bps(ref, 1 << 63)
    assert K == Kr and np.array_equal(to_host(t, np.uint64), ref)
    t = to_dev(a)
    o = torch.empty_like(t)
    K = pp.pp_partition_stable(t, o, 1 << 63)
    ref = a.copy()
    Kr = oracle.partition_standard(ref, 1 << 63)
    assert K == Kr and np.array_equal(to_host(o, np.uint64), ref)


def case_dist():
    """Loopback transport: P emulated ranks on one GPU (pp_dist_loopback_*)."""
    if not hasattr(pp, "pp_partition_dist_loopback"):
        return
    a = synth.uniform_u64_np(400_009, 41)
    ns = [100_000, 0, 150_000, 150_009]
    t = to_dev(a)
    pp.reset_params()
    pp.pp_dist_set_staging(1 << 16)
    K = pp.pp_partition_dist_loopback(t, ns, 1 << 63)
    oracle.check_partition(a, to_host(t, np.uint64), 1 << 63, K)
    t = to_dev(a)
    pp.pp_set_param("dist_small", 4096)
    pp.pp_quicksort_dist_loopback(t, ns)
    ref = a.copy()
    oracle.quicksort(ref)
    assert np.array_equal(to_host(t, np.uint64), ref)


CASES = {"partition": case_partition, "quicksort": case_quicksort, "bps_stable": case_bps_stable,
         "dist": case_dist}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for name, fn in CASES.items():
        if args.only and name not in args.only.split(","):
            continue
        fn()
        torch.cuda.synchronize()
        print(f"sanitize case {name}: ok", flush=True)
