"""EREW shadow-writer audit of the partition (test infrastructure; run by
tests/test_gpu_audit.py in a subprocess with PP_LIB_PATH pointing at the
debug build libpp_audit.so).

PAPER.md:229-238 (the EREW model: no two processors write one cell at once)
and SPEC's element-level auditor: every store of a key by the
partition's kernels bumps a per-key counter -- 1 for the Smoothed Striding
group kernel, 1 << 16 for the cleanup kernels (include/pp.h pp_audit_set).
Per call this checks
  - each key is written at most once by the group kernel and at most once by
    the cleanup (EREW per phase);
  - the group kernel writes exactly the keys of its full lines
    [head, head + n_lines * line_keys) -- every line read once and written
    once (Prop. 4.2's one pass) -- and nothing when the
    path has no group step;
  - the cleanup writes exactly 2 M keys (M misplaced pairs, pp_last_stats),
    and, when no group step ran before it, exactly the misplaced positions of
    the input;
  - the result is the oracle's partition (split, predicate, per-side
    multisets).
Prints one line per case and "EREW AUDIT OK" at the end; exits non-zero on
the first violation.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_12532_b200 as pp  # noqa: E402
from gpu_util import to_dev, to_host  # noqa: E402

U64_MAX = (1 << 64) - 1
U32_MAX = (1 << 32) - 1


def run_case(a: np.ndarray, pivot: int, off: int, params: dict) -> str:
    dt = a.dtype
    n = a.size
    pad = np.zeros(off, dtype=dt)
    buf = to_dev(np.concatenate([pad, a, pad]))
    view = buf[off:off + n]
    shadow = torch.zeros(n, dtype=torch.int32, device=view.device)
    for k, v in params.items():
        pp.pp_set_param(k, v)
    try:
        pp.pp_audit_set(shadow, view)
        split = pp.pp_partition(view, pivot)
        torch.cuda.synchronize()
        pp.pp_audit_set(None)
        st = pp.pp_last_stats()
    finally:
        pp.reset_params()
    out = to_host(view, dt)
    oracle.check_partition(a, out, pivot, split)
    full = to_host(buf, dt)
    assert np.all(full[:off] == 0) and np.all(full[off + n:] == 0), "write outside the keys"
    sh = shadow.cpu().numpy().view(np.uint32)
    grp, cln = sh & 0xFFFF, sh >> 16
    assert grp.max(initial=0) <= 1, f"a key written {grp.max()} times by the group kernel"
    assert cln.max(initial=0) <= 1, f"a key written {cln.max()} times by the cleanup"
    path = st["path"] if st["n"] == n else 0  # (0: the call returned before any kernel, e.g. n < 2)
    if path == 2:
        lo, hi = st["head"], st["head"] + st["n_lines"] * st["line_keys"]
        want = np.zeros(n, dtype=np.uint32)
        want[lo:hi] = 1
        assert np.array_equal(grp, want), "group kernel did not write exactly its full lines once"
        assert int(cln.sum()) == 2 * st["M"], (int(cln.sum()), st["M"])
    else:
        assert grp.sum() == 0, "group writes on a path without a group step"
        K = split
        mis = np.zeros(n, dtype=bool)
        mis[:K] = a[:K] >= pivot
        mis[K:] = a[K:] < pivot
        assert np.array_equal(cln == 1, mis), "cleanup did not write exactly the misplaced keys"
    return (f"n={n} {dt.name} off={off} {params} path={path} split={split} "
            f"group_writes={int(grp.sum())} cleanup_writes={int(cln.sum())} M={st['M']}")


def main() -> int:
    assert torch.cuda.is_available()
    assert os.path.basename(pp.LIB_PATH) == "libpp_audit.so", pp.LIB_PATH
    rng = np.random.default_rng(229)
    cases = []
    for dt, mx in ((np.uint64, U64_MAX), (np.uint32, U32_MAX)):
        for n in (1, 37, 5000, 40_000, 300_007, 1 << 22):
            a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
            for mu in (0.01, 0.5, 0.99):
                p = int(mx * mu)
                cases.append((a, p, int(rng.integers(0, 4)), {}))
            cases.append((a, 0, 1, {}))
            cases.append((a, mx, 2, {}))
        a = rng.integers(0, mx, size=1 << 21, dtype=dt, endpoint=True)
        p = int(mx // 2)
        for params in ({"cleanup_chain": 0}, {"cleanup_chain": 1}, {"cleanup_chain": 0, "cleanup_bitmap": 0},
                       {"path": 3}, {"path": 1}, {"strided": 1}, {"tile": 2048}, {"g": 37}):
            cases.append((a, p, 3, params))
        # structured inputs: already partitioned, reverse partitioned, alternating
        n = 1 << 20
        half = np.concatenate([np.zeros(n // 2, dtype=dt), np.full(n - n // 2, mx, dtype=dt)])
        cases.append((half, 1, 0, {}))
        cases.append((half[::-1].copy(), 1, 0, {}))
        alt = np.where(np.arange(n) % 2 == 0, dt(0), dt(mx)).astype(dt)
        cases.append((alt, 1, 1, {}))
    for a, p, off, params in cases:
        print(run_case(a, p, off, params), flush=True)
    print("EREW AUDIT OK")
    return 0


if __name__ == "__main__":
    sys.exit(main())
