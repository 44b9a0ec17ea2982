"""Seeded fuzzing of the CUDA paths against the CPU oracle: random sizes,
base alignments, key distributions, pivots and tuning-parameter
combinations (paths, group counts, cleanup tails,
Strided offsets, bin sorts, quicksort thresholds).  Deterministic (fixed
seeds), so a failure reproduces."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle

pytestmark = pytest.mark.gpu

U64_MAX = (1 << 64) - 1
U32_MAX = (1 << 32) - 1


@pytest.fixture(scope="module")
def pp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2004_12532_b200 as m
    m.load()
    m.reset_params()
    yield m
    m.reset_params()


def _keys(rng, n, dt, mx):
    kind = rng.integers(0, 7)
    if kind == 0:
        return rng.integers(0, mx, size=n, dtype=dt, endpoint=True), "uniform"
    if kind == 1:
        return rng.integers(0, int(rng.integers(1, 50)), size=n).astype(dt), "alphabet"
    if kind == 2:
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        return np.sort(a), "sorted"
    if kind == 3:
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        return np.sort(a)[::-1].copy(), "reverse"
    if kind == 4:  # clusters inside a wide range
        c = rng.integers(0, 64, size=n).astype(np.uint64) << np.uint64(40 if dt == np.uint64 else 26)
        return (c + rng.integers(0, 100, size=n).astype(np.uint64)).astype(dt), "clusters"
    if kind == 5:  # whole blocks of 1024 true or false
        blocks = rng.integers(0, 2, size=n // 1024 + 1).astype(bool)
        t = np.repeat(blocks, 1024)[:n]
        lo = rng.integers(0, mx // 2, size=n, dtype=dt)
        return np.where(t, lo, lo + dt(mx // 2 + 1)).astype(dt), "blocks"
    return np.full(n, rng.integers(0, mx, dtype=dt, endpoint=True), dtype=dt), "constant"


def _pivot(rng, a, mx):
    choice = rng.integers(0, 5)
    if choice == 0 or a.size == 0:
        return int(rng.integers(0, mx, endpoint=True, dtype=np.uint64 if mx == U64_MAX else np.uint32))
    if choice == 1:
        return int(a[rng.integers(0, a.size)])
    if choice == 2:
        return int(np.sort(a)[a.size // 2])
    return [0, 1, mx][int(rng.integers(0, 3))]


PARTITION_PARAMS = [
    {}, {"path": 1}, {"path": 3}, {"small_n": 0}, {"small_n": 0, "min_lines_per_group": 1},
    {"g": 3}, {"g": 64}, {"cleanup_chain": 1},
    {"cleanup_chain": 0}, {"cleanup_chain": 0, "small_n": 0},
    {"cleanup_bitmap": 0}, {"strided": 1}, {"strided": 1, "small_n": 0},
]


def test_fuzz_partition(pp):
    from gpu_util import to_dev, to_host
    import os
    rng = np.random.default_rng(int(os.environ.get("PP_FUZZ_SEED", 2004_12532)))
    for it in range(int(os.environ.get("PP_FUZZ_ITERS", 160))):
        dt, mx = ((np.uint64, U64_MAX) if rng.integers(0, 2) else (np.uint32, U32_MAX))
        n = int(rng.choice([rng.integers(0, 100), rng.integers(100, 70000), rng.integers(70000, 3_000_000)]))
        a, kind = _keys(rng, n, dt, mx)
        p = _pivot(rng, a, mx)
        off = int(rng.integers(0, 4))
        params = PARTITION_PARAMS[int(rng.integers(0, len(PARTITION_PARAMS)))]
        algo = int(rng.integers(0, 6))  # 0-3: in-place partition, 4: BPS, 5: Standard Algorithm
        for k, v in params.items():
            pp.pp_set_param(k, v)
        try:
            buf = to_dev(np.concatenate([np.zeros(off, dtype=dt), a, np.zeros(3, dtype=dt)]))
            view = buf[off:off + n]
            ctx = (it, n, kind, p, off, params, algo)
            if algo == 4:
                split = pp.pp_partition_bps(view, p)
                ref = a.copy()
                assert split == oracle.partition_bps(ref, p, 4096), ctx
                assert np.array_equal(to_host(view, dt), ref), ctx
            elif algo == 5:
                out = torch.zeros_like(view)
                split = pp.pp_partition_stable(view, out, p)
                ref = a.copy()
                assert split == oracle.partition_standard(ref, p), ctx
                assert np.array_equal(to_host(out, dt), ref), ctx
            else:
                split = pp.pp_partition(view, p)
                oracle.check_partition(a, to_host(view, dt), p, split)
            full = to_host(buf, dt)
            assert np.all(full[:off] == 0) and np.all(full[off + n:] == 0), ctx
        finally:
            pp.reset_params()


QUICKSORT_PARAMS = [
    {}, {"leaf": 1000}, {"leaf": 4096}, {"leaf": 2000}, {"leaf": 8192},
    {"qs_small": 0}, {"qs_small": 1 << 18}, {"qs_cta_max": 1 << 16}, {"qs_heavy": 1 << 17},
    {"qs_heavy": 0}, {"qs_waves": 1}, {"qs_lanes": 1}, {"qs_lanes": 2, "qs_cta_max": 1 << 18},
    {"qs_pivot": 1}, {"qs_pivot": 2}, {"qs_deep": 0},
    {"qs_early": 1}, {"qs_early": 1, "qs_small": 1 << 17, "qs_cta_max": 1 << 19},
    {"qs_dev": 1}, {"qs_dev": 1, "qs_heavy": 0}, {"qs_dev": 1, "qs_heavy": 0, "qs_pivot": 2},
    {"qs_dev": 1, "qs_dev_check": 1, "qs_heavy": 0}, {"qs_dev": 1, "qs_dev_check": 1, "qs_heavy": 0, "qs_waves": 8},
]


def test_fuzz_quicksort(pp):
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(1732)
    for it in range(60):
        dt, mx = ((np.uint64, U64_MAX) if rng.integers(0, 2) else (np.uint32, U32_MAX))
        n = int(rng.choice([rng.integers(0, 300), rng.integers(300, 100000), rng.integers(100000, 2_000_000)]))
        a, kind = _keys(rng, n, dt, mx)
        off = int(rng.integers(0, 4))
        params = QUICKSORT_PARAMS[int(rng.integers(0, len(QUICKSORT_PARAMS)))]
        for k, v in params.items():
            pp.pp_set_param(k, v)
        try:
            buf = to_dev(np.concatenate([np.zeros(off, dtype=dt), a, np.zeros(3, dtype=dt)]))
            view = buf[off:off + n]
            pp.pp_quicksort(view)
            ref = a.copy()
            oracle.quicksort(ref)
            assert np.array_equal(to_host(view, dt), ref), (it, n, kind, off, params)
            full = to_host(buf, dt)
            assert np.all(full[:off] == 0) and np.all(full[off + n:] == 0)
        finally:
            pp.reset_params()
