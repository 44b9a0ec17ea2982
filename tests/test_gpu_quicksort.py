"""GPU parity: the CUDA quicksort (through the C ABI) against the CPU oracle sort."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

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


def _sort_gpu(pp, a: np.ndarray, offset: int = 0, **params):
    from gpu_util import to_dev, to_host
    for k, v in params.items():
        pp.pp_set_param(k, v)
    try:
        pad = np.zeros(offset, dtype=a.dtype)
        buf = to_dev(np.concatenate([pad, a, pad]))
        view = buf[offset:offset + a.size]
        pp.pp_quicksort(view)
        full = to_host(buf, a.dtype)
        assert np.all(full[:offset] == 0) and np.all(full[offset + a.size:] == 0)
        return full[offset:offset + a.size]
    finally:
        pp.reset_params()


def _oracle_sorted(a):
    b = a.copy()
    oracle.quicksort(b)
    return b


def _cases(dt, mx, n, rng):
    yield rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
    yield rng.integers(0, 1000, size=n).astype(dt)
    yield np.full(n, 7, dtype=dt)
    yield np.full(n, mx, dtype=dt)
    yield np.arange(n, dtype=dt)
    yield np.arange(n, dtype=dt)[::-1].copy()
    yield (rng.integers(0, 2, size=n).astype(dt) * dt(mx))


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_small_sizes(pp, dt, mx):
    rng = np.random.default_rng(1)
    for n in list(range(0, 40)) + [255, 256, 257, 4095, 4096, 4097, 8191, 8192, 8193, 12289, 16383, 16384,
                                   16385, 20000, 32769]:
        for a in _cases(dt, mx, n, rng):
            for off in (0, 1):
                out = _sort_gpu(pp, a, off)
                assert np.array_equal(out, _oracle_sorted(a)), (n, off)


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
@pytest.mark.parametrize("dev", [0, 1])
def test_medium_sizes(pp, dt, mx, dev):
    """Host-built (qs_dev = 0) and device-built (qs_dev = 1: qs_build_kernel
    makes every lane level below qs_heavy) level loops."""
    rng = np.random.default_rng(2)
    for n in (100_003, 1 << 20, 3_000_017):
        for a in _cases(dt, mx, n, rng):
            out = _sort_gpu(pp, a, 3, qs_dev=dev)
            assert np.array_equal(out, _oracle_sorted(a)), n


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
@pytest.mark.parametrize("params", [{"leaf": 300}, {"leaf": 1000}, {"leaf": 4096}, {"leaf": 8192},
                                    {"qs_waves": 1}, {"qs_waves": 16, "leaf": 1000},
                                    {"qs_heavy": 1 << 17}, {"qs_heavy": 0}, {"qs_small": 0}, {"strided": 1},
                                    {"qs_lanes": 1}, {"qs_lanes": 2}, {"qs_lanes": 2, "qs_small": 1 << 17},
                                    {"qs_early": 1}, {"qs_early": 1, "qs_lanes": 1}, {"qs_early": 0},
                                    {"qs_deep": 0}, {"qs_deep": 3}, {"qs_deep": 0, "qs_cta_max": 1 << 12},
                                    {"qs_pivot": 1}, {"qs_pivot": 2}, {"qs_pivot": 2, "qs_cta_max": 1 << 16},
                                    {"qs_prio": 0}, {"qs_prio": 0, "qs_lanes": 1},
                                    {"qs_dev": 1}, {"qs_dev": 1, "qs_heavy": 0},
                                    {"qs_dev": 1, "qs_heavy": 0, "qs_waves": 16},
                                    {"qs_dev": 1, "qs_heavy": 0, "qs_pivot": 2},
                                    {"qs_dev": 1, "qs_heavy": 0, "qs_small": 1 << 17},
                                    {"qs_dev": 1, "qs_heavy": 0, "qs_pivot": 1, "leaf": 1000},
                                    {"qs_dev": 1, "qs_dev_check": 1, "qs_heavy": 0},
                                    {"qs_dev": 1, "qs_dev_check": 1, "qs_heavy": 0, "qs_waves": 16},
                                    {"qs_dev": 1, "qs_dev_check": 1, "qs_heavy": 0, "qs_pivot": 2}])
def test_qs_parameters(pp, dt, mx, params):
    """Bin sizes (both bin-sort CTA shapes), level balancing, the
    heavy-segment batched cleanup, the per-CTA recursion, the Strided
    offsets, the stream layout without priorities (qs_prio = 0: lane 0
    on the caller's stream) and the device-built levels (qs_dev = 1, from the
    first lane level on with qs_heavy = 0) all give the oracle's sorted
    output; with qs_dev_check every device-built level list must equal the
    host's plan of the same children (order, groups incl. the straggler
    take-back, first tasks, depth, bounds)."""
    rng = np.random.default_rng(4)
    for n in (5000, 300_007):
        for a in list(_cases(dt, mx, n, rng))[:3]:
            out = _sort_gpu(pp, a, 1, **params)
            assert np.array_equal(out, _oracle_sorted(a)), (n, params)


def test_big_path_forced(pp):
    """Force the multi-CTA partition for mid-size segments (qs_cta_max small)."""
    rng = np.random.default_rng(3)
    for a in (rng.integers(0, U64_MAX, size=2_000_003, dtype=np.uint64, endpoint=True),
              rng.integers(0, 50, size=2_000_003).astype(np.uint64)):
        out = _sort_gpu(pp, a, 1, qs_cta_max=1 << 16)
        assert np.array_equal(out, _oracle_sorted(a))


@pytest.mark.parametrize("kind", ["uniform", "dup1000"])
def test_config5_full(pp, kind):
    """n = 2^28 u64 (BASELINE config 5), byte for byte against the oracle's
    serial quicksort of the same seed-regenerated input (north_star (4);
    ~25 s of host time per input); both level loops (host-built, and
    device-built with qs_dev = 1), and the 8-GPU form through 8 emulated
    ranks."""
    n = 1 << 28
    if kind == "uniform":
        t = synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda")
        ref = synth.uniform_u64_np(n, synth.SEEDS["c5"])
    else:
        t = synth.mod_range_u64_torch(n, synth.SEEDS["c5"], 1000, "cuda")
        ref = synth.mod_range_u64_np(n, synth.SEEDS["c5"], 1000)
    t2 = t.clone()
    t8 = t.clone()
    pp.pp_quicksort(t)
    oracle.quicksort(ref)
    out = t.cpu().numpy().view(np.uint64)
    assert np.array_equal(out, ref)
    # the device-built level loop (qs_dev = 1) on the same input
    pp.pp_set_param("qs_dev", 1)
    try:
        pp.pp_quicksort(t2)
    finally:
        pp.reset_params()
    assert np.array_equal(t2.cpu().numpy().view(np.uint64), ref)
    # config 5 on 8 GPUs: the distributed quicksort (spanning segments
    # partitioned across ranks, the rest sorted locally) with 8 emulated ranks
    # of 2^25 keys on this GPU (loopback transport, the product code path)
    del t2
    pp.pp_quicksort_dist_loopback(t8, [n // 8] * 8)
    assert np.array_equal(t8.cpu().numpy().view(np.uint64), ref)


@pytest.mark.parametrize("leaf", [0, 1000, 4096, 8192, 12000, 10240])
def test_bin_sorts_clustered(pp, leaf):
    """Bins whose keys cluster inside a wide range: the counting bin sort sees
    crowded buckets (> 48 keys in a bucket while the shift is > 0) and hands
    the bin to the merge sort (qs_leaf_handoff_kernel); buckets at and around
    the limit; every bin capacity gives the oracle's order."""
    rng = np.random.default_rng(9)
    cases = []
    # 100 clusters of 50 distinct keys each + the maximum: runs of 50 equal tops
    cl = (np.arange(100, dtype=np.uint64)[:, None] << np.uint64(40)) + np.arange(50, dtype=np.uint64)[None, :]
    cases.append(np.concatenate([cl.reshape(-1), np.array([U64_MAX], dtype=np.uint64)]))
    # one cluster of 6000 distinct small keys + two huge ones: a run of 6000 -> fallback
    cases.append(np.concatenate([np.arange(6000, dtype=np.uint64), np.array([1 << 63, U64_MAX], dtype=np.uint64)]))
    # clusters of 80 (just above the run limit) and of 64 (at it)
    for w in (80, 64, 65, 47, 48, 49, 20, 300):
        c = (np.arange(60, dtype=np.uint64)[:, None] << np.uint64(45)) + np.arange(w, dtype=np.uint64)[None, :]
        cases.append(np.concatenate([c.reshape(-1), np.array([U64_MAX - 5], dtype=np.uint64)]))
    # duplicates of few values spread over the whole range
    cases.append(rng.choice(np.array([0, 5, 1 << 40, 1 << 63, U64_MAX], dtype=np.uint64), size=8000))
    for a in cases:
        a = a[rng.permutation(a.size)]
        for n in (a.size, min(a.size, 8192), min(a.size, 16384), min(a.size, 12345), 300):
            b = a[:n].copy()
            out = _sort_gpu(pp, b, 1, leaf=leaf)
            assert np.array_equal(out, _oracle_sorted(b)), (leaf, n)
    # the same clusters inside a large quicksort (bins from the per-CTA recursion)
    big = np.concatenate([c.reshape(-1) for c in [cl] * 40] + [synth.uniform_u64_np(300000, 3)])
    big = big[rng.permutation(big.size)]
    out = _sort_gpu(pp, big, 0, leaf=leaf)
    assert np.array_equal(out, _oracle_sorted(big))


@pytest.mark.parametrize("kind", ["uniform", "dup1000"])
def test_quicksort_2pow30(pp, kind):
    """4x config 5 (2^30 u64 = 8 GiB): beyond the benchmarked size (segment
    lists, bin slots, heavy-segment batches all scale); the output equals the
    library sort (torch.sort on the order-preserving image)."""
    from gpu_util import order_key
    n = 1 << 30
    t = (synth.uniform_u64_torch(n, 77, "cuda") if kind == "uniform"
         else synth.mod_range_u64_torch(n, 77, 1000, "cuda"))
    ref = torch.sort(order_key(t)).values
    pp.pp_quicksort(t)
    assert torch.equal(order_key(t), ref)
    del t, ref
    torch.cuda.empty_cache()



def test_quicksort_last_stats(pp):
    """pp_quicksort_last_stats: the level loop partitions every key once per
    level while its segment is above qs_small (level_keys >= n for n above it),
    and every key ends in a small segment or a leaf list (or an all-equal
    range, which no list holds): small_keys + leaf_keys <= n."""
    from gpu_util import to_dev
    n = 1 << 22
    a = synth.uniform_u64_np(n, 4)
    t = to_dev(a)
    pp.pp_quicksort(t)
    st = pp.pp_quicksort_last_stats()
    assert st["n"] == n and st["levels"] >= 5 and st["level_keys"] >= 5 * n
    assert 0 < st["small_keys"] + st["leaf_keys"] <= n and st["nsmall"] > 0
    t = to_dev(np.full(1000, 5, dtype=np.uint64))
    pp.pp_quicksort(t)
    st = pp.pp_quicksort_last_stats()
    assert st["n"] == 1000 and st["levels"] == 0 and st["leaf_keys"] == 1000


def test_deep_segments_take_the_ninther(pp):
    """Segments deeper than qs_deep switch from the median of 3 to Tukey's
    ninther (the guard against inputs that make the median of 3 peel off a
    few keys per level): with qs_deep = 0 every level segment (device-side
    pivots) and every big segment (host-read pivots, qs_cta_max small) uses
    it; the result is still the oracle's sort, in a similar number of levels."""
    from gpu_util import to_dev, to_host
    for a in (synth.uniform_u64_np(3_000_017, 7), synth.mod_range_u64_np(2_000_003, 8, 1000),
              np.concatenate([np.arange(1 << 20, dtype=np.uint64), np.arange(1 << 20, dtype=np.uint64)[::-1]])):
        ref = _oracle_sorted(a)
        levels = []
        for params in ({}, {"qs_deep": 0}, {"qs_deep": 0, "qs_cta_max": 1 << 16}, {"qs_pivot": 2},
                       {"qs_pivot": 2, "qs_cta_max": 1 << 16}):
            for k, v in params.items():
                pp.pp_set_param(k, v)
            try:
                t = to_dev(a)
                pp.pp_quicksort(t)
                levels.append(pp.pp_quicksort_last_stats()["levels"])
            finally:
                pp.reset_params()
            assert np.array_equal(to_host(t, np.uint64), ref), params
        # (the arrangement a partition leaves depends on the group layout, so the
        # median of 3 on the sorted / reversed halves may take ~3x the levels of
        # the ninther; the depth guard QS_DEEP = 2 log2 n + 16 bounds it)
        assert max(levels) <= 3 * min(levels) + 4, levels


@pytest.mark.parametrize("kind", ["uniform", "dup1000"])
def test_device_built_levels_match_host_plan(pp, kind):
    """qs_dev = 1 with qs_dev_check: at every device-built level of a 2^25-key
    config-5-like sort the list qs_build_kernel made equals the host's plan
    of the same children (order, group counts incl. the straggler take-back,
    first tasks, depth, bounds), and the output is sorted."""
    from gpu_util import to_dev, to_host
    n = 1 << 25
    a = synth.uniform_u64_np(n, 5) if kind == "uniform" else synth.mod_range_u64_np(n, 5, 1000)
    ref = np.sort(a)
    for extra in ({}, {"qs_waves": 16}, {"qs_heavy": 0}, {"qs_heavy": 0, "qs_pivot": 2}):
        t = to_dev(a)
        pp.pp_set_param("qs_dev", 1)
        pp.pp_set_param("qs_dev_check", 1)
        try:
            for k, v in extra.items():
                pp.pp_set_param(k, v)
            pp.pp_quicksort(t)
        finally:
            pp.reset_params()
        assert np.array_equal(to_host(t, np.uint64), ref), extra
