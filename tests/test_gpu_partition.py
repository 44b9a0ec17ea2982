"""GPU parity: the CUDA partition (through the C ABI) against the CPU oracle."""
import functools
import os

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


def _run(pp, a: np.ndarray, pivot: int, offset: int = 0, **params):
    from gpu_util import to_dev, to_host
    for k, v in params.items():
        pp.pp_set_param(k, v)
    try:
        pad = np.zeros(offset, dtype=a.dtype)
        buf = to_dev(np.concatenate([pad, a, pad]))
        view = buf[offset:offset + a.size]
        split = pp.pp_partition(view, pivot)
        out = to_host(view, a.dtype)
        # the padding must be untouched
        full = to_host(buf, a.dtype)
        assert np.all(full[:offset] == 0) and np.all(full[offset + a.size:] == 0)
        return split, out
    finally:
        pp.reset_params()


def _pivots(a, mx):
    ps = {0, 1, mx, mx // 2}
    if a.size:
        ps.add(int(np.sort(a)[a.size // 2]))
        ps.add(int(a[0]))
    return sorted(ps)


SMALL_NS = list(range(0, 71)) + [127, 128, 129, 511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096,
                                  4097, 8191, 8192, 8193, 10007, 32767, 32768, 32769, 65537]


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
@pytest.mark.parametrize("path", [1, 2, 3])
def test_edge_sizes(pp, dt, mx, path):
    rng = np.random.default_rng(100 + path)
    for n in SMALL_NS:
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for p in _pivots(a, mx):
            for off in (0, 1, 3):
                split, out = _run(pp, a, p, off, path=path, small_n=0,
                                  min_lines_per_group=1)
                oracle.check_partition(a, out, p, split)


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_all_patterns_small(pp, dt):
    """All 2^n predecessor/successor patterns for n <= 10, tagged keys, all paths."""
    for path in (1, 2, 3):
        for n in range(0, 11):
            for mask in range(1 << n):
                bits = np.array([(mask >> i) & 1 for i in range(n)], dtype=bool)
                idx = np.arange(n, dtype=dt)
                a = np.where(bits, idx, idx + 1000).astype(dt)
                split, out = _run(pp, a, 1000, 0, path=path, small_n=0, min_lines_per_group=1)
                oracle.check_partition(a, out, 1000, split)


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_alphabet_duplicates(pp, dt, mx):
    """Duplicate-heavy keys over a tiny alphabet, pivots spanning all cases."""
    rng = np.random.default_rng(5)
    for n in (1000, 5000, 70001, 300007):
        a = rng.integers(0, 4, size=n).astype(dt)
        for p in range(5):
            for path in (2, 3):
                split, out = _run(pp, a, p, 1, path=path, small_n=0, min_lines_per_group=2)
                oracle.check_partition(a, out, p, split)


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
@pytest.mark.parametrize("g", [1, 2, 7, 64, 0])
def test_groups_and_windows(pp, dt, mx, g):
    """Medium n, forced group counts (large windows exercise the multi-CTA
    cleanup), several offsets and pivot fractions."""
    rng = np.random.default_rng(g + 17)
    for n in (100003, 1 << 20, 3000017):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for frac in (0.0, 0.01, 0.5, 0.99, 1.0):
            p = min(mx, int(frac * (mx + 1)))
            split, out = _run(pp, a, p, 2, path=2, g=g, small_n=0)
            oracle.check_partition(a, out, p, split)


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
@pytest.mark.parametrize("chain", [0, 1])
def test_cleanup_tails(pp, dt, mx, chain):
    """The fused scan/swap cleanup tail and the 3-kernel chain give
    oracle-exact results, including large windows (forced g) and ragged n."""
    rng = np.random.default_rng(31 + chain)
    for n, g in ((1 << 20, 0), (3_000_017, 0), (3_000_017, 5), (1 << 22, 100), (777_777, 296)):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for frac in (0.0, 0.2, 0.5, 1.0):
            p = min(mx, int(frac * (mx + 1)))
            split, out = _run(pp, a, p, 1, cleanup_chain=chain, g=g)
            oracle.check_partition(a, out, p, split)
            assert pp.pp_last_stats()["path"] == 2


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_cleanup_only_large(pp, dt, mx):
    """Cleanup-only path on whole arrays: dirty set = [0, n), tiles larger
    than the one-round-trip size (exercises the general walk / select)."""
    rng = np.random.default_rng(23)
    for n in (3_000_017, 1 << 22):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for frac in (0.3, 0.5):
            p = int(frac * (mx + 1))
            split, out = _run(pp, a, p, 3, path=3)
            oracle.check_partition(a, out, p, split)
            st = pp.pp_last_stats() if False else None


def test_structured_inputs(pp):
    """Already partitioned / reverse / all-true / all-false / alternating (u32)
    and whole-line adversarial patterns (u64)."""
    n = 1_000_003
    for pat in synth.ADV_PATTERNS:
        a = synth.adversarial_u32_np(n, pat, 9)
        split, out = _run(pp, a, synth.ADV_PIVOT_U32, 1)
        oracle.check_partition(a, out, synth.ADV_PIVOT_U32, split)
    # line-granular blocks of predecessors (window stress)
    rng = np.random.default_rng(3)
    line = 1024
    nl = 3001
    blocks = rng.integers(0, 2, size=nl).astype(bool)
    a = np.where(np.repeat(blocks, line), np.uint64(5), np.uint64(1 << 40)).astype(np.uint64)
    a ^= rng.integers(0, 4, size=a.size).astype(np.uint64)
    for g in (0, 8, 1000):
        split, out = _run(pp, a, 100, 0, g=g)
        oracle.check_partition(a, out, 100, split)


def test_determinism(pp):
    n = 3_000_001
    a = synth.uniform_u64_np(n, 42)
    s1, o1 = _run(pp, a, 1 << 63, 1)
    s2, o2 = _run(pp, a, 1 << 63, 1)
    assert s1 == s2 and np.array_equal(o1, o2)


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_ss_groups_parity(pp, dt):
    """The Smoothed Striding partial partition step's per-group outputs (T_i,
    v_i) equal the oracle's, and the array is partially partitioned
     with v_min <= K <= v_max."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(8)
    mx = U64_MAX if dt == np.uint64 else U32_MAX
    for n, g, off in ((1 << 20, 0, 0), (1 << 20, 37, 1), (777777, 5, 3), (5_000_000, 0, 2)):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        p = int(np.sort(a)[n // 3])
        buf = to_dev(np.concatenate([np.zeros(off, dtype=dt), a]))
        view = buf[off:]
        T, vlo, vhi, info = pp.pp_ss_groups(view, p, g)
        h, nl, LK, gg = info["head"], info["n_lines"], info["line_keys"], info["g"]
        s = (nl + gg - 1) // gg
        X = synth.ss_offsets(info["seed"], s, gg) if info["seed"] else np.zeros(s, dtype=np.uint64)
        T2, vlo2, vhi2 = oracle.ss_groups(a, h, nl, LK, gg, X, p)
        assert np.array_equal(T, T2)
        assert np.array_equal(vlo, vlo2 - h) and np.array_equal(vhi, vhi2 - h)
        out = to_host(view, dt)
        region = out[h:h + nl * LK]
        vmin, vmax = int(vlo.min()), int(vhi.max())
        assert np.all(region[:vmin] < p) and np.all(region[vmax:] >= p)
        assert vmin <= int(T.sum()) <= vmax
        assert np.array_equal(np.sort(out), np.sort(a))


@pytest.mark.parametrize("kind", ["uniform", "whole_lines"])
def test_ss_groups_prop42_bounds(pp, kind):
    """The GPU's per-group outputs obey the paper's statements about the
    Smoothed Striding step (Prop. 4.2, 1140-1150, 1160-1166),
    on a full-chunk layout with g = 16 groups of s = 1024 lines: each group's
    first successor lies within g*b of g*T_i; every group's predecessor
    fraction is within the Hoeffding + union-bound delta of the array's
    (eps = 1e-6); the window is below 4 n delta'."""
    from gpu_util import to_dev
    rng = np.random.default_rng(1166)
    g = 16
    info0 = pp.pp_ss_groups(to_dev(np.zeros(1 << 16, dtype=np.uint64)), 1, g)[3]
    b = info0["line_keys"]
    s = 1024
    n = g * s * b
    if kind == "uniform":
        a = rng.integers(0, U64_MAX, size=n, dtype=np.uint64, endpoint=True)
        p = 1 << 63
    else:  # every line all-predecessor or all-successor: the largest per-line variance
        lines = rng.integers(0, 2, size=n // b).astype(bool)
        a = np.where(np.repeat(lines, b), np.uint64(1), np.uint64(3)).astype(np.uint64)
        p = 2
    mu = float(np.mean(a < np.uint64(p)))
    T, vlo, vhi, info = pp.pp_ss_groups(to_dev(a), p, g)
    assert info["g"] == g and info["head"] == 0 and info["n_lines"] == g * s
    eps = 1e-6
    for i in range(g):
        if int(T[i]) < s * b:
            assert abs(int(vlo[i]) - g * int(T[i])) <= g * b, (i, int(vlo[i]), int(T[i]))
    delta = np.sqrt(np.log(2 * g / eps) / (2 * s))
    mui = T.astype(np.float64) / (s * b)
    assert np.all(np.abs(mui - mu) < delta), (float(np.abs(mui - mu).max()), delta)
    assert int(vhi.max()) - int(vlo.min()) < 4 * n * np.sqrt(np.log(n / eps) / s)
    assert int(T.sum()) == oracle.count(a, p)


def test_async_and_stats(pp):
    from gpu_util import to_dev
    n = 1 << 20
    a = synth.uniform_u64_np(n, 7)
    t = to_dev(a)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    pp.pp_partition_async_u64(t, 1 << 63, d)
    torch.cuda.synchronize()
    K = oracle.count(a, 1 << 63)
    assert int(d.item()) == K
    st = pp.pp_last_stats()
    assert st["K"] == K and st["n"] == n
    assert st["aux_bytes"] < 0.01 * n * 8


@pytest.mark.parametrize("chunk", [0, 4096, 5000, 1 << 16])
def test_host_variant(pp, chunk):
    """Host-buffer partition (streamed chunks, uploads from both ends,
    predecessors written to the front / successors to the back): the host
    result passes the oracle checks for ragged chunk counts, pivot extremes
    and pinned as well as pageable memory."""
    if chunk:
        pp.pp_set_param("host_chunk", chunk)
    try:
        for dt in (np.uint64, np.uint32):
            mx = U64_MAX if dt == np.uint64 else U32_MAX
            for n in (1, 7, 4095, 4097, 200003, 1 << 20):
                a = (synth.uniform_u64_np(n, 11) if dt == np.uint64 else synth.uniform_u32_np(n, 11))
                f = pp.pp_partition_host_u64 if dt == np.uint64 else pp.pp_partition_host_u32
                for p in (0, mx // 100, mx // 2, mx - mx // 100, mx):
                    b = a.copy()
                    split = f(b, p)
                    oracle.check_partition(a, b, p, split)
            # pinned host memory
            a = synth.uniform_u64_np(300007, 12)
            pin = torch.empty(a.size, dtype=torch.int64, pin_memory=True)
            pv = pin.numpy().view(np.uint64)
            np.copyto(pv, a)
            split = pp.pp_partition_host_u64(pv, 1 << 63)
            oracle.check_partition(a, pv, 1 << 63, split)
    finally:
        pp.reset_params()


def test_invalid_args(pp):
    import ctypes
    L = pp.load()
    out = ctypes.c_uint64(0)
    # misaligned device pointer
    t = torch.zeros(16, dtype=torch.int64, device="cuda")
    assert L.pp_partition_u64(t.data_ptr() + 4, 8, 5, None, ctypes.byref(out)) == 1
    # host pointer passed as device pointer
    h = np.zeros(16, dtype=np.uint64)
    assert L.pp_partition_u64(h.ctypes.data, 16, 5, None, ctypes.byref(out)) == 1
    # empty
    assert L.pp_partition_u64(None, 0, 5, None, ctypes.byref(out)) == 0 and out.value == 0


def test_caller_workspace(pp):
    """pp_set_workspace: a caller-owned buffer of
    pp_workspace_bytes(n, ., op) suffices for partition and quicksort; a too
    small one fails with PP_E_NOMEM and leaves a partition's array untouched."""
    from gpu_util import to_dev
    try:
        for n, dt in ((3_000_017, np.uint64), (5_000_011, np.uint32), (1 << 15, np.uint64)):
            a = synth.uniform_u64_np(n, 41) if dt == np.uint64 else synth.uniform_u32_np(n, 41)
            kb = a.itemsize
            p = (1 << 63) if dt == np.uint64 else (1 << 31)
            wb = pp.pp_workspace_bytes(n, kb, 0)
            assert 0 < wb < 0.05 * n * kb + (1 << 20)
            ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
            pp.pp_set_workspace(ws)
            t = to_dev(a)
            K = pp.pp_partition(t, p)
            oracle.check_partition(a, t.cpu().numpy().view(dt), p, K)
            assert pp.pp_last_aux_bytes() <= wb
            # quicksort: op 1 bound
            wq = pp.pp_workspace_bytes(n, kb, 1)
            assert wq >= wb
            wsq = torch.empty(wq, dtype=torch.uint8, device="cuda")
            pp.pp_set_workspace(wsq)
            t = to_dev(a)
            pp.pp_quicksort(t)
            assert np.array_equal(t.cpu().numpy().view(dt), np.sort(a))
            # too small: NOMEM, array untouched for a partition
            tiny = torch.empty(256, dtype=torch.uint8, device="cuda")
            pp.pp_set_workspace(tiny)
            t = to_dev(a)
            with pytest.raises(pp.PPError):
                pp.pp_partition(t, p)
            assert np.array_equal(t.cpu().numpy().view(dt), a)
            pp.pp_set_workspace(None)
        import ctypes
        h = np.zeros(4096, dtype=np.uint8)
        addr = (h.ctypes.data + 255) & ~255  # host memory is rejected
        assert pp.load().pp_set_workspace(ctypes.c_void_p(addr), 1024) == 1
    finally:
        pp.pp_set_workspace(None)


# ----------------------------------------------------------------------------
# BASELINE configs at full size (checks via oracle count + device properties)
# ----------------------------------------------------------------------------

def _full_check(pp, t, pivot, K_oracle):
    from gpu_util import check_partition_device
    inp = t.clone()
    split = pp.pp_partition(t, pivot)
    check_partition_device(inp, t, pivot, split, K_oracle)
    return split


def test_config1_exact(pp):
    from gpu_util import to_dev
    n = 1 << 20
    a = synth.uniform_u64_np(n, synth.SEEDS["c1"])
    t = to_dev(a)
    split = pp.pp_partition(t, 1 << 63)
    oracle.check_partition(a, t.cpu().numpy().view(np.uint64), 1 << 63, split)


@pytest.mark.parametrize("mu", [0.01, 0.5, 0.99])
def test_config2_full(pp, mu):
    n = 1 << 27
    p = synth.PIVOT_MU[mu]
    t = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
    host = t.cpu().numpy().view(np.uint64)
    K = oracle.count(host, p)
    _full_check(pp, t, p, K)
    st = pp.pp_last_stats()
    assert st["path"] in (2, 4) and st["W"] < 0.05 * n
    assert st["aux_bytes"] < 0.001 * n * 8


@functools.lru_cache(maxsize=None)
def _oracle_count_c3(n: int, p: int, chunk: int = 1 << 27) -> int:
    """K = #keys < p over the seed-regenerated c3 input, computed by the
    oracle chunk by chunk on the host (threads: numpy and the ctypes oracle
    release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    def one(s):
        return oracle.count(synth.uniform_u64_np(min(chunk, n - s), synth.SEEDS["c3"], offset=s), p)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        return sum(ex.map(one, range(0, n, chunk)))


def test_config3_single_gpu_full(pp):
    """n = 2^33 u64 (64 GiB, BASELINE config 3 at P = 1), pivot 2^63, exact:
    (1) split == the oracle's count over the whole seed-regenerated input
    (host, chunkwise); (2) the predicate on every position (device);
    (3) exact multiset equality by value-range bucketing: the
    key space is cut into 64 equal ranges, and for each range the output's
    keys and the regenerated input's keys in it are gathered and sorted with
    the library sort and compared element by element.  Given (1) and (2),
    whole-array multiset equality is equivalent to the per-side check (3)."""
    n = 1 << 33
    p = 1 << 63
    t = torch.empty(n, dtype=torch.int64, device="cuda")
    synth.uniform_u64_torch(n, synth.SEEDS["c3"], "cuda", out=t, chunk=1 << 27)
    split = pp.pp_partition(t, p)
    _check_c3_exact(t, n, p, split)


@pytest.mark.parametrize("P", [2, 8])
def test_config3_loopback_ranks_full(pp, P):
    """BASELINE config 3 at P = 2 and 8: the same 2^33 keys as P contiguous
    shards of 2^33 / P (key i depends only on the global index i), partitioned
    by the distributed code (local partitions, all-gather of the counts, the
    planned exchange of misplaced ranges) with P emulated ranks on this GPU
    (loopback transport), checked exactly like the single-GPU run: the GLOBAL
    array is the partition of P:272-281."""
    n = 1 << 33
    p = 1 << 63
    t = torch.empty(n, dtype=torch.int64, device="cuda")
    synth.uniform_u64_torch(n, synth.SEEDS["c3"], "cuda", out=t, chunk=1 << 27)
    split = pp.pp_partition_dist_loopback(t, [n // P] * P, p)
    _check_c3_exact(t, n, p, split)


def _check_c3_exact(t, n, p, split):
    from gpu_util import order_key, order_pivot
    K_oracle = _oracle_count_c3(n, p)
    assert split == K_oracle
    pv = order_pivot(p, torch.int64)
    C = 1 << 28
    for s in range(0, n, C):
        ko = order_key(t[s:s + C])
        idx = torch.arange(s, s + ko.numel(), device="cuda")
        assert bool(((ko < pv) == (idx < split)).all())
    del ko, idx
    B = 64  # ranges of 2^58 keys: the top 6 bits of the unsigned key
    Ci = 1 << 27
    chunk_in = torch.empty(Ci, dtype=torch.int64, device="cuda")
    for b in range(B):
        outs, ins = [], []
        for s in range(0, n, C):
            x = t[s:s + C]
            outs.append(x[((x >> 58) & 63) == b])
        for s in range(0, n, Ci):
            m = min(Ci, n - s)
            synth.uniform_u64_torch(m, synth.SEEDS["c3"], "cuda", offset=s, out=chunk_in[:m], chunk=Ci)
            x = chunk_in[:m]
            ins.append(x[((x >> 58) & 63) == b])
        o = torch.sort(order_key(torch.cat(outs))).values
        del outs
        i = torch.sort(order_key(torch.cat(ins))).values
        del ins
        assert o.numel() == i.numel() and torch.equal(o, i), f"multiset differs in key range {b}"
        del o, i
    torch.cuda.empty_cache()


def test_config4_zipf_full(pp):
    """BASELINE config 4 Zipf case: n = 1,000,000,007 u32 keys, Zipf(1.1)
    ranks - 1 on [0, 2^32) (duplicate-heavy: ~10.5% of keys are 0), pivot =
    the sample median (SURVEY §8(c) reading 17).  Split against the oracle's
    count on the host; predicate and per-side multisets on the device."""
    from gpu_util import check_partition_device
    n = 1_000_000_007
    t = synth.zipf_u32_torch(n, 1.1, synth.SEEDS["c4"], "cuda")
    wide = t.to(torch.int64) & 0xFFFFFFFF
    pivot = int(torch.sort(wide).values[n // 2])  # sample median (library sort)
    del wide
    K = oracle.count(t.cpu().numpy().view(np.uint32), pivot)
    inp = t.clone()
    split = pp.pp_partition(t, pivot)
    check_partition_device(inp, t, pivot, split, K)


@pytest.mark.parametrize("pat", list(synth.ADV_PATTERNS))
def test_config4_adversarial_full(pp, pat):
    n = 1_000_000_007
    t = synth.adversarial_u32_torch(n, pat, synth.SEEDS["c4"], "cuda")
    K = {"partitioned": n // 2, "reverse": n // 2, "all_true": n, "all_false": 0,
         "alternating": (n + 1) // 2}[pat]
    # the closed-form K is pinned against the oracle count on a prefix sample
    host_prefix = t[:1_000_003].cpu().numpy().view(np.uint32)
    Kp = oracle.count(host_prefix, synth.ADV_PIVOT_U32)
    exp_p = {"partitioned": 1_000_003, "reverse": 0, "all_true": 1_000_003, "all_false": 0,
             "alternating": 500_002}[pat]
    assert Kp == exp_p
    _full_check(pp, t, synth.ADV_PIVOT_U32, K)


def test_group_kernel_dirty_smem(pp):
    """The group kernel right after other kernels (dirty shared memory), both
    key widths and instantiations (default, Strided)."""
    rng = np.random.default_rng(7)
    for strided in (0, 1):
        for dt, mx in ((np.uint64, U64_MAX), (np.uint32, U32_MAX)):
            for n in (3_000_017, 1 << 22):
                a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
                for frac in (0.01, 0.5):
                    p = int(frac * (mx + 1))
                    split, out = _run(pp, a, p, 1, strided=strided)
                    oracle.check_partition(a, out, p, split)


@pytest.mark.parametrize("strided", [0, 1])
def test_strided_ablation(pp, strided):
    """the Strided Algorithm (X = 0) and
    Smoothed Striding on uniform keys and on the stride-aligned adversary
    (stride = the library's group count): both give a correct partition; on
    the adversary the Strided window covers most of the array while the
    smoothed one stays small."""
    n = 1 << 24
    a = synth.uniform_u64_np(n, 21)
    # g = 32 groups of 512 chunks each (the smoothing averages over chunks)
    s, out = _run(pp, a, 1 << 63, 0, strided=strided, g=32)
    oracle.check_partition(a, out, 1 << 63, s)
    pp.pp_set_param("strided", strided)
    pp.pp_set_param("g", 32)
    try:
        from gpu_util import to_dev, to_host
        t = to_dev(a)
        pp.pp_partition(t, 1 << 63)
        st = pp.pp_last_stats()
        g, lk = st["g"], st["line_keys"]
        assert g == 32
        adv = synth.stride_aligned_u64_np(n, 22, lk, g)
        t = to_dev(adv)
        s = pp.pp_partition(t, 1 << 63)
        w = pp.pp_last_stats()["W"] / n
        oracle.check_partition(adv, to_host(t, np.uint64), 1 << 63, s)
    finally:
        pp.reset_params()
    if strided:
        assert w > 0.9, w
    else:
        assert w < 0.15, w


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_standard_algorithm_bytewise(pp, dt):
    """the GPU Standard Algorithm (stable, out of place,
    PAPER.md:284-311) equals the oracle's Standard Algorithm byte for byte
    (stability makes the output unique); edge sizes around the 4096-key tile,
    duplicates, pivot extremes; the input is left untouched."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(31)
    mx = U64_MAX if dt == np.uint64 else U32_MAX
    sizes = [0, 1, 2, 31, 32, 33, 4095, 4096, 4097, 8191, 12289, 100003, 1 << 20]
    for n in sizes:
        for a in (rng.integers(0, mx, size=n, dtype=dt, endpoint=True), rng.integers(0, 5, size=n).astype(dt)):
            for p in sorted({0, 1, 2, mx // 3, mx}):
                ref = a.copy()
                k_ref = oracle.partition_standard(ref, p)
                t_in = to_dev(a)
                t_out = torch.zeros_like(t_in)
                k = pp.pp_partition_stable(t_in, t_out, p)
                assert k == k_ref, (n, p)
                assert np.array_equal(to_host(t_out, dt), ref), (n, p)
                assert np.array_equal(to_host(t_in, dt), a)


def test_standard_algorithm_config2(pp):
    """Config 2 size (2^27 u64, three pivots): byte-exact against the oracle's
    Standard Algorithm, async variant (split to device memory)."""
    from gpu_util import to_host
    n = 1 << 27
    a = synth.uniform_u64_np(n, synth.SEEDS["c2"])
    t_in = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
    t_out = torch.empty_like(t_in)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for mu, p in synth.PIVOT_MU.items():
        pp.pp_partition_stable_async_u64(t_in, t_out, p, d)
        ref = a.copy()
        k_ref = oracle.partition_standard(ref, p)
        assert int(d.item()) == k_ref
        assert np.array_equal(to_host(t_out, np.uint64), ref), mu


def test_standard_algorithm_rejects_overlap(pp):
    import ctypes
    L = pp.load()
    t = torch.zeros(64, dtype=torch.int64, device="cuda")
    out = ctypes.c_uint64(0)
    assert L.pp_partition_stable_u64(t.data_ptr(), t.data_ptr() + 8 * 8, 32, 5, None, ctypes.byref(out)) == 1


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_bps_bytewise(pp, dt):
    """the GPU Blocked-Prefix-Sum partition (low-space form,
    PAPER.md:319-478, 1466-1486) equals the CPU oracle's byte for byte (the
    algorithm is deterministic): sizes around the 4096-key block and the
    one-CTA MakeSuccessorHeavy threshold, both sides of the role swap,
    duplicates, pivot extremes, unaligned bases."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(41)
    mx = U64_MAX if dt == np.uint64 else U32_MAX
    for n in (0, 1, 2, 3, 100, 4095, 4096, 4097, 8191, 20480, 20481, 40000, 100003, 1 << 20, 3_000_017):
        for a in (rng.integers(0, mx, size=n, dtype=dt, endpoint=True), rng.integers(0, 4, size=n).astype(dt)):
            for p in sorted({0, 1, 2, mx // 100, mx // 2, mx - mx // 100, mx}):
                ref = a.copy()
                k_ref = oracle.partition_bps(ref, p, 4096)
                t = to_dev(a)
                k = pp.pp_partition_bps(t, p)
                assert k == k_ref, (n, p)
                assert np.array_equal(to_host(t, dt), ref), (n, p)


def test_bps_golden_make_successor_heavy(pp, golden):
    """The SPEC.md:344 MakeSuccessorHeavy example (Fig. 1)
    through the GPU Blocked-Prefix-Sum partition: byte for byte equal to the
    oracle's BPS, whose MakeSuccessorHeavy stage the golden value pins."""
    from gpu_util import to_dev, to_host
    for ex in golden["make_successor_heavy"]:
        for dt in (np.uint64, np.uint32):
            a = np.array(ex["keys"], dtype=dt)
            msh = a.copy()
            oracle.bps_make_successor_heavy(msh, ex["pivot"], False)
            assert msh.tolist() == ex["output"]
            ref = a.copy()
            k_ref = oracle.partition_bps(ref, ex["pivot"], 4096)
            t = to_dev(a)
            assert pp.pp_partition_bps(t, ex["pivot"]) == k_ref
            assert np.array_equal(to_host(t, dt), ref), ex["cite"]


def test_bps_config2(pp):
    """Config 2 (2^27 u64, the three pivots), async variant: byte for byte
    against the oracle."""
    from gpu_util import to_host
    n = 1 << 27
    a = synth.uniform_u64_np(n, synth.SEEDS["c2"])
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for mu, p in synth.PIVOT_MU.items():
        t = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
        pp.pp_partition_bps_async_u64(t, p, d)
        ref = a.copy()
        k_ref = oracle.partition_bps(ref, p, 4096)
        assert int(d.item()) == k_ref
        assert np.array_equal(to_host(t, np.uint64), ref), mu


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_stable_inplace_bytewise(pp, dt):
    """The in-place stable partition (tile partitions + rotation merges)
    equals the oracle's Standard Algorithm byte for byte (the stable result is
    unique): sizes around the 4096-key tile and odd segment
    counts at every level, pivot extremes, duplicates, unaligned bases."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(73 + (dt == np.uint64))
    mx = U64_MAX if dt == np.uint64 else U32_MAX
    for n in (0, 1, 2, 31, 4095, 4096, 4097, 8192, 12289, 3 * 4096 + 5, 100_003, (1 << 20) + 7, 3_000_017):
        for a in (rng.integers(0, mx, size=n, dtype=dt, endpoint=True), rng.integers(0, 5, size=n).astype(dt)):
            for p in sorted({0, 1, 3, mx // 3, mx // 2, mx}):
                ref = a.copy()
                k_ref = oracle.partition_standard(ref, p)
                for off in (0, 1):
                    buf = to_dev(np.concatenate([np.zeros(off, dt), a]))
                    t = buf[off:]
                    k = pp.pp_partition_stable_inplace(t, p)
                    assert k == k_ref, (n, p)
                    assert np.array_equal(to_host(t, dt), ref), (n, p, off)


def test_stable_inplace_config2(pp):
    """Config 2 (2^27 u64, mu = 0.5): byte for byte against the oracle."""
    from gpu_util import to_host
    n = 1 << 27
    a = synth.uniform_u64_np(n, synth.SEEDS["c2"])
    t = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
    k = pp.pp_partition_stable_inplace(t, 1 << 63)
    ref = a.copy()
    assert k == oracle.partition_standard(ref, 1 << 63)
    assert np.array_equal(to_host(t, np.uint64), ref)
