"""GPU: the C-ABI multi-GPU partition and quicksort (pp_dist_*).

* The product code path at P > 1 on one GPU: the loopback transport runs P
  emulated ranks (host threads, disjoint slices of one device array) through
  the SAME plan -> rounds -> staging -> place code and the one-sided share
  rule as the NCCL path (pp_*_dist_loopback_*), checked against the oracle.
* The NCCL transport itself on a single-rank communicator (one GPU)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2004_12532_b200 as m
    m.load()
    m.reset_params()
    uid = m.pp_dist_unique_id()
    m.pp_dist_init(uid, 1, 0, torch.cuda.current_device())
    yield m
    m.pp_dist_finalize()


def test_dist_single_rank(pp):
    from gpu_util import to_dev
    for dt, n, p in ((np.uint64, 1 << 20, 1 << 63), (np.uint64, 3_000_017, 1 << 61),
                     (np.uint32, 2_000_003, 1 << 31), (np.uint64, 0, 5)):
        a = (synth.uniform_u64_np(n, 77) if dt == np.uint64 else synth.uniform_u32_np(n, 77))
        t = to_dev(a) if n else torch.empty(0, dtype=torch.int64, device="cuda")
        K = pp.pp_partition_dist(t, p)
        out = t.cpu().numpy().view(dt)
        oracle.check_partition(a, out, p, K)


def test_quicksort_dist_single_rank(pp):
    from gpu_util import to_dev
    rng = np.random.default_rng(3)
    for a in (synth.uniform_u64_np(1_000_003, 5), rng.integers(0, 9, size=200_001).astype(np.uint64),
              synth.uniform_u32_np(300_007, 6)):
        t = to_dev(a)
        pp.pp_quicksort_dist(t)
        ref = a.copy()
        oracle.quicksort(ref)
        assert np.array_equal(t.cpu().numpy().view(a.dtype), ref)


def test_dist_finalize_and_reinit(pp):
    pp.pp_dist_finalize()
    uid = pp.pp_dist_unique_id()
    pp.pp_dist_init(uid, 1, 0, torch.cuda.current_device())
    with pytest.raises(pp.PPError):
        pp.pp_dist_init(uid, 1, 0, torch.cuda.current_device())  # already initialised


@pytest.mark.parametrize("P,dt", [(2, np.uint64), (3, np.uint64), (4, np.uint32), (8, np.uint64)])
def test_emulated_ranks_staging_free_exchange(pp, P, dt):
    """SURVEY §8(f) #1 core, emulated on one GPU (the profiling guide's advice
    for multi-rank logic with fewer GPUs than ranks): P "ranks" are
    contiguous, uneven shards of one device array; each partitions its shard
    with the library, the exchange plan pairs the misplaced ranges
    (pp_dist_plan, the same host arithmetic as the NCCL path), and the
    staging-free primitive pp_swap_ranges swaps each piece one-sidedly.  The
    whole array must then be a partition (oracle checks) with K = sum t_r."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(P * 7 + (dt == np.uint64))
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    w = np.dtype(dt).itemsize
    for total in (1000, 300_007, 1 << 22):
        cuts = np.sort(rng.integers(0, total, size=P - 1))
        ns = np.diff(np.concatenate([[0], cuts, [total]])).astype(np.uint64)
        a = rng.integers(0, mx, size=total, dtype=dt, endpoint=True)
        for p in (int(mx // 3), int(mx // 2), int(mx - mx // 10), 0):
            t = to_dev(a)
            ts, base = [], 0
            for r in range(P):
                view = t[base:base + int(ns[r])]
                ts.append(pp.pp_partition(view, p) if ns[r] else 0)
                base += int(ns[r])
            K, rows = pp.pp_dist_plan(ns, ts, 1 << 40)
            assert K == sum(ts)
            ptr = t.data_ptr()
            pieces = [(ptr + w * f, ptr + w * tt, ln) for (_, rf, f, rt, tt, ln) in rows]
            if pieces:
                pp.pp_swap_ranges(pieces, w)
            oracle.check_partition(a, to_host(t, dt), p, K)


@pytest.mark.parametrize("P,dt", [(2, np.uint64), (5, np.uint32), (8, np.uint64)])
def test_emulated_ranks_p2p_shares(pp, P, dt):
    """The one-sided exchange as pp_partition_dist runs it with dist_p2p=1,
    emulated on one GPU: every emulated rank executes only ITS share
    (pp_dist_p2p_pieces: half of each matched run, addresses of its own shard
    and of the partner's) with pp_swap_ranges, ranks one after another; the
    union of the shares partitions the whole array."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(P * 11 + (dt == np.uint64))
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    w = np.dtype(dt).itemsize
    for total in (999, 500_001, 1 << 21):
        cuts = np.sort(rng.integers(0, total, size=P - 1))
        ns = [int(x) for x in np.diff(np.concatenate([[0], cuts, [total]]))]
        a = rng.integers(0, mx, size=total, dtype=dt, endpoint=True)
        for p in (int(mx // 2), int(mx // 7), int(mx - mx // 5)):
            t = to_dev(a)
            ts, base = [], 0
            for r in range(P):
                ts.append(pp.pp_partition(t[base:base + ns[r]], p) if ns[r] else 0)
                base += ns[r]
            ptr = t.data_ptr()
            for r in rng.permutation(P):
                rows = pp.pp_dist_p2p_pieces(ns, ts, int(r))
                if rows:
                    pp.pp_swap_ranges([(ptr + w * ga, ptr + w * gb, ln) for (_, ga, _, gb, ln) in rows], w)
            oracle.check_partition(a, to_host(t, dt), p, sum(ts))


_IPC_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2004_12532_b200 as pp
pp.load(build_if_missing=False)
handle, off, n = bytes.fromhex(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
remote = pp.pp_ipc_import(handle, off)
assert pp.pp_ipc_import(handle, off) == remote  # cached mapping
mine = torch.arange(n, dtype=torch.int64, device="cuda") + 1_000_000
# swap the parent's [n/4, n/4 + n/2) with my [0, n/2), half the range per piece
h = n // 2
pieces = [(remote + 8 * (n // 4), mine.data_ptr(), h // 2),
          (remote + 8 * (n // 4 + h // 2), mine.data_ptr() + 8 * (h // 2), h - h // 2)]
pp.pp_swap_ranges(pieces, 8)
torch.cuda.synchronize()
got = mine[:h].cpu().numpy()
assert np.array_equal(got, np.arange(n // 4, n // 4 + h) * 3), got[:4]
pp.pp_ipc_close_all()
print("child ok")
"""


def test_ipc_export_import_two_processes(pp, tmp_path):
    """CUDA IPC path of the one-sided exchange on one GPU with two processes
    (no kernel waits on another): the parent exports a range inside a larger
    allocation (handle + offset), a child process maps it, swaps half of it
    with its own buffer through pp_swap_ranges, and both sides see the
    exchanged keys."""
    import os
    import subprocess
    import sys
    n = 1 << 20
    big = torch.zeros(n + 4096, dtype=torch.int64, device="cuda")
    t = big[1000:1000 + n]  # an interior range: the offset matters
    t.copy_(torch.arange(n, dtype=torch.int64, device="cuda") * 3)
    torch.cuda.synchronize()
    handle, off = pp.pp_ipc_export(t)
    assert len(handle) == 64 and off >= 8000 and off % 8 == 0  # allocation base <= big's start
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "ipc_child.py"
    script.write_text(_IPC_CHILD)
    r = subprocess.run([sys.executable, str(script), root, handle.hex(), str(off), str(n)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "child ok" in r.stdout, r.stderr[-2000:]
    out = t.cpu().numpy()
    h = n // 2
    assert np.array_equal(out[n // 4:n // 4 + h], np.arange(h) + 1_000_000)
    assert np.array_equal(out[:n // 4], np.arange(n // 4) * 3)
    assert np.array_equal(out[n // 4 + h:], np.arange(n // 4 + h, n) * 3)
    assert int(big[:1000].abs().sum()) == 0 and int(big[1000 + n:].abs().sum()) == 0


def test_partition_dist_p2p_param_single_rank(pp):
    """dist_p2p=1 on a one-rank communicator: the local partition alone (no
    peers to map); the parameter round-trips and resets."""
    from gpu_util import to_dev, to_host
    a = synth.uniform_u64_np(1 << 18, 5)
    pp.pp_set_param("dist_p2p", 1)
    try:
        assert pp.pp_get_param("dist_p2p") == 1
        t = to_dev(a)
        K = pp.pp_partition_dist(t, 1 << 63)
        oracle.check_partition(a, to_host(t, np.uint64), 1 << 63, K)
    finally:
        pp.reset_params()
    assert pp.pp_get_param("dist_p2p") == 0


def test_dist_last_timing_single_rank(pp):
    """pp_dist_last_timing after a one-rank pp_partition_dist: the three
    phase times are set (non-negative, local partition > 0) and no bytes
    moved between GPUs."""
    from gpu_util import to_dev
    a = synth.uniform_u64_np(1 << 20, 17)
    t = to_dev(a)
    pp.pp_partition_dist(t, 1 << 63)
    tm = pp.pp_dist_last_timing()
    assert tm["local_ms"] > 0 and tm["gather_ms"] >= 0 and tm["exchange_ms"] >= 0
    assert tm["bytes"] == 0


# ---------------------------------------------------------------------------
# P > 1 through the product code (loopback transport)
# ---------------------------------------------------------------------------
def _shards(rng, total, P, kind):
    """Shard sizes summing to total: ragged, with empty shards (kind 'empty'),
    or equal."""
    if kind == "equal":
        ns = [total // P] * P
        ns[-1] += total - sum(ns)
        return ns
    cuts = np.sort(rng.integers(0, total + 1, size=P - 1))
    ns = [int(x) for x in np.diff(np.concatenate([[0], cuts, [total]]))]
    if kind == "empty" and P > 2:
        ns[1] += ns[0]
        ns[0] = 0  # an empty first shard
        ns[-2] += ns[-1]
        ns[-1] = 0  # and an empty last one
    return ns


def _keys(rng, total, dt, dist_kind):
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    if dist_kind == "uniform":
        return rng.integers(0, mx, size=total, dtype=dt, endpoint=True)
    if dist_kind == "dup":
        return rng.integers(0, 1000, size=total).astype(dt)
    if dist_kind == "equal":
        return np.full(total, 12345, dtype=dt)
    if dist_kind == "max":
        return np.full(total, mx, dtype=dt)
    raise ValueError(dist_kind)


@pytest.mark.parametrize("P", [2, 3, 5, 8])
@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
@pytest.mark.parametrize("p2p", [0, 1])
def test_loopback_partition(pp, P, dt, p2p):
    """Global partition of P contiguous shards (ragged, empty, equal) by the
    product exchange: oracle checks (1)-(3) on the whole array, K = oracle
    count; pivots 0, MAX, mid and skewed; staging caps 4 KiB .. 256 MiB (the
    staged path runs hundreds of rounds at 4 KiB)."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(1000 * P + 10 * (dt == np.uint64) + p2p)
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    pp.pp_set_param("dist_p2p", p2p)
    try:
        for total, kind, cap in ((1, "ragged", 1 << 12), (977, "empty", 1 << 12), (300_007, "ragged", 1 << 12),
                                 (1_000_003, "empty", 1 << 16), (1 << 22, "equal", 256 << 20)):
            ns = _shards(rng, total, P, kind)
            a = _keys(rng, total, dt, "uniform")
            pp.pp_dist_set_staging(cap)
            for pivot in (0, mx, (mx + 1) // 2, int(mx // 100), int(rng.integers(0, mx, dtype=dt))):
                t = to_dev(a)
                K = pp.pp_partition_dist_loopback(t, ns, pivot)
                assert K == oracle.count(a, pivot)
                oracle.check_partition(a, to_host(t, dt), pivot, K)
    finally:
        pp.pp_dist_set_staging(256 << 20)
        pp.reset_params()


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
@pytest.mark.parametrize("p2p", [0, 1])
def test_loopback_partition_overlap(pp, P, dt, p2p):
    """The count-first overlapped exchange (dist_overlap = 1, SURVEY §8(f)
    #1) through the product code: per-chunk counts, one record all-gather,
    chunk-unit plan, every chunk's partition enqueued up front, the exchange
    of step k after chunk k (staged rounds or one-sided swaps, local swaps on
    the rank holding K); K = the oracle count and the oracle's checks on the
    whole array, for 1, 3 and 8 chunks per shard, ragged / empty shards,
    pivots 0, MAX, mid, skewed and random, staging caps 4 KiB and 64 KiB."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(5000 * P + 10 * (dt == np.uint64) + p2p)
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    pp.pp_set_param("dist_p2p", p2p)
    pp.pp_set_param("dist_overlap", 1)
    try:
        for C in (1, 3, 8):
            pp.pp_set_param("dist_chunks", C)
            for total, kind, cap in ((1, "ragged", 1 << 12), (977, "empty", 1 << 12), (300_007, "ragged", 1 << 12),
                                     (1_000_003, "empty", 1 << 16)):
                ns = _shards(rng, total, P, kind) if P > 1 else [total]
                a = _keys(rng, total, dt, "uniform")
                pp.pp_dist_set_staging(cap)
                for pivot in (0, mx, (mx + 1) // 2, int(mx // 100), int(rng.integers(0, mx, dtype=dt))):
                    t = to_dev(a)
                    K = pp.pp_partition_dist_loopback(t, ns, pivot)
                    assert K == oracle.count(a, pivot), (C, total, pivot)
                    oracle.check_partition(a, to_host(t, dt), pivot, K)
    finally:
        pp.pp_dist_set_staging(256 << 20)
        pp.reset_params()


def test_dist_overlap_single_rank(pp):
    """dist_overlap through the NCCL transport on a one-rank communicator
    (count pass, record all-gather, chunked local partitions; the rank's
    chunks exchange among themselves by local swaps) and its timing record."""
    from gpu_util import to_dev
    pp.pp_set_param("dist_overlap", 1)
    try:
        for dt, n, p, C in ((np.uint64, 1 << 20, 1 << 63, 8), (np.uint64, 3_000_017, 1 << 61, 5),
                            (np.uint32, 2_000_003, 1 << 31, 3), (np.uint64, 0, 5, 8)):
            pp.pp_set_param("dist_chunks", C)
            a = (synth.uniform_u64_np(n, 78) if dt == np.uint64 else synth.uniform_u32_np(n, 78))
            t = to_dev(a) if n else torch.empty(0, dtype=torch.int64, device="cuda")
            K = pp.pp_partition_dist(t, p)
            oracle.check_partition(a, t.cpu().numpy().view(dt), p, K)
            tm = pp.pp_dist_last_timing()
            assert tm["local_ms"] >= 0 and tm["exchange_ms"] >= 0 and tm["bytes"] == 0
    finally:
        pp.reset_params()


def test_loopback_partition_deterministic(pp):
    """Two runs of the loopback exchange give identical bytes (EREW
    determinism): the plan and the pieces are a pure function
    of the input."""
    from gpu_util import to_dev
    a = synth.uniform_u64_np(2_000_003, 91)
    ns = [300_000, 0, 700_000, 1_000_003]
    outs = []
    for _ in range(2):
        t = to_dev(a)
        pp.pp_dist_set_staging(1 << 16)
        pp.pp_partition_dist_loopback(t, ns, 1 << 63)
        outs.append(t.cpu().numpy())
    pp.pp_dist_set_staging(256 << 20)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("P", [2, 3, 5, 8])
@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_loopback_quicksort(pp, P, dt):
    """Distributed quicksort through the product code (batched pivot gather,
    batched partition of the spanning segments, gather-sort of small spanning
    segments, local sorts), byte for byte against oracle.quicksort; small
    dist_small forces several distributed levels, the default takes the
    gather-sort path."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(77 * P + (dt == np.uint64))
    try:
        for total, kind, dk, small in ((2, "ragged", "uniform", 1 << 16), (1000, "empty", "uniform", 1 << 16),
                                       (200_003, "ragged", "uniform", 1000), (300_001, "empty", "dup", 1000),
                                       (100_000, "equal", "equal", 1000), (50_001, "ragged", "max", 1000),
                                       (1 << 20, "equal", "uniform", 1 << 16)):
            pp.pp_set_param("dist_small", small)
            ns = _shards(rng, total, P, kind)
            a = _keys(rng, total, dt, dk)
            t = to_dev(a)
            pp.pp_quicksort_dist_loopback(t, ns)
            ref = a.copy()
            oracle.quicksort(ref)
            assert np.array_equal(to_host(t, dt), ref), (total, kind, dk, small)
    finally:
        pp.reset_params()


@pytest.mark.parametrize("P", [2, 3, 8])
def test_loopback_quicksort_boundary_split(pp, P):
    """dist_split = 1 (pivots of spanning segments at the sample quantile of
    their rank boundary): the same global sort, byte for byte against
    oracle.quicksort, on ragged / empty / equal shards and duplicate keys."""
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(91 * P)
    try:
        pp.pp_set_param("dist_split", 1)
        for total, kind, dk, small in ((200_003, "ragged", "uniform", 1000), (300_001, "empty", "dup", 1000),
                                       (100_000, "equal", "equal", 1000), (1 << 20, "ragged", "uniform", 1 << 16),
                                       (1 << 20, "equal", "dup", 1 << 12)):
            pp.pp_set_param("dist_small", small)
            ns = _shards(rng, total, P, kind)
            a = _keys(rng, total, np.uint64, dk)
            t = to_dev(a)
            pp.pp_quicksort_dist_loopback(t, ns)
            ref = a.copy()
            oracle.quicksort(ref)
            assert np.array_equal(to_host(t, np.uint64), ref), (total, kind, dk, small)
    finally:
        pp.reset_params()


def test_loopback_quicksort_p2p(pp):
    """The distributed quicksort with the one-sided exchange."""
    from gpu_util import to_dev, to_host
    a = synth.uniform_u64_np(400_009, 5)
    ns = [100_000, 0, 150_000, 150_009]
    pp.pp_set_param("dist_p2p", 1)
    pp.pp_set_param("dist_small", 2000)
    try:
        t = to_dev(a)
        pp.pp_quicksort_dist_loopback(t, ns)
    finally:
        pp.reset_params()
    ref = a.copy()
    oracle.quicksort(ref)
    assert np.array_equal(to_host(t, np.uint64), ref)


@pytest.mark.parametrize("fault", [1, 2])
@pytest.mark.parametrize("rank", [0, 2])
def test_loopback_failure_agreement(pp, fault, rank):
    """A rank that fails its local step (fault 1) is reported by EVERY rank
    (status agreement; no hang); a rank that never arrives (fault 2) makes
    the others time out (dist_timeout_ms) instead of hanging.  The array stays
    a permutation of the input."""
    import time
    from gpu_util import to_dev, to_host
    a = synth.uniform_u64_np(500_000, 8)
    ns = [100_000, 150_000, 200_000, 50_000]
    pp.pp_set_param("dist_fault", fault)
    pp.pp_set_param("dist_fault_rank", rank)
    pp.pp_set_param("dist_timeout_ms", 3000)
    try:
        for call in ("partition", "quicksort"):
            t = to_dev(a)
            t0 = time.time()
            with pytest.raises(pp.PPError) as ei:
                if call == "partition":
                    pp.pp_partition_dist_loopback(t, ns, 1 << 63)
                else:
                    pp.pp_quicksort_dist_loopback(t, ns)
            assert time.time() - t0 < 60
            assert ei.value.status in (4, 5)  # PP_E_NCCL (timeout) / PP_E_INTERNAL (injected)
            assert np.array_equal(np.sort(to_host(t, np.uint64)), np.sort(a))
    finally:
        pp.reset_params()
    # the library still works afterwards
    t = to_dev(a)
    K = pp.pp_partition_dist_loopback(t, ns, 1 << 63)
    oracle.check_partition(a, to_host(t, np.uint64), 1 << 63, K)


def test_loopback_fuzz(pp):
    """Seeded fuzz of the product exchange at P > 1 (loopback): random rank
    counts, shard sizes (empty ones included), key widths, key alphabets,
    pivots, staging caps and exchange paths; partition against the oracle's
    checks, quicksort byte for byte against oracle.quicksort."""
    import os
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(int(os.environ.get("PP_FUZZ_SEED", 20_0412_532)))
    try:
        for trial in range(40):
            P = int(rng.integers(2, 9))
            dt = np.uint64 if rng.random() < 0.6 else np.uint32
            mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
            total = [0, 1, 7, 1000, 65_537, 333_333, 1 << 20][int(rng.integers(0, 7))]
            ns = _shards(rng, total, P, str(rng.choice(["ragged", "empty", "equal"])))
            alpha = int(rng.choice([2, 1000, 0]))
            a = (rng.integers(0, alpha, size=total).astype(dt) if alpha
                 else rng.integers(0, mx, size=total, dtype=dt, endpoint=True))
            pp.reset_params()
            pp.pp_set_param("dist_p2p", int(rng.integers(0, 2)))
            pp.pp_set_param("dist_small", int(rng.choice([64, 5000, 1 << 16])))
            pp.pp_set_param("qs_pivot", int(rng.integers(0, 3)))
            pp.pp_set_param("dist_overlap", int(rng.integers(0, 2)))
            pp.pp_set_param("dist_chunks", int(rng.choice([1, 2, 5, 8])))
            pp.pp_dist_set_staging(int(rng.choice([16, 4096, 1 << 20, 256 << 20])))
            ctx = (trial, P, dt, total, ns, alpha)
            if rng.random() < 0.5:
                cands = [0, mx, int(a[rng.integers(0, total)]) if total else 1, int(rng.integers(0, mx, dtype=dt))]
                pivot = cands[int(rng.integers(0, len(cands)))]  # (rng.choice would round through float64)
                t = to_dev(a) if total else torch.empty(0, dtype=torch.int64 if dt == np.uint64 else torch.int32,
                                                       device="cuda")
                K = pp.pp_partition_dist_loopback(t, ns, pivot)
                assert K == oracle.count(a, pivot), ctx
                if total:
                    oracle.check_partition(a, to_host(t, dt), pivot, K)
            elif total:
                t = to_dev(a)
                pp.pp_quicksort_dist_loopback(t, ns)
                ref = a.copy()
                oracle.quicksort(ref)
                assert np.array_equal(to_host(t, dt), ref), ctx
    finally:
        pp.pp_dist_set_staging(256 << 20)
        pp.reset_params()
