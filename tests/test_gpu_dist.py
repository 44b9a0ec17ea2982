"""GPU: the C-ABI multi-GPU partition (pp_dist_*) on a single-rank NCCL
communicator (only one GPU is available to the tests; the exchange logic
with several ranks is covered on CPU by tests/test_dist.py)."""
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
