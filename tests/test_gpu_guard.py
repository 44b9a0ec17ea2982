"""GPU: out-of-bounds and race checks of our own (compute-sanitizer is closed
on this GPU pool -- DESIGN.md §10): every kernel family runs on a key range
embedded between guard bands, and with a caller workspace whose tail past the
declared bound (pp_workspace_bytes) is a guard band; no guard byte may change
(memcheck's out-of-bounds writes).  Race proxy (racecheck / synccheck): the
same input partitioned and sorted repeatedly while other kernels compete for
the SMs must give byte-identical outputs (the library is deterministic by
construction; a race shows up as a different arrangement or a
wrong result)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

pytestmark = pytest.mark.gpu

G = 4096  # guard keys on each side
SENT64 = np.uint64(0xDEADBEEFCAFEF00D)
SENT32 = np.uint32(0xDEADBEEF)


@pytest.fixture(scope="module")
def pp():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2004_12532_b200 as m
    m.load()
    m.reset_params()
    yield m
    m.pp_set_workspace(None)
    m.reset_params()


def _guarded(a):
    from gpu_util import to_dev
    sent = SENT64 if a.dtype == np.uint64 else SENT32
    g = np.full(G, sent, dtype=a.dtype)
    buf = to_dev(np.concatenate([g, a, g]))
    return buf, buf[G:G + a.size]


def _guards_ok(buf, n, dt):
    h = buf.cpu().numpy().view(dt)
    sent = SENT64 if dt == np.uint64 else SENT32
    return bool(np.all(h[:G] == sent) and np.all(h[G + n:] == sent)), h[G:G + n]


class _GuardedWorkspace:
    """Caller workspace = the declared bound + a guard tail of 1 MiB."""

    def __init__(self, pp, n, kb, op):
        self.pp = pp
        self.need = pp.pp_workspace_bytes(n, kb, op)
        self.tail = 1 << 20
        self.ws = torch.full(((self.need + self.tail + 255) // 8,), -0x2152411035014111, dtype=torch.int64,
                             device="cuda")  # 0xDEADBEEFCAFEEFEF pattern
        self.start = self.need // 8 + 1

    def __enter__(self):
        # the library gets exactly the declared bound; the tail is ours
        self.pp._check(self.pp.load().pp_set_workspace(self.ws.data_ptr(), self.need), "pp_set_workspace")
        return self

    def __exit__(self, *exc):
        self.pp.pp_set_workspace(None)

    def tail_ok(self):
        return bool((self.ws[self.start:] == -0x2152411035014111).all())


PART_CASES = [{}, {"small_n": 1 << 12, "cleanup_chain": 1}, {"small_n": 1 << 12, "cleanup_chain": 0},
              {"small_n": 1 << 12, "cleanup_chain": 0, "cleanup_bitmap": 0}, {"path": 3}, {"path": 1},
              {"strided": 1}]


@pytest.mark.parametrize("params", PART_CASES)
@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_partition_guards(pp, params, dt):
    rng = np.random.default_rng(len(params) * 3 + (dt == np.uint64))
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    for n in (1, 999, 70_001, 1_000_003, 1 << 22):
        if params.get("path") == 1 and n > 100_000:
            continue
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        p = int(rng.integers(0, mx, dtype=dt))
        with _GuardedWorkspace(pp, n, a.itemsize, 0) as ws:
            for k, v in params.items():
                pp.pp_set_param(k, v)
            try:
                buf, view = _guarded(a)
                K = pp.pp_partition(view, p)
                torch.cuda.synchronize()
            finally:
                pp.reset_params()
            assert ws.tail_ok(), ("workspace written past its declared bound", params, n)
        ok, out = _guards_ok(buf, n, dt)
        assert ok, ("keys written outside [keys, keys+n)", params, n)
        oracle.check_partition(a, out, p, K)


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_quicksort_guards(pp, dt):
    rng = np.random.default_rng(17 + (dt == np.uint64))
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    for n, kind in ((2, "u"), (5000, "u"), (300_007, "u"), (300_007, "dup"), (1 << 22, "u"), (1 << 22, "dup")):
        a = (rng.integers(0, mx, size=n, dtype=dt, endpoint=True) if kind == "u"
             else rng.integers(0, 1000, size=n).astype(dt))
        with _GuardedWorkspace(pp, n, a.itemsize, 1) as ws:
            buf, view = _guarded(a)
            pp.pp_quicksort(view)
            torch.cuda.synchronize()
            assert ws.tail_ok(), ("workspace written past its declared bound", n, kind)
        ok, out = _guards_ok(buf, n, dt)
        assert ok, ("keys written outside the range", n, kind)
        ref = a.copy()
        oracle.quicksort(ref)
        assert np.array_equal(out, ref)


def test_bps_stable_dist_guards(pp):
    from gpu_util import to_dev, to_host
    a = synth.uniform_u64_np(300_007, 5)
    buf, view = _guarded(a)
    K = pp.pp_partition_bps(view, 1 << 63)
    ok, out = _guards_ok(buf, a.size, np.uint64)
    assert ok
    oracle.check_partition(a, out, 1 << 63, K)
    src_buf, src = _guarded(a)
    dst_buf, dst = _guarded(np.zeros_like(a))
    K = pp.pp_partition_stable(src, dst, 1 << 63)
    ok1, _ = _guards_ok(src_buf, a.size, np.uint64)
    ok2, out = _guards_ok(dst_buf, a.size, np.uint64)
    assert ok1 and ok2
    ref = a.copy()
    assert oracle.partition_standard(ref, 1 << 63) == K and np.array_equal(out, ref)
    buf, view = _guarded(a)
    K = pp.pp_partition_stable_inplace(view, 1 << 63)
    ok, out = _guards_ok(buf, a.size, np.uint64)
    assert ok and K == oracle.partition_standard(ref.copy(), 1 << 63) and np.array_equal(out, ref)
    buf, view = _guarded(a)
    ns = [100_000, 0, 150_000, 50_007]
    pp.pp_dist_set_staging(1 << 14)
    try:
        K = pp.pp_partition_dist_loopback(view, ns, 1 << 63)
    finally:
        pp.pp_dist_set_staging(256 << 20)
    ok, out = _guards_ok(buf, a.size, np.uint64)
    assert ok
    oracle.check_partition(a, out, 1 << 63, K)


def test_race_proxy_determinism_under_contention(pp):
    """Outputs byte-identical across repeated runs while a competing stream
    keeps kernels resident on the SMs (different CTA placement and timing on
    every run)."""
    from gpu_util import to_dev
    a = synth.uniform_u64_np(1 << 22, 99)
    q = synth.uniform_u64_np(1 << 21, 98)
    side = torch.cuda.Stream()
    x = torch.randn(4096, 4096, device="cuda")
    ref_p = ref_q = None
    for rep in range(6):
        with torch.cuda.stream(side):
            for _ in range(rep):
                x = (x @ x).clamp_(-1, 1)
        for params in ({}, {"cleanup_chain": 0}, {"cleanup_chain": 1}):
            for k, v in params.items():
                pp.pp_set_param(k, v)
            t = to_dev(a)
            pp.pp_partition(t, 1 << 63)
            pp.reset_params()
            h = t.cpu().numpy()
            if rep == 0 and not params:
                ref_p = h
            elif not params:
                assert np.array_equal(h, ref_p), "partition output differs between runs"
        t = to_dev(q)
        pp.pp_quicksort(t)
        hq = t.cpu().numpy()
        if rep == 0:
            ref_q = hq
        else:
            assert np.array_equal(hq, ref_q)
    torch.cuda.synchronize()
