"""GPU: every data-carrying C-ABI entry point on real data against the oracle
(entry points the other suites reach only through their error paths):
pp_quicksort_host_u64, pp_partition_async_u32, and the north-star symbols
pp_partition(keys, n, pivot) -> split / pp_quicksort(keys, n) called directly
through ctypes (PAPER.md:272-281 partition, PAPER.md:1701-1732 quicksort)."""
import ctypes

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
    yield m
    m.reset_params()


@pytest.mark.parametrize("pinned", [False, True])
def test_quicksort_host_u64(pp, pinned):
    rng = np.random.default_rng(5)
    for a in (np.zeros(0, np.uint64), np.array([7], np.uint64), rng.integers(0, 9, size=1000).astype(np.uint64),
              synth.uniform_u64_np(1_000_003, 3), synth.mod_range_u64_np(2_000_001, 4, 1000)):
        if pinned:
            h = torch.empty(a.size, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
            h[:] = a
        else:
            h = a.copy()
        pp.pp_quicksort_host_u64(h)
        ref = a.copy()
        oracle.quicksort(ref)
        assert np.array_equal(h, ref)


def test_partition_async_u32(pp):
    from gpu_util import to_dev, to_host
    rng = np.random.default_rng(6)
    d = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    for n in (0, 1, 37, 5000, 40_000, 1_000_003, 1 << 24):
        a = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        for p in (0, 1 << 31, (1 << 32) - 1, int(rng.integers(0, 1 << 32))):
            t = to_dev(a) if n else torch.empty(0, dtype=torch.int32, device="cuda")
            pp.pp_partition_async_u32(t, p, d)
            K = int(d.item())
            assert K == oracle.count(a, p)
            oracle.check_partition(a, to_host(t, np.uint32), p, K)


def test_async_rejects_narrow_split_word(pp):
    t = torch.zeros(100, dtype=torch.int32, device="cuda")
    with pytest.raises((TypeError, ValueError)):
        pp.pp_partition_async_u32(t, 5, torch.zeros(1, dtype=torch.int32, device="cuda"))


def test_north_star_symbols(pp):
    """pp_partition(keys, n, pivot) -> split and pp_quicksort(keys, n) on the
    legacy default stream, called as plain C functions."""
    from gpu_util import to_dev, to_host
    L = pp.load()
    for n in (1, 1000, 1 << 20, 3_000_017):
        a = synth.uniform_u64_np(n, 11)
        t = to_dev(a)
        torch.cuda.synchronize()
        split = L.pp_partition(ctypes.c_void_p(t.data_ptr()), n, 1 << 63)
        assert split != (1 << 64) - 1, L.pp_last_error()
        assert split == oracle.count(a, 1 << 63)
        oracle.check_partition(a, to_host(t, np.uint64), 1 << 63, split)
        t = to_dev(a)
        torch.cuda.synchronize()
        assert L.pp_quicksort(ctypes.c_void_p(t.data_ptr()), n) == 0, L.pp_last_error()
        ref = a.copy()
        oracle.quicksort(ref)
        assert np.array_equal(to_host(t, np.uint64), ref)
