"""Input generators: numpy and torch versions agree byte for byte (CPU)."""
import numpy as np
import torch

import synth


def test_uniform_np_torch_agree():
    for seed in (0, 1, 0xC0FFEE02, (1 << 64) - 1):
        for off in (0, 12345):
            a = synth.uniform_u64_np(1000, seed, off)
            t = synth.uniform_u64_torch(1000, seed, "cpu", off).numpy().view(np.uint64)
            assert np.array_equal(a, t)
            a32 = synth.uniform_u32_np(1000, seed, off)
            t32 = synth.uniform_u32_torch(1000, seed, "cpu", off).numpy().view(np.uint32)
            assert np.array_equal(a32, t32)
            m = synth.mod_range_u64_np(1000, seed, 1000, off)
            tm = synth.mod_range_u64_torch(1000, seed, 1000, "cpu", off).numpy().view(np.uint64)
            assert np.array_equal(m, tm) and m.max() < 1000


def test_splitmix_known_value():
    # splitmix64 with state seed=0: first output is fmix64(0x9E3779B97F4A7C15)
    # = 0xE220A8397B1DCDAF (the published first output of splitmix64(0)).
    assert int(synth.uniform_u64_np(1, 0)[0]) == 0xE220A8397B1DCDAF


def test_shard_offsets_compose():
    full = synth.uniform_u64_np(4096, 99)
    parts = [synth.uniform_u64_np(1024, 99, o) for o in range(0, 4096, 1024)]
    assert np.array_equal(full, np.concatenate(parts))


def test_zipf_torch_matches_truncated_law():
    """The device Zipf(1.1) sampler (rejection-inversion) against the exact
    truncated law P(rank = k) = k^-1.1 / (zeta(1.1) - zeta(1.1, 2^32 + 1))
    (Hurwitz zeta, scipy): P(key = 0), P(key < 7), P(key < 217) within 5 sigma."""
    from scipy.special import zeta
    s = 1.1
    Z = zeta(s) - zeta(s, 2.0 ** 32 + 1)
    n = 300_000
    z = synth.zipf_u32_torch(n, s, 123, "cpu").numpy().view(np.uint32)
    for thr in (1, 7, 217):
        p = sum(k ** -s for k in range(1, thr + 1)) / Z
        sigma = (p * (1 - p) / n) ** 0.5
        assert abs((z < thr).mean() - p) < 5 * sigma, (thr, (z < thr).mean(), p)


def test_adversarial_patterns():
    n = 1001
    for pat in synth.ADV_PATTERNS:
        a = synth.adversarial_u32_np(n, pat, 3)
        t = synth.adversarial_u32_torch(n, pat, 3, "cpu").numpy().view(np.uint32)
        assert np.array_equal(a, t), pat
        k = int(np.sum(a < synth.ADV_PIVOT_U32))
        exp = {"partitioned": n // 2, "reverse": n // 2, "all_true": n, "all_false": 0,
               "alternating": (n + 1) // 2}[pat]
        assert k == exp, pat
