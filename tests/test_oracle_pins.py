"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names what fixes the oracle: a library routine (numpy sort /
searchsorted / cumsum / stable argsort), brute force over all small inputs,
a closed form or invariant from PAPER.md, or a SPEC.md worked example stored
under tests/golden/ with its citation.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

U64_MAX = (1 << 64) - 1
U32_MAX = (1 << 32) - 1


def _props(inp, out, pivot, split):
    """(1)-(3) of SURVEY §8(c), checked with numpy only."""
    inp = np.asarray(inp)
    out = np.asarray(out)
    K = int(np.searchsorted(np.sort(inp), np.array(pivot, dtype=inp.dtype), side="left"))
    assert split == K
    assert np.all(out[:K] < pivot) and np.all(out[K:] >= pivot)
    assert np.array_equal(np.sort(out), np.sort(inp))


# ----------------------------------------------------------------------------
# SPEC.md worked examples (tests/golden/spec_examples.json)
# ----------------------------------------------------------------------------

def test_golden_partition(golden):
    for ex in golden["partition"]:
        for dt in (np.uint64, np.uint32):
            a = np.array(ex["keys"], dtype=dt)
            b = a.copy()
            assert oracle.partition_two_pointer(b, ex["pivot"]) == ex["split"], ex["cite"]
            _props(a, b, ex["pivot"], ex["split"])
            c = a.copy()
            assert oracle.partition_standard(c, ex["pivot"]) == ex["split"], ex["cite"]
            assert c.tolist() == ex["stable_output"], ex["cite"]
            assert oracle.count(a, ex["pivot"]) == ex["split"]


def test_golden_make_successor_heavy(golden):
    """SPEC.md:344 worked example of Fig. 1 MakeSuccessorHeavy
    pins the oracle's ARRANGEMENT (swap order and recursion split), not only
    Lemma 3.1's prefix property; both key widths."""
    for ex in golden["make_successor_heavy"]:
        for dt in (np.uint64, np.uint32):
            a = np.array(ex["keys"], dtype=dt)
            oracle.bps_make_successor_heavy(a, ex["pivot"], False)
            assert a.tolist() == ex["output"], ex["cite"]


def test_golden_is_partitioned(golden):
    for ex in golden["is_partitioned"]:
        a = np.array(ex["keys"], dtype=np.uint64)
        assert oracle.is_partitioned(a, ex["pivot"], ex["k"]) == ex["expect"], ex["cite"]


def test_golden_prefix_sum(golden):
    for ex in golden["prefix_sum"]:
        assert oracle.prefix_sum(ex["input"]).tolist() == ex["output"], ex["cite"]


def test_golden_block_start_index(golden):
    """Fig. 3 GetBlockStartIndex through ss_groups: with all keys successors,
    v_i is the start of U_i's first line; with U_i's first line all
    predecessors (T_i = b), v_i is the start of its second line.  The oracle's
    0-based offsets are X0 = (X + 1) mod g (reading: 1-based i, X)."""
    for ex in golden["block_start_index"]:
        g, b, i1, j1 = ex["g"], ex["b"], ex["i"], ex["j"]
        X0 = [(x + 1) % g for x in ex["X_1based"]]
        n_lines = g * len(X0)
        a = np.full(n_lines * b, 100, dtype=np.uint64)       # all successors (pivot 50)
        if j1 == 2:
            # make U_i's first line (found with j=1 on an all-successor array) predecessors
            T, vlo, _ = oracle.ss_groups(a, 0, n_lines, b, g, X0, 50)
            first = int(vlo[i1 - 1])
            a[first:first + b] = 1
        T, vlo, vhi = oracle.ss_groups(a, 0, n_lines, b, g, X0, 50)
        assert int(vlo[i1 - 1]) + 1 == ex["start_1based"], ex["cite"]
        assert vlo[i1 - 1] == vhi[i1 - 1]


# ----------------------------------------------------------------------------
# count: closed form vs a library routine
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_count_vs_searchsorted(dt, mx):
    rng = np.random.default_rng(1)
    for n in (0, 1, 2, 7, 1000, 4097):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for p in (0, 1, mx // 2, mx, int(a[0]) if n else 5):
            ref = int(np.searchsorted(np.sort(a), np.array(p, dtype=dt), side="left"))
            assert oracle.count(a, p) == ref


# ----------------------------------------------------------------------------
# two-pointer and standard partitions: brute force over all tiny inputs
# ----------------------------------------------------------------------------

def test_bruteforce_alphabet4():
    """Every array over {0,1,2,3} with n <= 6 (5461 arrays) x pivots 0..4."""
    for n in range(0, 7):
        for tup in itertools.product(range(4), repeat=n):
            a = np.array(tup, dtype=np.uint64)
            for p in range(5):
                b = a.copy()
                k = oracle.partition_two_pointer(b, p)
                _props(a, b, p, k)
                c = a.copy()
                k2 = oracle.partition_standard(c, p)
                assert k2 == k
                # stable => unique: a library stable sort by the predicate
                ref = a[np.argsort(~(a < p), kind="stable")]
                assert np.array_equal(c, ref)


def test_bruteforce_patterns_tagged():
    """All 2^n predecessor/successor patterns for n <= 12 with distinct keys
    (identity of each key tracked by value)."""
    for n in range(0, 13):
        for mask in range(1 << n):
            bits = np.array([(mask >> i) & 1 for i in range(n)], dtype=bool)
            idx = np.arange(n, dtype=np.uint32)
            a = np.where(bits, idx, idx + 1000).astype(np.uint32)   # pred < 1000 <= succ
            b = a.copy()
            k = oracle.partition_two_pointer(b, 1000)
            _props(a, b, 1000, k)
            c = a.copy()
            assert oracle.partition_standard(c, 1000) == k
            assert np.array_equal(c, a[np.argsort(~bits, kind="stable")])


@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_random_partitions_vs_library(dt, mx):
    rng = np.random.default_rng(7)
    for n in (1, 2, 3, 100, 5000, 65537):
        a = rng.integers(0, mx, size=n, dtype=dt, endpoint=True)
        for p in (0, 1, mx, mx // 3, int(a[n // 2])):
            b = a.copy()
            k = oracle.partition_two_pointer(b, p)
            _props(a, b, p, k)
            c = a.copy()
            assert oracle.partition_standard(c, p) == k
            assert np.array_equal(c, a[np.argsort(~(a < p), kind="stable")])


# ----------------------------------------------------------------------------
# prefix sum: library cumsum
# ----------------------------------------------------------------------------

def test_prefix_sum_vs_cumsum():
    rng = np.random.default_rng(3)
    for n in list(range(0, 40)) + [1023, 1024, 1025, 99991]:
        d = rng.integers(0, 2, size=n).astype(np.uint64)
        assert np.array_equal(oracle.prefix_sum(d), np.cumsum(d, dtype=np.uint64))
        w = rng.integers(0, 1 << 20, size=n).astype(np.uint64)     # general summands
        assert np.array_equal(oracle.prefix_sum(w), np.cumsum(w, dtype=np.uint64))


# ----------------------------------------------------------------------------
# quicksort: unique output => numpy.sort byte for byte
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("dt,mx", [(np.uint64, U64_MAX), (np.uint32, U32_MAX)])
def test_quicksort_vs_numpy(dt, mx):
    rng = np.random.default_rng(11)
    cases = []
    for n in (0, 1, 2, 3, 15, 16, 17, 33, 1000, 100003):
        cases.append(rng.integers(0, mx, size=n, dtype=dt, endpoint=True))
        cases.append(rng.integers(0, 1000, size=n).astype(dt))        # duplicate-heavy
        cases.append(np.full(n, 7, dtype=dt))                         # all equal
        cases.append(np.full(n, mx, dtype=dt))                        # all MAX
        cases.append(np.arange(n, dtype=dt))                          # sorted
        cases.append(np.arange(n, dtype=dt)[::-1].copy())             # reverse
        cases.append(rng.integers(0, 2, size=n).astype(dt) * dt(mx))  # {0, MAX}
    for a in cases:
        b = a.copy()
        oracle.quicksort(b)
        assert np.array_equal(b, np.sort(a))


# ----------------------------------------------------------------------------
# Smoothed Striding group statistics
# ----------------------------------------------------------------------------

def _groups_bruteforce(a, base, n_lines, b, g, X, pivot):
    """Independent enumeration: line q of chunk j belongs to group
    i = (q - X[j]) mod g (inverse of the Fig. 3 map); the group's elements in
    group order are its positions in ascending order."""
    members = [[] for _ in range(g)]
    for line in range(n_lines):
        j, q = divmod(line, g)
        i = (q - int(X[j])) % g
        members[i].extend(range(base + line * b, base + line * b + b))
    T = np.zeros(g, dtype=np.uint64)
    vlo = np.zeros(g, dtype=np.uint64)
    vhi = np.zeros(g, dtype=np.uint64)
    for i in range(g):
        pos = sorted(members[i])
        t = sum(1 for x in pos if a[x] < pivot)
        T[i] = t
        if not pos:
            vlo[i], vhi[i] = base + n_lines * b, base
        elif t == len(pos):
            vlo[i] = vhi[i] = pos[-1] + 1
        else:
            vlo[i] = vhi[i] = pos[t]
    return T, vlo, vhi, members


@pytest.mark.parametrize("g,b,n_lines,base", [(4, 2, 8, 0), (4, 2, 9, 3), (7, 4, 40, 1),
                                              (16, 8, 100, 0), (3, 16, 2, 5), (5, 4, 0, 0)])
def test_ss_groups_bruteforce(g, b, n_lines, base):
    rng = np.random.default_rng(g * 1000 + b)
    s = (n_lines + g - 1) // g
    for trial in range(20):
        n = base + n_lines * b + 3
        a = rng.integers(0, 100, size=n).astype(np.uint64)
        X = rng.integers(0, g, size=max(1, s))
        p = int(rng.integers(0, 101))
        T, vlo, vhi = oracle.ss_groups(a, base, n_lines, b, g, X, p)
        T2, vlo2, vhi2, members = _groups_bruteforce(a, base, n_lines, b, g, X, p)
        assert np.array_equal(T, T2) and np.array_equal(vlo, vlo2) and np.array_equal(vhi, vhi2)
        # window invariant: partition each group (stably,
        # in group order) and check A[x] pred for x < v_min, succ for x >= v_max
        if n_lines:
            c = a.copy()
            for i in range(g):
                pos = sorted(members[i])
                vals = c[pos]
                c[pos] = vals[np.argsort(~(vals < p), kind="stable")]
            vmin, vmax = int(vlo.min()), int(vhi.max())
            region = slice(base, base + n_lines * b)
            r = c[region]
            lo, hi = vmin - base, vmax - base
            assert np.all(r[:lo] < p) and np.all(r[hi:] >= p)
            assert lo <= int(T.sum()) <= hi


def test_ss_offsets_generator():
    """Range and determinism of the counter-based offset generator."""
    for g in (1, 2, 7, 444, 1 << 20):
        X = synth.ss_offsets(0xABC, 1000, g)
        assert X.dtype == np.uint64 and X.min() >= 0 and X.max() < g
        assert np.array_equal(X, synth.ss_offsets(0xABC, 1000, g))
    X = synth.ss_offsets(5, 200000, 8)
    counts = np.bincount(X.astype(np.int64), minlength=8)
    assert counts.min() > 0.9 * 25000 and counts.max() < 1.1 * 25000


def test_strided_vs_smoothed_window_on_stride_aligned_adversary():
    """SURVEY §8(f) #2 / PAPER.md:836-849 vs 865-913: on the stride-aligned
    adversary (line j true iff j mod g < g/2) the Strided Algorithm (X = 0)
    leaves almost the whole region unresolved (groups are all-true or
    all-false), while uniformly random offsets X (Smoothed Striding) leave a
    window of a few chunks.  Checked with the oracle's group statistics."""
    g, b, s = 16, 32, 256
    n_lines = g * s
    a = synth.stride_aligned_u64_np(n_lines * b, 3, b, g)
    p = 1 << 63
    def window(X):
        T, vlo, vhi = oracle.ss_groups(a, 0, n_lines, b, g, X, p)
        assert int(T.sum()) == oracle.count(a, p)
        return (int(vhi.max()) - int(vlo.min())) / (n_lines * b)
    w_strided = window(np.zeros(s, dtype=np.uint64))
    w_smooth = window(synth.ss_offsets(0x5EEDC0DE2004, s, g))
    assert w_strided > 0.9, w_strided
    assert w_smooth < 0.25, w_smooth


def test_stride_aligned_np_torch_agree():
    a = synth.stride_aligned_u64_np(5000, 11, 64, 6)
    t = synth.stride_aligned_u64_torch(5000, 11, 64, 6, "cpu").numpy().view(np.uint64)
    assert np.array_equal(a, t)
    line = np.arange(5000) // 64
    assert np.array_equal(a < (1 << 63), (line % 6) < 3)


def _succ_heavy(pred: np.ndarray) -> bool:
    """Lemma 3.1: every t-prefix holds >= t/4 successors."""
    succ = np.cumsum(~pred)
    t = np.arange(1, pred.size + 1)
    return bool(np.all(4 * succ >= t))


@pytest.mark.parametrize("rev", [False, True])
def test_bps_make_successor_heavy_lemma(rev):
    """MakeSuccessorHeavy: on every predecessor/successor
    pattern with at least half successors (in the view), the result is a
    permutation of the input whose every prefix is successor-heavy."""
    for n in range(0, 13):
        for mask in range(1 << n):
            bits = np.array([(mask >> i) & 1 for i in range(n)], dtype=bool)  # True = view predecessor
            if 2 * int(bits.sum()) > n:
                continue  # the phase requires >= half successors
            idx = np.arange(n, dtype=np.uint64)
            # keys: view predecessor <=> key < 1000 (rev: view predecessor <=> key >= 1000)
            pred_key = bits if not rev else ~bits
            a = np.where(pred_key, idx, idx + 1000).astype(np.uint64)
            if rev:
                a = a[::-1].copy()
            b = a.copy()
            oracle.bps_make_successor_heavy(b, 1000, rev)
            assert np.array_equal(np.sort(a), np.sort(b))
            view = b[::-1] if rev else b
            vpred = (view < 1000) if not rev else (view >= 1000)
            assert _succ_heavy(vpred), (n, mask, rev)


@pytest.mark.parametrize("B", [1, 2, 3, 4, 8])
def test_bps_partition_bruteforce(B):
    """The Blocked-Prefix-Sum partition (low-space form
    PAPER.md:1466-1486): every 2^n pattern for n <= 12 (tagged keys, both
    role-swap sides), block sizes 1..8 so the Reorder recursion runs several
    levels; (1)-(3) hold and no Reorder swap broke Lemma 3.4 (the oracle
    raises if one did)."""
    for n in range(0, 13):
        for mask in range(1 << n):
            bits = np.array([(mask >> i) & 1 for i in range(n)], dtype=bool)
            idx = np.arange(n, dtype=np.uint64)
            a = np.where(bits, idx, idx + 1000).astype(np.uint64)
            b = a.copy()
            k = oracle.partition_bps(b, 1000, B)
            oracle.check_partition(a, b, 1000, k)


@pytest.mark.parametrize("dt", [np.uint64, np.uint32])
def test_bps_partition_random(dt):
    """Larger random and duplicate-heavy arrays, several pivots and block
    sizes (deep Reorder recursions), ragged last blocks."""
    rng = np.random.default_rng(77)
    mx = (1 << 64) - 1 if dt == np.uint64 else (1 << 32) - 1
    for n in (0, 1, 5, 97, 1000, 4096, 4097, 20001, 100003):
        for a in (rng.integers(0, mx, size=n, dtype=dt, endpoint=True), rng.integers(0, 4, size=n).astype(dt)):
            for p in (0, 1, 2, mx // 100, mx // 2, mx - mx // 100, mx):
                for B in (4, 64, 4096):
                    b = a.copy()
                    k = oracle.partition_bps(b, p, B)
                    oracle.check_partition(a, b, p, k)


def _prop42_inputs(rng, n_lines, b, g):
    """Uniform keys, and whole-line patterns (every line all-predecessor or
    all-successor with probability 1/2: the largest per-line variance the
    proof's Y_i(j) in [0, 1] allow)."""
    n = n_lines * b
    uni = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    lines = rng.integers(0, 2, size=n_lines).astype(bool)
    whole = np.where(np.repeat(lines, b), np.uint64(1), np.uint64(3)).astype(np.uint64)
    return [(uni, 1 << 63), (whole, 2)]


def _check_prop42(T, vlo, n_lines, b, g, mu, eps):
    """PAPER.md:1160-1166 (0-based): group i's first successor lies in the
    chunk of its (T_i)-th element, so |v_i - g T_i| <= g b
    (Hoeffding + union bound over the g groups): with probability >= 1 - eps
    every |mu_i - mu| < delta, delta = sqrt(ln(2 g / eps) / (2 s)); Prop. 4.2
    (PAPER.md:1086-1099): v_max - v_min < 4 n delta' with
    s = ln(n / eps) / delta'^2."""
    s = n_lines // g
    n = n_lines * b
    for i in range(g):
        if int(T[i]) < s * b:
            assert abs(int(vlo[i]) - g * int(T[i])) <= g * b, (i, int(vlo[i]), int(T[i]))
    delta = np.sqrt(np.log(2 * g / eps) / (2 * s))
    mui = T.astype(np.float64) / (s * b)
    assert np.all(np.abs(mui - mu) < delta), (float(np.abs(mui - mu).max()), delta)
    d2 = np.sqrt(np.log(n / eps) / s)
    assert int(vlo.max()) - int(vlo.min()) < 4 * n * d2


def test_prop42_smoothed_striding_bounds():
    """The oracle's Smoothed Striding step obeys Prop. 4.2's statements on
    full-chunk layouts (n_lines a multiple of g), over several offset draws."""
    rng = np.random.default_rng(1099)
    g, b, s = 16, 8, 4096
    n_lines = g * s
    for a, p in _prop42_inputs(rng, n_lines, b, g):
        mu = float(np.mean(a < np.uint64(p)))
        for seed in (1, 2, 3):
            X = synth.ss_offsets(seed, s, g)
            T, vlo, _ = oracle.ss_groups(a, 0, n_lines, b, g, X, p)
            assert int(T.sum()) == oracle.count(a, p)
            _check_prop42(T, vlo, n_lines, b, g, mu, 1e-6)
