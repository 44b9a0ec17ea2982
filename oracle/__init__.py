"""CPU oracle for the in-place parallel partition (+ quicksort) of arxiv 2004.12532.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (paper_2004_12532_b200/) never imports it and shares no code with
it; the arithmetic lives in ``pp_oracle.c`` (plain serial C, every function
citing the PAPER.md passage it follows), this file only marshals numpy arrays.

Pins: tests/test_oracle_pins.py (brute force, closed forms, library routines,
SPEC.md worked examples).  Functions and their pin status:

- count            : pinned (closed form; numpy.searchsorted on a library sort)
- two_pointer      : pinned ((1) split, (2) predicate, (3) multiset; brute force)
- standard         : pinned (stable => unique; equals a numpy stable argsort
                     by the predicate; SPEC.md:296 example)
- prefix_sum       : pinned (numpy.cumsum; SPEC.md:287 example)
- quicksort        : pinned (numpy.sort byte-for-byte)
- ss_groups        : pinned (brute-force group enumeration in the test and
                     the window invariant PAPER.md:999-1001 on partitioned data)
- bps_make_successor_heavy : pinned (Lemma 3.1: every t-prefix holds >= t/4
                     successors, brute force over all small patterns; a
                     permutation of the input)
- partition_bps    : pinned ((1)-(3) by brute force over all small patterns
                     and several block sizes; Lemma 3.4's conflict-freeness
                     checked inside on every swap)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

U64P = ctypes.POINTER(ctypes.c_uint64)
U32P = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile pp_oracle.c -> liboracle.so (plain gcc -O2, serial)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64 = ctypes.c_uint64
        for sfx, P, K in (("u64", U64P, ctypes.c_uint64), ("u32", U32P, ctypes.c_uint32)):
            getattr(L, f"oracle_count_{sfx}").argtypes = [P, u64, K]
            getattr(L, f"oracle_count_{sfx}").restype = u64
            getattr(L, f"oracle_is_partitioned_{sfx}").argtypes = [P, u64, K, u64]
            getattr(L, f"oracle_is_partitioned_{sfx}").restype = ctypes.c_int
            getattr(L, f"oracle_partition_two_pointer_{sfx}").argtypes = [P, u64, K]
            getattr(L, f"oracle_partition_two_pointer_{sfx}").restype = u64
            getattr(L, f"oracle_partition_standard_{sfx}").argtypes = [P, u64, K, U64P, P]
            getattr(L, f"oracle_partition_standard_{sfx}").restype = u64
            getattr(L, f"oracle_quicksort_{sfx}").argtypes = [P, u64]
            getattr(L, f"oracle_quicksort_{sfx}").restype = None
            getattr(L, f"oracle_ss_groups_{sfx}").argtypes = [P, u64, u64, u64, u64, U64P, K,
                                                              U64P, U64P, U64P]
            getattr(L, f"oracle_ss_groups_{sfx}").restype = None
            getattr(L, f"oracle_bps_make_successor_heavy_{sfx}").argtypes = [P, u64, K, ctypes.c_int]
            getattr(L, f"oracle_bps_make_successor_heavy_{sfx}").restype = None
            getattr(L, f"oracle_partition_bps_{sfx}").argtypes = [P, u64, K, u64, U64P]
            getattr(L, f"oracle_partition_bps_{sfx}").restype = u64
        L.oracle_prefix_sum_recursive.argtypes = [U64P, u64]
        L.oracle_prefix_sum_recursive.restype = None
        _lib = L
    return _lib


def _sfx(a: np.ndarray):
    if a.dtype == np.uint64:
        return "u64", U64P, ctypes.c_uint64
    if a.dtype == np.uint32:
        return "u32", U32P, ctypes.c_uint32
    raise TypeError(f"oracle keys must be uint64 or uint32, got {a.dtype}")


def _ptr(a: np.ndarray, P):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(P)


def count(a: np.ndarray, pivot: int) -> int:
    sfx, P, K = _sfx(a)
    return int(getattr(lib(), f"oracle_count_{sfx}")(_ptr(a, P), a.size, K(pivot)))


def is_partitioned(a: np.ndarray, pivot: int, k: int) -> bool:
    sfx, P, K = _sfx(a)
    return bool(getattr(lib(), f"oracle_is_partitioned_{sfx}")(_ptr(a, P), a.size, K(pivot), k))


def partition_two_pointer(a: np.ndarray, pivot: int) -> int:
    """In place; returns the split."""
    sfx, P, K = _sfx(a)
    return int(getattr(lib(), f"oracle_partition_two_pointer_{sfx}")(_ptr(a, P), a.size, K(pivot)))


def partition_standard(a: np.ndarray, pivot: int) -> int:
    """In place (through Theta(n) scratch); stable; returns the split."""
    sfx, P, K = _sfx(a)
    S = np.empty(max(1, a.size), dtype=np.uint64)
    C = np.empty(max(1, a.size), dtype=a.dtype)
    return int(getattr(lib(), f"oracle_partition_standard_{sfx}")(
        _ptr(a, P), a.size, K(pivot), _ptr(S, U64P), _ptr(C, P)))


def bps_make_successor_heavy(a: np.ndarray, pivot: int, rev: bool = False) -> None:
    """In place: the Preprocessing phase on the view
    (reversed, with roles swapped, when rev)."""
    sfx, P, K = _sfx(a)
    getattr(lib(), f"oracle_bps_make_successor_heavy_{sfx}")(_ptr(a, P), a.size, K(pivot), int(rev))


def partition_bps(a: np.ndarray, pivot: int, B: int = 4096) -> int:
    """In place: the Blocked-Prefix-Sum partition, low-space form
     with blocks of B keys; returns the split.
    Raises if a Reorder swap broke Lemma 3.4."""
    sfx, P, K = _sfx(a)
    S = np.empty(a.size // B + 2, dtype=np.uint64)
    k = int(getattr(lib(), f"oracle_partition_bps_{sfx}")(_ptr(a, P), a.size, K(pivot), B, _ptr(S, U64P)))
    if k == (1 << 64) - 1:
        raise AssertionError("BPS Reorder: a swap target was not a successor of the reordered prefix")
    return k


def quicksort(a: np.ndarray) -> None:
    sfx, P, K = _sfx(a)
    getattr(lib(), f"oracle_quicksort_{sfx}")(_ptr(a, P), a.size)


def prefix_sum(d) -> np.ndarray:
    s = np.ascontiguousarray(np.asarray(d, dtype=np.uint64)).copy()
    lib().oracle_prefix_sum_recursive(_ptr(s, U64P), s.size)
    return s


def ss_groups(a: np.ndarray, base: int, n_lines: int, b: int, g: int, X, pivot: int):
    """Per-group (T_i, vlo_i, vhi_i) of the Smoothed Striding partial partition
    step over the region a[base : base + n_lines*b] (see pp_oracle.c).
    X = the s = ceil(n_lines/g) random chunk offsets in {0..g-1} (an input)."""
    sfx, P, K = _sfx(a)
    assert base + n_lines * b <= a.size
    X = np.ascontiguousarray(np.asarray(X, dtype=np.uint64))
    assert X.size >= (n_lines + g - 1) // g
    T = np.zeros(g, dtype=np.uint64)
    vlo = np.zeros(g, dtype=np.uint64)
    vhi = np.zeros(g, dtype=np.uint64)
    getattr(lib(), f"oracle_ss_groups_{sfx}")(_ptr(a, P), base, n_lines, b, g, _ptr(X, U64P), K(pivot),
                                             _ptr(T, U64P), _ptr(vlo, U64P), _ptr(vhi, U64P))
    return T, vlo, vhi


# ----------------------------------------------------------------------------
# Checkers, comparing a candidate output with the
# oracle's own result on the same input.
# ----------------------------------------------------------------------------

def check_partition(inp: np.ndarray, out: np.ndarray, pivot: int, split: int) -> None:
    """(1) split == oracle count; (2) predicate holds before the split and
    fails after it; (3) per-side sorted contents equal the oracle's sides."""
    K = count(inp, pivot)
    assert split == K, f"split {split} != oracle K {K}"
    assert is_partitioned(out, pivot, split), "predicate violated"
    ref = inp.copy()
    k2 = partition_two_pointer(ref, pivot)
    assert k2 == K
    assert np.array_equal(np.sort(out[:K]), np.sort(ref[:K])), "true-side multiset differs"
    assert np.array_equal(np.sort(out[K:]), np.sort(ref[K:])), "false-side multiset differs"
