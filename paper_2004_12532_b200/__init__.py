"""B200-native in-place parallel partition and quicksort (arxiv 2004.12532).

Thin Python binding over the C ABI in ``include/pp.h`` (``libpp.so``, built
in-tree by ``_build.py``).  Argument marshalling only: every step of the
partition / quicksort runs in the library's CUDA kernels.  There is no CPU
fallback: if ``libpp.so`` is missing or fails to load, every call raises.

Function names mirror the C ABI:

    pp_partition_u64(keys, pivot) -> split        (keys: CUDA int64/uint64 tensor)
    pp_partition_u32(keys, pivot) -> split        (keys: CUDA int32/uint32 tensor)
    pp_partition_async_u64/u32(keys, pivot, d_split)
    pp_quicksort_u64/u32(keys)
    pp_partition_host_u64/u32(np_array, pivot) -> split   (host buffers)
    pp_quicksort_host_u64(np_array)
    pp_partition(keys, pivot) / pp_quicksort(keys)         (dtype dispatch)
    pp_partition_stable(keys_in, keys_out, pivot) -> split (Standard Algorithm, out of place)
    pp_partition_bps(keys, pivot) -> split           (Blocked-Prefix-Sum, low-space form)
    pp_ss_groups(keys, pivot, g=0) -> (T, vlo, vhi, info)

int64/int32 tensors are treated as their unsigned bit patterns (torch lacks
most uint64 ops); pivots are Python ints in the unsigned range.
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
# PP_LIB_PATH: load another build of the library (A/B timing in tools/ only)
LIB_PATH = os.environ.get("PP_LIB_PATH") or os.path.join(_PKG, "libpp.so")
HEADER = os.path.join(_ROOT, "include", "pp.h")

PP_OK = 0
STATUS = {0: "PP_OK", 1: "PP_E_INVAL", 2: "PP_E_CUDA", 3: "PP_E_NOMEM", 4: "PP_E_NCCL", 5: "PP_E_INTERNAL"}

_lib = None


class PPError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def load(build_if_missing: bool = True):
    """Load libpp.so (building it in-tree first if it is missing/stale and
    nvcc is available).  Raises if the library cannot be loaded."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        from . import _build
        if not _build.up_to_date():
            try:
                _build.build()
            except Exception as e:  # no nvcc: only acceptable if a built .so exists
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(f"libpp.so missing and build failed: {e}") from e
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libpp.so not found at {LIB_PATH}; run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    u64, u32, vp, i64 = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int64
    P64 = ctypes.POINTER(ctypes.c_uint64)
    st = ctypes.c_int
    sig = {
        "pp_partition_u64": ([vp, u64, u64, vp, P64], st),
        "pp_partition_u32": ([vp, u64, u32, vp, P64], st),
        "pp_partition_async_u64": ([vp, u64, u64, vp, vp], st),
        "pp_partition_async_u32": ([vp, u64, u32, vp, vp], st),
        "pp_quicksort_u64": ([vp, u64, vp], st),
        "pp_quicksort_u32": ([vp, u64, vp], st),
        "pp_partition_host_u64": ([vp, u64, u64, P64], st),
        "pp_reset_params": ([], None),
        "pp_swap_ranges_u64": ([vp, u64, vp], st),
        "pp_swap_ranges_u32": ([vp, u64, vp], st),
        "pp_partition_stable_u64": ([vp, vp, u64, u64, vp, P64], st),
        "pp_partition_bps_u64": ([vp, u64, u64, vp, P64], st),
        "pp_partition_bps_u32": ([vp, u64, u32, vp, P64], st),
        "pp_partition_bps_async_u64": ([vp, u64, u64, vp, vp], st),
        "pp_partition_stable_u32": ([vp, vp, u64, u32, vp, P64], st),
        "pp_partition_stable_inplace_u64": ([vp, u64, u64, vp, P64], st),
        "pp_partition_stable_inplace_u32": ([vp, u64, u32, vp, P64], st),
        "pp_partition_stable_async_u64": ([vp, vp, u64, u64, vp, vp], st),
        "pp_partition_host_u32": ([vp, u64, u32, P64], st),
        "pp_quicksort_host_u64": ([vp, u64], st),
        "pp_partition": ([vp, u64, u64], u64),
        "pp_quicksort": ([vp, u64], st),
        "pp_ss_groups_u64": ([vp, u64, u64, u64, vp, P64, P64, P64, P64], st),
        "pp_ss_groups_u32": ([vp, u64, u32, u64, vp, P64, P64, P64, P64], st),
        "pp_max_groups": ([], u64),
        "pp_workspace_bytes": ([u64, ctypes.c_int, ctypes.c_int], u64),
        "pp_last_aux_bytes": ([], u64),
        "pp_set_workspace": ([ctypes.c_void_p, u64], st),
        "pp_last_stats": ([P64], st),
        "pp_set_param": ([ctypes.c_char_p, i64], st),
        "pp_get_param": ([ctypes.c_char_p], i64),
        "pp_status_string": ([st], ctypes.c_char_p),
        "pp_last_error": ([], ctypes.c_char_p),
        "pp_launch_count": ([ctypes.c_int], u64),
        "pp_timing": ([ctypes.c_int], None),
        "pp_timing_read": ([ctypes.POINTER(ctypes.c_double)], st),
        "pp_dist_unique_id": ([vp], st),
        "pp_dist_init": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int], st),
        "pp_partition_dist_u64": ([vp, u64, u64, vp, P64], st),
        "pp_partition_dist_u32": ([vp, u64, u32, vp, P64], st),
        "pp_dist_set_staging": ([u64], st),
        "pp_quicksort_dist_u64": ([vp, u64, vp], st),
        "pp_quicksort_dist_u32": ([vp, u64, vp], st),
        "pp_dist_plan": ([P64, P64, ctypes.c_int, u64, P64, u64, P64, P64], st),
        "pp_dist_finalize": ([], st),
        "pp_dist_p2p_pieces": ([P64, P64, ctypes.c_int, ctypes.c_int, P64, u64, P64], st),
        "pp_ipc_export": ([vp, vp, P64], st),
        "pp_ipc_import": ([vp, u64, ctypes.POINTER(ctypes.c_void_p)], st),
        "pp_ipc_close_all": ([], st),
        "pp_dist_last_timing": ([ctypes.POINTER(ctypes.c_double)], st),
        "pp_quicksort_last_stats": ([P64], st),
        "pp_audit_set": ([vp, vp, u64, ctypes.c_int], st),
        "pp_partition_dist_loopback_u64": ([vp, P64, ctypes.c_int, u64, P64], st),
        "pp_partition_dist_loopback_u32": ([vp, P64, ctypes.c_int, u32, P64], st),
        "pp_quicksort_dist_loopback_u64": ([vp, P64, ctypes.c_int], st),
        "pp_quicksort_dist_loopback_u32": ([vp, P64, ctypes.c_int], st),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("PP_LIB_PATH") and not hasattr(L, name):
            continue  # an older build loaded for an A/B comparison (tools/ only)
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(pp_[a-z0-9_]+)\s*\(", txt)))


def _check(status: int, where: str):
    if status != PP_OK:
        raise PPError(status, where, load().pp_last_error().decode())


def _stream_ptr(stream=None, device=None) -> int:
    """The stream the call is enqueued on: the given one, else the current
    stream of the keys' device (not of the current device)."""
    import torch
    if stream is not None:
        return stream.cuda_stream
    return torch.cuda.current_stream(device).cuda_stream


def _split_word(d_split, keys) -> int:
    """Device address of the 8-byte split word of the async variants."""
    import torch
    if not d_split.is_cuda or d_split.device != keys.device:
        raise ValueError("d_split must be a CUDA tensor on the keys' device")
    if d_split.dtype not in (torch.int64, torch.uint64) or d_split.numel() < 1:
        raise TypeError("d_split must hold at least one int64/uint64 word")
    return d_split.data_ptr()


def _key_kind(t) -> str:
    import torch
    if not t.is_cuda:
        raise ValueError("keys must be a CUDA tensor (use pp_partition_host_* for host arrays)")
    if not t.is_contiguous():
        raise ValueError("keys must be contiguous")
    if t.dtype in (torch.int64, torch.uint64):
        return "u64"
    if t.dtype in (torch.int32, torch.uint32):
        return "u32"
    raise TypeError(f"unsupported key dtype {t.dtype}")


def _pivot(p: int, kind: str) -> int:
    p = int(p)
    hi = (1 << 64) if kind == "u64" else (1 << 32)
    if not 0 <= p < hi:
        raise ValueError(f"pivot {p} out of range for {kind}")
    return p


def pp_partition_u64(keys, pivot: int, stream=None) -> int:
    assert _key_kind(keys) == "u64"
    out = ctypes.c_uint64(0)
    _check(load().pp_partition_u64(keys.data_ptr(), keys.numel(), _pivot(pivot, "u64"), _stream_ptr(stream, keys.device),
                                   ctypes.byref(out)), "pp_partition_u64")
    return int(out.value)


def pp_partition_u32(keys, pivot: int, stream=None) -> int:
    assert _key_kind(keys) == "u32"
    out = ctypes.c_uint64(0)
    _check(load().pp_partition_u32(keys.data_ptr(), keys.numel(), _pivot(pivot, "u32"), _stream_ptr(stream, keys.device),
                                   ctypes.byref(out)), "pp_partition_u32")
    return int(out.value)


def pp_partition_async_u64(keys, pivot: int, d_split, stream=None) -> None:
    assert _key_kind(keys) == "u64"
    _check(load().pp_partition_async_u64(keys.data_ptr(), keys.numel(), _pivot(pivot, "u64"),
                                         _stream_ptr(stream, keys.device), _split_word(d_split, keys)),
           "pp_partition_async_u64")


def pp_partition_async_u32(keys, pivot: int, d_split, stream=None) -> None:
    assert _key_kind(keys) == "u32"
    _check(load().pp_partition_async_u32(keys.data_ptr(), keys.numel(), _pivot(pivot, "u32"),
                                         _stream_ptr(stream, keys.device), _split_word(d_split, keys)),
           "pp_partition_async_u32")


def pp_quicksort_u64(keys, stream=None) -> None:
    assert _key_kind(keys) == "u64"
    _check(load().pp_quicksort_u64(keys.data_ptr(), keys.numel(), _stream_ptr(stream, keys.device)), "pp_quicksort_u64")


def pp_quicksort_u32(keys, stream=None) -> None:
    assert _key_kind(keys) == "u32"
    _check(load().pp_quicksort_u32(keys.data_ptr(), keys.numel(), _stream_ptr(stream, keys.device)), "pp_quicksort_u32")


def pp_partition_bps(keys, pivot: int, stream=None) -> int:
    """The paper's Blocked-Prefix-Sum partition, low-space form
    (PAPER.md:319-478, 1466-1486), in place; returns the split."""
    kind = _key_kind(keys)
    out = ctypes.c_uint64(0)
    f = load().pp_partition_bps_u64 if kind == "u64" else load().pp_partition_bps_u32
    _check(f(keys.data_ptr(), keys.numel(), _pivot(pivot, kind), _stream_ptr(stream, keys.device), ctypes.byref(out)),
           "pp_partition_bps")
    return int(out.value)


def pp_partition_bps_async_u64(keys, pivot: int, d_split, stream=None) -> None:
    assert _key_kind(keys) == "u64"
    _check(load().pp_partition_bps_async_u64(keys.data_ptr(), keys.numel(), _pivot(pivot, "u64"),
                                             _stream_ptr(stream, keys.device), _split_word(d_split, keys)),
           "pp_partition_bps_async_u64")


def pp_partition_stable(keys_in, keys_out, pivot: int, stream=None) -> int:
    """The Standard Algorithm: stable, out of place;
    keys_out receives the partition of keys_in; returns the split."""
    kind = _key_kind(keys_in)
    assert _key_kind(keys_out) == kind and keys_out.numel() == keys_in.numel()
    out = ctypes.c_uint64(0)
    f = load().pp_partition_stable_u64 if kind == "u64" else load().pp_partition_stable_u32
    _check(f(keys_in.data_ptr(), keys_out.data_ptr(), keys_in.numel(), _pivot(pivot, kind), _stream_ptr(stream, keys_in.device),
             ctypes.byref(out)), "pp_partition_stable")
    return int(out.value)


def pp_partition_stable_inplace(keys, pivot: int, stream=None) -> int:
    """Stable partition IN PLACE (tile partitions + rotation merges,
    O(n log n) work): the Standard Algorithm's output; returns the split."""
    kind = _key_kind(keys)
    out = ctypes.c_uint64(0)
    f = load().pp_partition_stable_inplace_u64 if kind == "u64" else load().pp_partition_stable_inplace_u32
    _check(f(keys.data_ptr(), keys.numel(), _pivot(pivot, kind), _stream_ptr(stream, keys.device), ctypes.byref(out)),
           "pp_partition_stable_inplace")
    return int(out.value)


def pp_partition_stable_async_u64(keys_in, keys_out, pivot: int, d_split, stream=None) -> None:
    assert _key_kind(keys_in) == "u64" and _key_kind(keys_out) == "u64"
    _check(load().pp_partition_stable_async_u64(keys_in.data_ptr(), keys_out.data_ptr(), keys_in.numel(),
                                                _pivot(pivot, "u64"), _stream_ptr(stream, keys_in.device),
                                                _split_word(d_split, keys_in)),
           "pp_partition_stable_async_u64")


def pp_partition(keys, pivot: int, stream=None) -> int:
    return (pp_partition_u64 if _key_kind(keys) == "u64" else pp_partition_u32)(keys, pivot, stream)


def pp_quicksort(keys, stream=None) -> None:
    (pp_quicksort_u64 if _key_kind(keys) == "u64" else pp_quicksort_u32)(keys, stream)


def pp_partition_host_u64(a: np.ndarray, pivot: int) -> int:
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    out = ctypes.c_uint64(0)
    _check(load().pp_partition_host_u64(a.ctypes.data, a.size, _pivot(pivot, "u64"), ctypes.byref(out)),
           "pp_partition_host_u64")
    return int(out.value)


def pp_partition_host_u32(a: np.ndarray, pivot: int) -> int:
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    out = ctypes.c_uint64(0)
    _check(load().pp_partition_host_u32(a.ctypes.data, a.size, _pivot(pivot, "u32"), ctypes.byref(out)),
           "pp_partition_host_u32")
    return int(out.value)


def pp_quicksort_host_u64(a: np.ndarray) -> None:
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    _check(load().pp_quicksort_host_u64(a.ctypes.data, a.size), "pp_quicksort_host_u64")


def pp_ss_groups(keys, pivot: int, g: int = 0, stream=None):
    """Run only the Smoothed Striding partial partition step; returns numpy
    (T, vlo, vhi) per group and info = {g, head, n_lines, line_keys, seed}."""
    kind = _key_kind(keys)
    L = load()
    cap = max(int(g), int(L.pp_max_groups()), 1)
    T = np.zeros(cap, dtype=np.uint64)
    vlo = np.zeros(cap, dtype=np.uint64)
    vhi = np.zeros(cap, dtype=np.uint64)
    info = np.zeros(6, dtype=np.uint64)
    P = ctypes.POINTER(ctypes.c_uint64)
    f = L.pp_ss_groups_u64 if kind == "u64" else L.pp_ss_groups_u32
    _check(f(keys.data_ptr(), keys.numel(), _pivot(pivot, kind), int(g), _stream_ptr(stream, keys.device),
             T.ctypes.data_as(P), vlo.ctypes.data_as(P), vhi.ctypes.data_as(P), info.ctypes.data_as(P)),
           "pp_ss_groups")
    gg = int(info[0])
    return T[:gg], vlo[:gg], vhi[:gg], {"g": gg, "head": int(info[1]), "n_lines": int(info[2]),
                                        "line_keys": int(info[3]), "seed": int(info[4])}


STAT_KEYS = ("n", "K", "W", "vmin", "vmax", "M", "g", "line_keys", "n_lines", "head", "aux_bytes", "path",
             "nTasks")


def pp_last_stats() -> dict:
    out = (ctypes.c_uint64 * 13)()
    _check(load().pp_last_stats(out), "pp_last_stats")
    return dict(zip(STAT_KEYS, [int(v) for v in out]))


QS_STAT_KEYS = ("n", "levels", "level_keys", "small_keys", "leaf_keys", "nsmall")


def pp_audit_set(shadow, keys=None) -> None:
    """EREW shadow-writer audit (libpp_audit.so only, include/pp.h): `shadow`
    is a zeroed int32 tensor with one counter per key of `keys` (same
    device); None switches the audit off."""
    import torch
    if shadow is None:
        _check(load().pp_audit_set(None, None, 0, 0), "pp_audit_set")
        return
    assert shadow.dtype == torch.int32 and shadow.numel() == keys.numel() and shadow.device == keys.device
    _check(load().pp_audit_set(shadow.data_ptr(), keys.data_ptr(), keys.numel(), keys.element_size()),
           "pp_audit_set")


def pp_quicksort_last_stats() -> dict:
    """Work statistics of the last quicksort (include/pp.h)."""
    out = (ctypes.c_uint64 * 6)()
    _check(load().pp_quicksort_last_stats(out), "pp_quicksort_last_stats")
    return dict(zip(QS_STAT_KEYS, [int(v) for v in out]))


def pp_set_param(name: str, value: int) -> None:
    _check(load().pp_set_param(name.encode(), int(value)), "pp_set_param")


def pp_get_param(name: str) -> int:
    return int(load().pp_get_param(name.encode()))


def pp_last_aux_bytes() -> int:
    return int(load().pp_last_aux_bytes())


def pp_workspace_bytes(n: int, key_bytes: int = 8, op: int = 0) -> int:
    return int(load().pp_workspace_bytes(n, key_bytes, op))


def pp_set_workspace(ws) -> None:
    """Use a caller-owned device buffer (a CUDA tensor, 256-B aligned) as the
    library workspace; None reverts to the internal one (pp.h)."""
    if ws is None:
        _check(load().pp_set_workspace(None, 0), "pp_set_workspace")
    else:
        _check(load().pp_set_workspace(ws.data_ptr(), ws.numel() * ws.element_size()), "pp_set_workspace")


def pp_launch_count(reset: bool = False) -> int:
    return int(load().pp_launch_count(1 if reset else 0))


def pp_dist_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().pp_dist_unique_id(buf), "pp_dist_unique_id")
    return buf.raw


def pp_dist_init(unique_id: bytes, nranks: int, rank: int, device: int) -> None:
    assert len(unique_id) == 128
    buf = ctypes.create_string_buffer(unique_id, 128)
    _check(load().pp_dist_init(buf, nranks, rank, device), "pp_dist_init")


def pp_partition_dist(shard, pivot: int, stream=None) -> int:
    """Global partition of a sharded array (collective; see include/pp.h)."""
    kind = _key_kind(shard)
    out = ctypes.c_uint64(0)
    f = load().pp_partition_dist_u64 if kind == "u64" else load().pp_partition_dist_u32
    _check(f(shard.data_ptr(), shard.numel(), _pivot(pivot, kind), _stream_ptr(stream, shard.device), ctypes.byref(out)),
           "pp_partition_dist")
    return int(out.value)


def pp_quicksort_dist(shard, stream=None) -> None:
    """Global sort of a sharded array (collective; see include/pp.h)."""
    kind = _key_kind(shard)
    f = load().pp_quicksort_dist_u64 if kind == "u64" else load().pp_quicksort_dist_u32
    _check(f(shard.data_ptr(), shard.numel(), _stream_ptr(stream, shard.device)), "pp_quicksort_dist")


def _shard_sizes(keys, ns):
    a = np.ascontiguousarray(np.asarray(ns, dtype=np.uint64))
    if int(a.sum()) != keys.numel():
        raise ValueError(f"shard sizes sum to {int(a.sum())}, keys has {keys.numel()}")
    return a


def pp_partition_dist_loopback(keys, ns, pivot: int) -> int:
    """The distributed partition with len(ns) emulated ranks on this GPU
    (rank r owns keys[sum(ns[:r]) : + ns[r]]); returns the global split."""
    kind = _key_kind(keys)
    a = _shard_sizes(keys, ns)
    out = ctypes.c_uint64(0)
    P64 = ctypes.POINTER(ctypes.c_uint64)
    f = load().pp_partition_dist_loopback_u64 if kind == "u64" else load().pp_partition_dist_loopback_u32
    _check(f(keys.data_ptr(), a.ctypes.data_as(P64), len(a), _pivot(pivot, kind), ctypes.byref(out)),
           "pp_partition_dist_loopback")
    return int(out.value)


def pp_quicksort_dist_loopback(keys, ns) -> None:
    """The distributed quicksort with len(ns) emulated ranks on this GPU."""
    kind = _key_kind(keys)
    a = _shard_sizes(keys, ns)
    P64 = ctypes.POINTER(ctypes.c_uint64)
    f = load().pp_quicksort_dist_loopback_u64 if kind == "u64" else load().pp_quicksort_dist_loopback_u32
    _check(f(keys.data_ptr(), a.ctypes.data_as(P64), len(a)), "pp_quicksort_dist_loopback")


def pp_dist_set_staging(nbytes: int) -> None:
    _check(load().pp_dist_set_staging(int(nbytes)), "pp_dist_set_staging")


def pp_dist_finalize() -> None:
    _check(load().pp_dist_finalize(), "pp_dist_finalize")


def pp_dist_plan(ns, ts, cap: int):
    """The exchange plan (host arithmetic): (K, rows) with rows of
    (round, rank_f, f, rank_t, t, len)."""
    P = len(ns)
    a = np.ascontiguousarray(np.asarray(ns, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(ts, dtype=np.uint64))
    P64 = ctypes.POINTER(ctypes.c_uint64)
    n_out = ctypes.c_uint64(0)
    K = ctypes.c_uint64(0)
    _check(load().pp_dist_plan(a.ctypes.data_as(P64), b.ctypes.data_as(P64), P, int(cap), None, 0,
                               ctypes.byref(n_out), ctypes.byref(K)), "pp_dist_plan")
    rows = np.zeros((max(1, n_out.value), 6), dtype=np.uint64)
    _check(load().pp_dist_plan(a.ctypes.data_as(P64), b.ctypes.data_as(P64), P, int(cap),
                               rows.ctypes.data_as(P64), n_out.value, ctypes.byref(n_out), ctypes.byref(K)),
           "pp_dist_plan")
    return int(K.value), [tuple(int(x) for x in r) for r in rows[: n_out.value]]


def pp_dist_p2p_pieces(ns, ts, rank: int):
    """The share of `rank` in the one-sided exchange (host arithmetic): rows
    of (rank_a, a, rank_b, b, len), global positions."""
    P = len(ns)
    a = np.ascontiguousarray(np.asarray(ns, dtype=np.uint64))
    b = np.ascontiguousarray(np.asarray(ts, dtype=np.uint64))
    P64 = ctypes.POINTER(ctypes.c_uint64)
    n_out = ctypes.c_uint64(0)
    _check(load().pp_dist_p2p_pieces(a.ctypes.data_as(P64), b.ctypes.data_as(P64), P, int(rank), None, 0,
                                     ctypes.byref(n_out)), "pp_dist_p2p_pieces")
    rows = np.zeros((max(1, n_out.value), 5), dtype=np.uint64)
    _check(load().pp_dist_p2p_pieces(a.ctypes.data_as(P64), b.ctypes.data_as(P64), P, int(rank),
                                     rows.ctypes.data_as(P64), n_out.value, ctypes.byref(n_out)),
           "pp_dist_p2p_pieces")
    return [tuple(int(x) for x in r) for r in rows[: n_out.value]]


def pp_ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64(0)
    _check(load().pp_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "pp_ipc_export")
    return h.raw, int(off.value)


def pp_ipc_import(handle: bytes, offset: int) -> int:
    """Maps an exported range in this process; returns its device address."""
    h = ctypes.create_string_buffer(bytes(handle), 64)
    out = ctypes.c_void_p(0)
    _check(load().pp_ipc_import(h, int(offset), ctypes.byref(out)), "pp_ipc_import")
    return int(out.value or 0)


def pp_dist_last_timing() -> dict:
    """Phases of this rank's last pp_partition_dist call (device events)."""
    a = (ctypes.c_double * 4)()
    _check(load().pp_dist_last_timing(a), "pp_dist_last_timing")
    return {"local_ms": a[0], "gather_ms": a[1], "exchange_ms": a[2], "bytes": int(a[3])}


def pp_ipc_close_all() -> None:
    _check(load().pp_ipc_close_all(), "pp_ipc_close_all")


def pp_swap_ranges(pieces, key_bytes: int = 8, stream=None) -> None:
    """Swap [a, a+len) <-> [b, b+len) for each (a, b, len) of device
    addresses (the staging-free exchange primitive)."""
    tri = np.ascontiguousarray(np.asarray(pieces, dtype=np.uint64).reshape(-1, 3))
    f = load().pp_swap_ranges_u64 if key_bytes == 8 else load().pp_swap_ranges_u32
    _check(f(tri.ctypes.data, tri.shape[0], _stream_ptr(stream, None)), "pp_swap_ranges")


def pp_timing(enable: bool) -> None:
    load().pp_timing(1 if enable else 0)


def pp_timing_read() -> dict:
    out = (ctypes.c_double * 4)()
    _check(load().pp_timing_read(out), "pp_timing_read")
    return {"calls": int(out[0]), "group_ms": out[1], "rest_ms": out[2], "total_ms": out[3]}


def reset_params() -> None:
    """Every tunable back to the library's default (C ABI pp_reset_params)."""
    load().pp_reset_params()
