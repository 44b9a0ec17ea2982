"""Helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

SIGN64 = -(1 << 63)


def to_dev(a: np.ndarray, dev="cuda") -> torch.Tensor:
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64).copy()).to(dev)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32).copy()).to(dev)
    raise TypeError(a.dtype)


def to_host(t: torch.Tensor, dtype) -> np.ndarray:
    a = t.cpu().numpy()
    return a.view(dtype)


def order_key(t: torch.Tensor) -> torch.Tensor:
    """Order-preserving int64 image of unsigned keys stored as int64/int32 bits."""
    if t.dtype == torch.int64:
        return t ^ SIGN64
    if t.dtype == torch.int32:
        return t.to(torch.int64) & 0xFFFFFFFF
    raise TypeError(t.dtype)


def order_pivot(p: int, dtype) -> int:
    if dtype == torch.int64:
        return p - (1 << 63)
    return p


def check_partition_host(inp: np.ndarray, out_t: torch.Tensor, pivot: int, split: int) -> None:
    """Exact checks (1)-(3) against the oracle on the host (small/medium n)."""
    out = to_host(out_t, inp.dtype)
    oracle.check_partition(inp, out, pivot, split)


def check_partition_device(inp_t: torch.Tensor, out_t: torch.Tensor, pivot: int, split: int,
                           K_oracle: int) -> None:
    """Full-size checks: (1) split == oracle K; (2) predicate on every position
    (device compare); (3) per-side multiset: the true side of the output equals
    the input's keys < pivot (as sorted multisets), same for the false side --
    sorting by torch.sort (library routine)."""
    assert split == K_oracle, f"split {split} != oracle {K_oracle}"
    ko = order_key(out_t)
    pv = order_pivot(pivot, out_t.dtype)
    assert bool((ko[:split] < pv).all()), "predicate fails left of split"
    assert bool((ko[split:] >= pv).all()), "predicate holds right of split"
    ki = order_key(inp_t)
    mask = ki < pv
    a = torch.sort(ki[mask]).values
    b = torch.sort(ko[:split]).values
    assert torch.equal(a, b), "true-side multiset differs"
    del a, b
    a = torch.sort(ki[~mask]).values
    b = torch.sort(ko[split:]).values
    assert torch.equal(a, b), "false-side multiset differs"
