"""Multi-GPU in-place partition of one array sharded contiguously over ranks
(BASELINE config 3).

One process per GPU.  Rank r holds the contiguous shard A[β_r, β_r + n_r) of
the global array.  A global partition needs exactly one exchange step:

1. every rank partitions its shard in place with the library
   (`pp_partition_*`), giving t_r keys < pivot at its front;
2. an allgather of (n_r, t_r, pivot) gives every rank K = Σ t_r and the same
   exchange plan (pure host arithmetic, `exchange_plan`);
3. misplaced successors left of K (the range [β_r + t_r, min(K, β_r + n_r)) of
   each rank left of K) are paired, in global order, with misplaced
   predecessors right of K ([max(K, β_r), β_r + t_r) of each rank right of
   K); each matched pair of ranges is swapped by a send/recv between the two
   owners (NCCL over NVLink, or gloo in the CPU tests) through a bounded
   staging buffer, in rounds.

A rank never has both kinds of misplaced keys (that would need
β_r + t_r < K < β_r + t_r), so every swap crosses two different ranks.  The
plan is deterministic, so the output is a pure function of the input.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional


@dataclass(frozen=True)
class Transfer:
    """Swap the successors at global [f, f+length) (owned by rank_f) with the
    predecessors at global [t, t+length) (owned by rank_t)."""
    rank_f: int
    f: int
    rank_t: int
    t: int
    length: int


def exchange_plan(ns: List[int], ts: List[int]) -> tuple:
    """(K, transfers) for shard sizes ns and local splits ts (rank order).

    Pairs the i-th misplaced successor (global order) with the i-th misplaced
    predecessor -- a merge of two interval lists."""
    P = len(ns)
    assert len(ts) == P and all(0 <= t <= n for n, t in zip(ns, ts))
    K = sum(ts)
    base = [0] * P
    for r in range(1, P):
        base[r] = base[r - 1] + ns[r - 1]
    F, T = [], []  # (rank, start, end) in global coordinates
    for r in range(P):
        b, n, t = base[r], ns[r], ts[r]
        fs, fe = b + t, min(K, b + n)
        if fs < fe:
            F.append([r, fs, fe])
        ts_, te = max(K, b), b + t
        if ts_ < te:
            T.append([r, ts_, te])
    assert sum(e - s for _, s, e in F) == sum(e - s for _, s, e in T)
    out = []
    i = j = 0
    while i < len(F) and j < len(T):
        rf, fs, fe = F[i]
        rt, ts_, te = T[j]
        m = min(fe - fs, te - ts_)
        out.append(Transfer(rf, fs, rt, ts_, m))
        F[i][1] += m
        T[j][1] += m
        if F[i][1] == fe:
            i += 1
        if T[j][1] == te:
            j += 1
    return K, out


def schedule_rounds(transfers: List[Transfer], world: int, cap: int):
    """Split the plan into pieces of <= cap elements and group them into
    rounds so that no rank receives more than cap elements per round (its
    staging size).  Computed identically on every rank from the global plan,
    so partners always meet in the same round (no cross-round waits, no
    deadlock).  Returns a list of rounds, each a list of Transfer pieces."""
    rounds = [[]]
    used = [0] * world
    for tr in transfers:
        s = 0
        while s < tr.length:
            m = min(cap, tr.length - s)
            if used[tr.rank_f] + m > cap or used[tr.rank_t] + m > cap:
                rounds.append([])
                used = [0] * world
            rounds[-1].append(Transfer(tr.rank_f, tr.f + s, tr.rank_t, tr.t + s, m))
            used[tr.rank_f] += m
            used[tr.rank_t] += m
            s += m
    return [r for r in rounds if r]


def my_ops(pieces: List[Transfer], rank: int, base: int):
    """The (peer, local_offset, length) swaps this rank takes part in."""
    ops = []
    for tr in pieces:
        if tr.rank_f == rank:
            ops.append((tr.rank_t, tr.f - base, tr.length))
        elif tr.rank_t == rank:
            ops.append((tr.rank_f, tr.t - base, tr.length))
    return ops


class Partitioner:
    """Global partition of a sharded array (one rank per GPU).

    `local_partition(shard, pivot) -> t` defaults to the library's CUDA
    partition; the CPU tests inject the oracle (the exchange logic is what
    they test).  `staging_bytes` bounds the receive buffer (o(n) aux)."""

    def __init__(self, device=None, group=None, staging_bytes: int = 256 << 20,
                 local_partition: Optional[Callable] = None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staging_bytes = staging_bytes
        if local_partition is None:
            from . import pp_partition
            local_partition = pp_partition
        self.local_partition = local_partition
        self.last_global_split = None
        self.last_plan = None

    def partition_u64(self, shard, pivot: int) -> int:
        return self.partition(shard, pivot)

    def partition(self, shard, pivot: int) -> int:
        torch, dist = self.torch, self.dist
        t = int(self.local_partition(shard, pivot))
        # allgather (n_r, t_r, pivot) -- pivot as two 32-bit halves so that
        # an int64 tensor can carry any unsigned 64-bit value
        mine = torch.tensor([shard.numel(), t, pivot >> 32, pivot & 0xFFFFFFFF], dtype=torch.int64,
                            device=self.device)
        allv = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allv, mine, group=self.group)
        rows = [v.tolist() for v in allv]
        if any((r[2], r[3]) != (pivot >> 32, pivot & 0xFFFFFFFF) for r in rows):
            raise ValueError("ranks passed different pivots")
        ns = [r[0] for r in rows]
        ts = [r[1] for r in rows]
        K, plan = exchange_plan(ns, ts)
        base = sum(ns[: self.rank])
        cap = max(1, self.staging_bytes // shard.element_size())
        rounds = schedule_rounds(plan, self.world, cap)
        self._execute(shard, [my_ops(r, self.rank, base) for r in rounds], cap)
        self.last_global_split = K
        self.last_plan = plan
        return K

    def _execute(self, shard, round_ops, cap):
        """Per round: send my misplaced range to the partner and receive the
        partner's range into staging, then copy staging into place (NCCL gives
        no ordering between a send and a receive on the same buffer)."""
        torch, dist = self.torch, self.dist
        need = max((sum(m for _, _, m in ops) for ops in round_ops), default=0)
        if need == 0:
            return
        staging = torch.empty(min(cap, need), dtype=shard.dtype, device=shard.device)
        for ops in round_ops:
            if not ops:
                continue
            p2p, soff, placed = [], 0, []
            for peer, off, m in ops:
                p2p.append(dist.P2POp(dist.isend, shard[off:off + m], peer, group=self.group))
                p2p.append(dist.P2POp(dist.irecv, staging[soff:soff + m], peer, group=self.group))
                placed.append((off, soff, m))
                soff += m
            for req in dist.batch_isend_irecv(p2p):
                req.wait()
            for off, so, m in placed:
                shard[off:off + m].copy_(staging[so:so + m])
