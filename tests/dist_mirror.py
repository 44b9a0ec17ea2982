"""TEST MIRROR (test infrastructure, not the product path) of the multi-GPU
in-place partition of one array sharded contiguously over ranks (BASELINE
config 3).  The product path is the C ABI
(pp_partition_dist_* / pp_quicksort_dist_*, csrc/pp_dist.cu); this is an
independent Python re-statement of its exchange plan and round schedule,
cross-checked against the C plan and run over torch.distributed (gloo) with
oracle local steps in tests/test_dist.py.

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


def p2p_pieces(ns: List[int], ts: List[int], rank: int):
    """The one-sided exchange share of `rank` (mirror of the C
    pp_dist_p2p_pieces): every matched run of the plan is swapped in place
    by the two ranks holding it -- the left rank (misplaced successors)
    takes the first ceil(len/2) pairs, the right rank the rest.  Rows of
    (rank_a, a, rank_b, b, len) in global positions."""
    _, plan = exchange_plan(ns, ts)
    out = []
    for tr in plan:
        h = (tr.length + 1) // 2
        if tr.rank_f == rank:
            out.append((tr.rank_f, tr.f, tr.rank_t, tr.t, h))
        if tr.rank_t == rank and tr.length > h:
            out.append((tr.rank_f, tr.f + h, tr.rank_t, tr.t + h, tr.length - h))
    return out


def chunk_bounds(n: int, C: int):
    """The C chunks [lo, hi) of an n-key shard under dist_overlap: length
    L = ceil(n / C) rounded up to a multiple of 64 (>= 64); the last chunks
    may be short or empty."""
    L = max(64, (-(-n // C) + 63) // 64 * 64) if n else 64
    return [(min(n, k * L), min(n, (k + 1) * L)) for k in range(C)]


def overlap_plan(ns: List[int], chunk_ts: List[List[int]], C: int):
    """Mirror of the count-first overlapped exchange (param dist_overlap):
    every chunk of every rank is one unit of `exchange_plan` (a chunk
    partitioned in place holds its predecessors first, exactly like a shard),
    and a matched run between chunk c of one rank and chunk c' of another can
    move once both are partitioned, i.e. at step max(c, c').  Unlike whole
    shards, two chunks of ONE rank (the rank holding K) can be matched: such
    a run is a local swap.  Returns
    (K, steps): steps[k] = [(rank_f, f_local, rank_t, t_local, len, c_f, c_t)]."""
    P = len(ns)
    units_n, units_t, owner = [], [], []
    for r in range(P):
        for k, (lo, hi) in enumerate(chunk_bounds(ns[r], C)):
            units_n.append(hi - lo)
            units_t.append(chunk_ts[r][k])
            owner.append((r, k))
    K, plan = exchange_plan(units_n, units_t)
    base = [0] * P
    for r in range(1, P):
        base[r] = base[r - 1] + ns[r - 1]
    steps = [[] for _ in range(C)]
    for tr in plan:
        (ra, ca), (rb, cb) = owner[tr.rank_f], owner[tr.rank_t]
        steps[max(ca, cb)].append((ra, tr.f - base[ra], rb, tr.t - base[rb], tr.length, ca, cb))
    return K, steps


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
            raise ValueError("the mirror needs an injected local_partition (tests use the oracle)")
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

    # ------------------------------------------------------------------
    # Distributed quicksort (BASELINE config 5 at P GPUs).
    # ------------------------------------------------------------------
    def sort(self, shard, local_sort: Optional[Callable] = None, small: int = 1 << 16) -> None:
        """Sort the global array (shards in rank order) ascending, unsigned.

        Segments spanning several ranks are split by the distributed
        partition (median-of-3 pivot from the three owning ranks, the x <= p
        progress step when the pivot is the minimum -- DESIGN.md reading
        R14); spanning segments of <= `small` keys are gathered to every
        participating rank, sorted there and each rank keeps its part.  Once
        no segment spans two ranks, every shard is a concatenation of whole
        segments in key order, so one local sort per rank finishes the job."""
        torch, dist = self.torch, self.dist
        if local_sort is None:
            raise ValueError("the mirror needs an injected local_sort (tests use the oracle)")
        bits = 64 if shard.element_size() == 8 else 32
        umask = (1 << bits) - 1
        n_me = torch.tensor([shard.numel()], dtype=torch.int64, device=self.device)
        alln = [torch.empty_like(n_me) for _ in range(self.world)]
        dist.all_gather(alln, n_me, group=self.group)
        ns = [int(v.item()) for v in alln]
        base = [0] * self.world
        for r in range(1, self.world):
            base[r] = base[r - 1] + ns[r - 1]
        N = sum(ns)
        me, b0 = self.rank, base[self.rank]

        def owner(x):
            r = 0
            while r + 1 < self.world and base[r + 1] <= x:
                r += 1
            return r

        def spans(lo, hi):
            return owner(lo) != owner(hi - 1)

        def piece(lo, hi):  # my local slice of global [lo, hi)
            a, b = max(lo, b0), min(hi, b0 + ns[me])
            return (a - b0, b - b0) if a < b else (0, 0)

        def values_at(positions):
            """Unsigned key values at global positions (allgather; each rank
            fills the positions it owns)."""
            mine = torch.zeros(2 * len(positions), dtype=torch.int64, device=self.device)
            for i, x in enumerate(positions):
                if b0 <= x < b0 + ns[me]:
                    mine[2 * i] = 1
                    mine[2 * i + 1] = shard[x - b0].to(torch.int64)
            allv = [torch.empty_like(mine) for _ in range(self.world)]
            dist.all_gather(allv, mine, group=self.group)
            out = []
            for i in range(len(positions)):
                for v in allv:
                    if int(v[2 * i]) == 1:
                        out.append(int(v[2 * i + 1]) & umask)
                        break
            return out

        segs = [(0, N)] if N > 1 else []
        while True:
            span = [s for s in segs if s[1] - s[0] > 1 and spans(*s)]
            if not span:
                break
            nxt = []
            for lo, hi in span:
                if hi - lo <= small:
                    self._gather_sort(shard, lo, hi, piece, ns, base, local_sort)
                    continue
                a, b, c = values_at([lo, lo + (hi - lo - 1) // 2, hi - 1])
                p = sorted([a, b, c])[1]
                pa, pb = piece(lo, hi)
                k = self.partition(shard[pa:pb], p)
                if k == 0:  # p is the segment minimum: split by x <= p
                    if p == umask:
                        continue  # all keys equal the maximum
                    k = self.partition(shard[pa:pb], p + 1)
                    nxt.append((lo + k, hi))  # [lo, lo+k) all equal p
                else:
                    nxt += [(lo, lo + k), (lo + k, hi)]
            segs = [s for s in nxt if s[1] - s[0] > 1]
        if shard.numel() > 1:
            local_sort(shard)

    def _gather_sort(self, shard, lo, hi, piece, ns, base, local_sort):
        """All ranks gather the (small) spanning segment, sort it, and each
        keeps its own part."""
        torch, dist = self.torch, self.dist
        lens = [max(0, min(hi, base[r] + ns[r]) - max(lo, base[r])) for r in range(self.world)]
        mx = max(lens)
        pa, pb = piece(lo, hi)
        buf = torch.zeros(mx, dtype=shard.dtype, device=shard.device)
        buf[: pb - pa] = shard[pa:pb]
        allv = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(allv, buf, group=self.group)
        full = torch.cat([v[:l] for v, l in zip(allv, lens)])
        local_sort(full)
        off = sum(lens[: self.rank])
        shard[pa:pb] = full[off:off + (pb - pa)]
