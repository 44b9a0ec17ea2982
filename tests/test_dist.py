"""Multi-GPU exchange step (BASELINE config 3) on CPU: the exchange plan and
its round schedule checked by an in-memory simulator, and the full
Partitioner over torch.distributed with the gloo backend at world sizes 2-4
(the local partition is the oracle here; the CUDA local partition is covered
by the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from dist_mirror import Partitioner, chunk_bounds, exchange_plan, my_ops, overlap_plan, schedule_rounds


def _simulate(shards, pivot):
    """Apply the plan to in-memory shards (each locally partitioned first)."""
    ts = []
    for s in shards:
        ts.append(oracle.partition_two_pointer(s, pivot))
    ns = [s.size for s in shards]
    K, plan = exchange_plan(ns, ts)
    base = np.cumsum([0] + ns[:-1])
    for tr in plan:
        a = shards[tr.rank_f][tr.f - base[tr.rank_f]: tr.f - base[tr.rank_f] + tr.length].copy()
        b = shards[tr.rank_t][tr.t - base[tr.rank_t]: tr.t - base[tr.rank_t] + tr.length].copy()
        shards[tr.rank_f][tr.f - base[tr.rank_f]: tr.f - base[tr.rank_f] + tr.length] = b
        shards[tr.rank_t][tr.t - base[tr.rank_t]: tr.t - base[tr.rank_t] + tr.length] = a
    return K, plan


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16, 64])
def test_plan_simulator(P):
    rng = np.random.default_rng(P)
    for trial in range(20):
        ns = list(rng.integers(0, 2000, size=P))
        if trial % 4 == 0:
            ns = [1000] * P
        glob = rng.integers(0, 100, size=sum(ns)).astype(np.uint64)
        pivot = int(rng.integers(0, 101))
        shards = np.split(glob.copy(), np.cumsum(ns)[:-1])
        K, plan = _simulate(shards, pivot)
        out = np.concatenate(shards) if shards else glob
        oracle.check_partition(glob, out, pivot, K)
        for tr in plan:
            assert tr.rank_f != tr.rank_t and tr.length > 0


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("C", [1, 2, 3, 8])
def test_overlap_plan_simulator(P, C):
    """The count-first overlapped exchange (dist_overlap) by simulation: the
    per-chunk counts fix the plan before any key moves; at step k every rank
    partitions its chunk k, then the runs of step k are swapped -- each touches
    only chunks <= k on both sides (already partitioned, never touched again
    by a local step) -- and the result is the global partition."""
    rng = np.random.default_rng(100 * P + C)
    for trial in range(12):
        ns = [int(x) for x in rng.integers(0, 700, size=P)]
        if trial % 3 == 0:
            ns = [512] * P
        if trial % 4 == 1 and P > 1:
            ns[0] = 0
        glob = rng.integers(0, 50, size=sum(ns)).astype(np.uint64)
        pivot = int(rng.integers(0, 51))
        shards = [x.copy() for x in np.split(glob, np.cumsum(ns)[:-1])] if P > 1 else [glob.copy()]
        bounds = [chunk_bounds(n, C) for n in ns]
        cts = [[oracle.count(shards[r][lo:hi], pivot) for lo, hi in bounds[r]] for r in range(P)]
        K, steps = overlap_plan(ns, cts, C)
        assert K == oracle.count(glob, pivot)
        for k in range(C):
            for r in range(P):
                lo, hi = bounds[r][k]
                assert oracle.partition_two_pointer(shards[r][lo:hi], pivot) == cts[r][k]
            for ra, a, rb, b, ln, ca, cb in steps[k]:
                # a run inside one rank (between two of its chunks) exists only on the rank holding K
                assert (ra != rb or ca != cb) and ln > 0 and max(ca, cb) == k
                assert bounds[ra][ca][0] <= a and a + ln <= bounds[ra][ca][1]
                assert bounds[rb][cb][0] <= b and b + ln <= bounds[rb][cb][1]
                x = shards[ra][a:a + ln].copy()
                shards[ra][a:a + ln] = shards[rb][b:b + ln]
                shards[rb][b:b + ln] = x
        oracle.check_partition(glob, np.concatenate(shards), pivot, K)


def test_plan_adversarial_counts():
    # all predecessors on the last rank, all successors on the first ...
    for ns, ts in (([4, 4, 4], [0, 0, 4]), ([5, 5], [5, 0]), ([3, 0, 7, 1], [0, 0, 7, 1]),
                   ([10, 10, 10, 10], [10, 0, 10, 0]), ([1] * 9, [0, 1] * 4 + [1])):
        K, plan = exchange_plan(ns, ts)
        assert K == sum(ts)
        moved_f = sum(tr.length for tr in plan)
        # misplaced successors left of K
        base, mis = 0, 0
        for n, t in zip(ns, ts):
            mis += max(0, min(K, base + n) - (base + t))
            base += n
        assert moved_f == mis


@pytest.mark.parametrize("cap", [1, 3, 7, 1000])
def test_schedule_rounds_cover_and_cap(cap):
    rng = np.random.default_rng(cap)
    for trial in range(30):
        P = int(rng.integers(2, 9))
        ns = [int(x) for x in rng.integers(0, 50, size=P)]
        ts = [int(rng.integers(0, n + 1)) for n in ns]
        K, plan = exchange_plan(ns, ts)
        rounds = schedule_rounds(plan, P, cap)
        for r in rounds:
            recv = [0] * P
            for tr in r:
                recv[tr.rank_f] += tr.length
                recv[tr.rank_t] += tr.length
            assert max(recv) <= cap
        # pieces cover the plan exactly, in order
        flat = [tr for r in rounds for tr in r]
        assert sum(t.length for t in flat) == sum(t.length for t in plan)
        base = np.cumsum([0] + ns[:-1])
        for rank in range(P):
            ops = [op for r in rounds for op in my_ops(r, rank, int(base[rank]))]
            assert all(0 <= off and off + m <= ns[rank] for _, off, m in ops)


def test_c_plan_matches_python_plan():
    """The C-ABI exchange plan (pp_dist_plan, C++) and the Python plan +
    round schedule (two independent implementations) agree piece by piece."""
    import paper_2004_12532_b200 as pp
    rng = np.random.default_rng(99)
    for trial in range(200):
        P = int(rng.integers(1, 12))
        ns = [int(x) for x in rng.integers(0, 300, size=P)]
        ts = [int(rng.integers(0, n + 1)) for n in ns]
        cap = int(rng.choice([1, 5, 17, 64, 1000]))
        K, plan = exchange_plan(ns, ts)
        rounds = schedule_rounds(plan, P, cap)
        py = [(ri, t.rank_f, t.f, t.rank_t, t.t, t.length) for ri, r in enumerate(rounds) for t in r]
        Kc, rows = pp.pp_dist_plan(ns, ts, cap)
        assert Kc == K
        assert rows == py


def test_p2p_shares_cover_the_plan_once():
    """One-sided exchange: the C share rule (pp_dist_p2p_pieces) equals the
    Python mirror for every rank, the shares of all ranks cover every pair of
    the plan exactly once, each rank's rows involve itself, and executing all
    shares (in any rank order) partitions the global array."""
    import paper_2004_12532_b200 as pp
    from dist_mirror import p2p_pieces
    rng = np.random.default_rng(2026)
    for trial in range(150):
        P = int(rng.integers(1, 10))
        ns = [int(x) for x in rng.integers(0, 200, size=P)]
        glob = rng.integers(0, 50, size=sum(ns)).astype(np.uint64)
        pivot = int(rng.integers(0, 51))
        shards = np.split(glob.copy(), np.cumsum(ns)[:-1]) if P > 1 else [glob.copy()]
        ts = []
        for sh in shards:  # local partition (any correct one)
            ts.append(oracle.partition_two_pointer(sh, pivot))
        K, plan = exchange_plan(ns, ts)
        pairs = {(tr.f + i, tr.t + i) for tr in plan for i in range(tr.length)}
        seen = []
        arr = np.concatenate(shards) if P > 1 else shards[0]
        for rank in rng.permutation(P):
            rows = pp.pp_dist_p2p_pieces(ns, ts, int(rank))
            assert rows == p2p_pieces(ns, ts, int(rank))
            for ra, a, rb, b, ln in rows:
                assert rank in (ra, rb) and ra != rb and ln > 0
                seen += [(a + i, b + i) for i in range(ln)]
                x = arr[a:a + ln].copy()
                arr[a:a + ln] = arr[b:b + ln]
                arr[b:b + ln] = x
        assert len(seen) == len(set(seen)) and set(seen) == pairs
        oracle.check_partition(glob, arr, pivot, K)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_per, seed, pivot, staging, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # uneven shards: rank r holds n_per + r*37 keys of one global array
        ns = [n_per + r * 37 for r in range(world)]
        off = sum(ns[:rank])
        host = synth.uniform_u64_np(ns[rank], seed, offset=off)
        shard = torch.from_numpy(host.view(np.int64).copy())

        def local(t, p):
            return oracle.partition_two_pointer(t.numpy().view(np.uint64), p)

        part = Partitioner(device="cpu", staging_bytes=staging, local_partition=local)
        K = part.partition(shard, pivot)
        mx = max(ns)
        padded = torch.zeros(mx, dtype=torch.int64)
        padded[: ns[rank]] = shard
        gathered = [torch.empty(mx, dtype=torch.int64) for r in range(world)]
        dist.all_gather(gathered, padded)
        if rank == 0:
            full = torch.cat([g[: ns[r]] for r, g in enumerate(gathered)])
            result_q.put((K, full.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


def _sort_worker(rank, world, port, ns, seed, kind, small, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        off = sum(ns[:rank])
        if kind == "uniform":
            host = synth.uniform_u64_np(ns[rank], seed, offset=off)
        elif kind == "dup":
            host = synth.mod_range_u64_np(ns[rank], seed, 7, offset=off)
        else:  # all equal, maximum key
            host = np.full(ns[rank], (1 << 64) - 1, dtype=np.uint64)
        shard = torch.from_numpy(host.view(np.int64).copy())

        def local_part(t, p):
            return oracle.partition_two_pointer(t.numpy().view(np.uint64), p)

        def local_sort(t):
            a = t.numpy().view(np.uint64)
            oracle.quicksort(a)

        part = Partitioner(device="cpu", staging_bytes=8 * 512, local_partition=local_part)
        part.sort(shard, local_sort=local_sort, small=small)
        mx = max(ns)
        padded = torch.zeros(mx, dtype=torch.int64)
        padded[: ns[rank]] = shard
        gathered = [torch.empty(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, padded)
        if rank == 0:
            full = torch.cat([g[: ns[r]] for r, g in enumerate(gathered)])
            result_q.put(full.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,small", [(2, "uniform", 64), (3, "dup", 100), (4, "uniform", 4096),
                                              (3, "maxeq", 50)])
def test_distributed_sort_gloo(world, kind, small):
    """Distributed quicksort over gloo (oracle local ops): the concatenated
    shards equal the oracle's sort of the global array."""
    ns = [3000 + 211 * r for r in range(world)]
    seed = 0xC0FFEE05
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sort_worker, args=(r, world, port, ns, seed, kind, small, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if kind == "uniform":
        glob = synth.uniform_u64_np(sum(ns), seed)
    elif kind == "dup":
        glob = synth.mod_range_u64_np(sum(ns), seed, 7)
    else:
        glob = np.full(sum(ns), (1 << 64) - 1, dtype=np.uint64)
    ref = glob.copy()
    oracle.quicksort(ref)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("world,staging", [(2, 1 << 20), (3, 4096), (4, 8 * 1000)])
def test_partitioner_gloo(world, staging):
    n_per, seed = 20000, 0xC0FFEE03
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    for pivot in (1 << 63, 1 << 60):
        procs = [ctx.Process(target=_worker, args=(r, world, port, n_per, seed, pivot, staging, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        K, out = q.get(timeout=120)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        ns = [n_per + r * 37 for r in range(world)]
        glob = synth.uniform_u64_np(sum(ns), seed)
        oracle.check_partition(glob, out, pivot, K)
        port = _free_port()
