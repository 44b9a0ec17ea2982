#!/usr/bin/env python
"""bench.py -- BASELINE metric: partition keys/s and GB/s (fraction of the HBM
read+write roofline) at 1/2/4/8 B200; quicksort keys/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[2], the configuration the metric is
quoted on "at 1/2/4/8 B200"): in-place partition of the GLOBAL
array of n = 2^33 uint64 keys (64 GiB), i.i.d. uniform from the splitmix64
stream (seed c3; key_i depends only on the global index i), pivot 2^63
(mu = 0.5), sharded contiguously over the N ranks (2^33/N keys per GPU:
64 GiB at N = 1, 8 GiB at N = 8) -- strong scaling.  One step = one full
partition of the whole array: at N = 1 pp_partition_async_u64 (all kernels
of the hot path); at N > 1 (torchrun) pp_partition_dist_u64 on every rank
(local partition, ncclAllGather of (status, n_r, t_r, pivot), the exchange of
misplaced ranges over NCCL/NVLink).  Before every timed step the shard is
restored from a pristine device copy (or regenerated when two copies do not
fit), untimed; each step is bracketed by a barrier + synchronize and CUDA
events on the launching stream; the step time is the max over ranks.  The
inputs (>= 8 GiB per GPU) are far larger than L2.

The c2 line (2^27 keys, mu = 0.01 / 0.5 / 0.99, aux memory), config 1, 4 and
5 and the comparison rows go to "extras" (rank 0, N = 1).

--impl reference: the CPU oracle (oracle/, serial two-pointer partition,
PAPER.md:1433-1436) on the host cores, on a bounded sample of the same
workload (the first 2^27 keys of the c3 array per step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOTAL = 1 << 33  # BASELINE config 3: the global array
N_C2 = 1 << 27     # BASELINE config 2
N_REF_SAMPLE = 1 << 27  # CPU oracle sample per step (the reference arm / cpu_baseline)
E2E_SAMPLE = 1 << 30    # per-rank host-buffer sample for the end-to-end number
PIVOT = 1 << 63
L2_FLUSH_BYTES = 512 << 20
METRIC = "partition keys/s and GB/s (fraction of HBM roofline) at 1/2/4/8 B200; quicksort keys/s"
WORKLOAD = ("c3: in-place partition of the global array, n=2^33 uint64 uniform keys (64 GiB), pivot 2^63 "
            "(mu=0.5), sharded contiguously over the GPUs (strong scaling)")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(n: int, alg_bytes: int):
    """DRAM bytes per launch of the group kernel from the committed ncu
    captures (profiles/ncu_summary.json): the capture of this very size when
    there is one (2^33 keys: one-pass dram metrics, no replay), else the c2
    capture's traffic per algorithmic byte times this launch's algorithmic
    bytes (said so in the line)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        exact = {(1 << 33): "ss_group_kernel_2^33", (1 << 27): "ss_group_kernel"}.get(n)
        if exact and exact in d:
            return d[exact]["dram_bytes_per_launch"], d[exact]["source"]
        e = d["ss_group_kernel"]
        return e["dram_bytes_per_launch"] / e["algorithmic_bytes"] * alg_bytes, "scaled from " + e["source"]
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """CPU oracle arm: the serial two-pointer partition on the host, each step
    a bounded sample of the headline workload (the first 2^27 keys of the c3
    array, fresh copy each step); rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth
    pristine = synth.uniform_u64_np(N_REF_SAMPLE, synth.SEEDS["c3"])
    work = np.empty_like(pristine)
    for _ in range(args.warmup):
        np.copyto(work, pristine)
        oracle.partition_two_pointer(work, PIVOT)
    times = []
    for _ in range(args.steps):
        np.copyto(work, pristine)
        t0 = time.perf_counter()
        split = oracle.partition_two_pointer(work, PIVOT)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = N_REF_SAMPLE * args.steps / tot
    sample = (f"first 2^27 keys of the c3 array (global indices 0..2^27-1) per step, {args.steps} timed steps, "
              f"fresh copy each, serial oracle on 1 host thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": N_TOTAL, "sample_keys_per_step": N_REF_SAMPLE, "pivot": PIVOT,
                   "split_of_sample": split},
        "gbs": 2 * 8 * N_REF_SAMPLE * args.steps / tot / 1e9,
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_baseline(budget_s: float = 12.0):
    """The oracle as it stands on a bounded sample of the headline workload
    (the first 2^27 keys of the c3 array), 1 host thread."""
    import oracle
    import synth
    pristine = synth.uniform_u64_np(N_REF_SAMPLE, synth.SEEDS["c3"])
    work = np.empty_like(pristine)
    times = []
    t_start = time.perf_counter()
    while len(times) < 2 or (time.perf_counter() - t_start < budget_s and len(times) < 40):
        np.copyto(work, pristine)
        t0 = time.perf_counter()
        oracle.partition_two_pointer(work, PIVOT)
        times.append(time.perf_counter() - t0)
    v = N_REF_SAMPLE * len(times) / sum(times)
    return {"value": v, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "sample": f"first 2^27 keys of the c3 array, {len(times)} runs of the serial two-pointer oracle, "
                      f"fresh copy each, 1 host thread", "host": host_info()}


def host_info():
    """The box's host (nproc, CPU model, RAM)."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            info["ram_gb"] = round(int(f.readline().split()[1]) / 2**20, 1)
    except OSError:
        pass
    return info


def cpu_quicksort_baseline(budget_s: float = 8.0):
    """Config 5's CPU rows on a bounded sample: the serial oracle quicksort
    (median-of-3) and numpy.sort as a library reference,
    1 host thread, on the first 2^24 keys of the c5 uniform input."""
    import oracle
    import synth
    m = 1 << 24
    a = synth.uniform_u64_np(m, synth.SEEDS["c5"])
    res = {}
    for name, fn in (("oracle_quicksort", oracle.quicksort), ("numpy_sort", lambda x: x.sort())):
        times = []
        t_start = time.perf_counter()
        while len(times) < 1 or (time.perf_counter() - t_start < budget_s / 2 and len(times) < 5):
            b = a.copy()
            t0 = time.perf_counter()
            fn(b)
            times.append(time.perf_counter() - t0)
        res[name] = {"keys_per_s": m / min(times), "ms": 1e3 * min(times)}
    res["sample"] = "first 2^24 keys of the c5 uniform input, 1 host thread"
    return res


def shard_range(rank: int, ws: int, n_total: int):
    """Contiguous shards of the global array in rank order (the last rank takes
    the remainder)."""
    per = n_total // ws
    off = rank * per
    return off, (n_total - off if rank == ws - 1 else per)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c1/c2/c4/c5 and comparison lines")
    ap.add_argument("--n-total", type=int, default=N_TOTAL,
                    help="global keys (default 2^33 = BASELINE config 3; smaller only for quick checks)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU code path (NCCL process group, pp_partition_dist) even at one rank")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2004_12532_b200 as pp
    import synth

    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep rank 0's stdout to the one JSON line
    if args.force_dist and "RANK" not in os.environ:  # one process without torchrun
        os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0", "MASTER_ADDR": "127.0.0.1",
                           "MASTER_PORT": os.environ.get("MASTER_PORT", "29533")})
    ws, rank, local = dist_env()
    dist_on = ws > 1 or args.force_dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)
    pp.load(build_if_missing=False)
    pp.reset_params()
    for kv in filter(None, os.environ.get("PP_BENCH_PARAMS", "").split(",")):  # A/B tuning (tools/ab_params.sh)
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    stream = torch.cuda.current_stream()

    n_total = args.n_total
    off, n = shard_range(rank, ws, n_total)
    seed = synth.SEEDS["c3"]
    work = torch.empty(n, dtype=torch.int64, device=dev)
    synth.uniform_u64_torch(n, seed, dev, offset=off, out=work, chunk=1 << 27)
    free, _ = torch.cuda.mem_get_info(dev)
    pristine = None
    if free > 8 * n + (6 << 30):  # a pristine copy fits: restore by D2D copy (else regenerate)
        pristine = work.clone()

    def restore():
        if pristine is not None:
            work.copy_(pristine)
        else:
            synth.uniform_u64_torch(n, seed, dev, offset=off, out=work, chunk=1 << 27)

    d_split = torch.zeros(1, dtype=torch.int64, device=dev)
    last_split = [None]
    if dist_on:
        # the library's own NCCL communicator (C ABI pp_dist_*): rank 0 makes
        # the unique id, the torch process group only carries its 128 bytes
        uid = [pp.pp_dist_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        pp.pp_dist_init(uid[0], ws, rank, local)

    def step():
        if dist_on:
            last_split[0] = pp.pp_partition_dist(work, PIVOT)
        else:
            pp.pp_partition_async_u64(work, PIVOT, d_split)

    def sync_all():
        torch.cuda.synchronize()
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        restore()
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps; each restored untimed, then bracketed by a
    #      barrier + synchronize and CUDA events on the launching stream.  No
    #      library-internal events here (an event between the group kernel and
    #      its PDL-launched cleanup costs ~12 us; tools/timing_overhead.py) ----
    pp.pp_timing(False)
    step_ms, launches = [], 0
    phases = []
    copy_ms = []  # the untimed restores: a D2D copy of the shard, the sustained copy rate at this size
    for i in range(args.steps):
        cs, ce = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs.record(stream)
        restore()
        ce.record(stream)
        sync_all()
        copy_ms.append(cs.elapsed_time(ce))
        pp.pp_launch_count(reset=True)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        step()
        e.record(stream)
        sync_all()
        launches += pp.pp_launch_count()
        step_ms.append(s.elapsed_time(e))
        if dist_on:
            phases.append(pp.pp_dist_last_timing())
    # ---- a second pass with the library's CUDA events around the group
    #      kernel on the launching stream: its live duration for the roofline ----
    reps2 = min(args.steps, 5)
    pp.pp_timing(True)
    for i in range(reps2):
        restore()
        torch.cuda.synchronize()
        step()
    torch.cuda.synchronize()
    tim = pp.pp_timing_read()
    pp.pp_timing(False)
    clocks = sampler.stop()
    split = int(d_split.item()) if not dist_on else last_split[0]
    stats = pp.pp_last_stats() if not dist_on else {}

    exchange = None
    tot_ms = sum(step_ms)
    if dist_on:
        t = torch.tensor(step_ms, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # per step: max over ranks
        step_ms = [float(x) for x in t.tolist()]
        tot_ms = sum(step_ms)
        k = max(len(phases), 1)
        loc = [sum(p[f] for p in phases) / k for f in ("local_ms", "gather_ms", "exchange_ms", "bytes")]
        tt = torch.tensor(loc, dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        lm, gm, xm, xb = (float(x) for x in tt.tolist())
        exchange = {"path": "one-sided CUDA IPC" if pp.pp_get_param("dist_p2p") else "NCCL send/recv via staging",
                    "local_partition_ms": lm, "allgather_ms": gm, "exchange_ms": xm, "bytes_per_gpu": xb,
                    "nvlink_gbs": (xb / (xm / 1e3) / 1e9) if xm > 0 else None,
                    "frac_of_900_gbs": (xb / (xm / 1e3) / 1e9 / 900.0) if xm > 0 else None,
                    "local_hbm_gbs": (16 * n / (lm / 1e3) / 1e9) if lm > 0 else None,
                    "timing": "library CUDA events on the call's stream (timed steps), per-rank means, max over ranks"}

    overlap = None
    if dist_on:
        try:
            main_split = last_split[0]
            overlap = measure_overlap(pp, torch, dist, dev, stream, args, restore, step, sync_all, last_split, n_total)
            overlap["split_matches_default"] = overlap.pop("split") == main_split
            last_split[0] = main_split
        except Exception as ex:  # an extra: the headline line must still print
            overlap = {"error": f"{type(ex).__name__}: {ex}"[:300]}
        finally:
            pp.pp_set_param("dist_overlap", 0)

    value = n_total * args.steps / (tot_ms / 1e3)
    ms_per_step = tot_ms / args.steps
    bytes_step = 2 * 8 * n_total
    peak, peak_kind = peaks()
    # dominant kernel: the Smoothed Striding group kernel (every full line read
    # once + written once): algorithmic bytes per launch
    line_keys = stats.get("line_keys", 1024)
    grp_bytes = 2 * 8 * stats.get("n_lines", n // 1024) * line_keys
    grp_ms = tim["group_ms"] / max(tim["calls"], 1)
    achieved = grp_bytes / (grp_ms / 1e3) / 1e9 if grp_ms > 0 else None
    traffic, traffic_src = ncu_traffic(n, grp_bytes)
    gbs = bytes_step / (ms_per_step / 1e3) / 1e9

    out = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOAD if n_total == N_TOTAL else f"{WORKLOAD} [reduced: n={n_total}]",
                   "n": n_total, "n_per_gpu": n, "pivot": PIVOT, "mu": 0.5,
                   "parallelism": f"dp{ws} (contiguous shards + NCCL exchange)" if dist_on else "single",
                   "l2": "inputs larger than L2 (>= 8 GiB per GPU); every step restores its shard untimed "
                         + ("(D2D copy from a pristine copy)" if pristine is not None else "(regenerated)")},
        "gbs": gbs,
        "frac_of_8tbs": gbs / ws / 8000.0,
        "frac_of_measured_hbm": gbs / ws / peak,
        "step_ms_min": min(step_ms), "step_ms_max": max(step_ms),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "ss_group_kernel", "peak_source": peak_kind, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": grp_bytes, "avg_launch_ms": grp_ms,
                     "kernel_share_of_step": (tim["group_ms"] / tim["total_ms"]) if tim["total_ms"] else None,
                     "sustained_copy_gbs_same_size": (16 * n / (statistics.median(copy_ms) / 1e3) / 1e9)
                     if pristine is not None else None,
                     "frac_of_sustained_copy": (achieved / (16 * n / (statistics.median(copy_ms) / 1e3) / 1e9))
                     if (pristine is not None and achieved) else None,
                     "timing": f"group kernel bracketed by CUDA events on the launching stream in a second pass "
                               f"of {reps2} steps (restored untimed); the timed steps run without these events"},
        "gpu_launches": launches,
        "clocks": clocks,
        **({"exchange": exchange} if exchange else {}),
        **({"exchange_overlap": overlap} if overlap else {}),
        "split": split,
        "window_frac": (stats.get("W", 0) / n) if stats else None,
        "aux_bytes": stats.get("aux_bytes"),
        "aux_frac": (stats.get("aux_bytes", 0) / (8 * n)) if stats else None,
    }
    if not dist_on:
        # split sanity vs the closed form: a device compare-and-count (torch)
        # of the restored input -- the oracle's exact check runs in the tests
        restore()
        C = 1 << 28
        out["split_ok"] = split == sum(int(((work[s:s + C] ^ (-(1 << 63))) < 0).sum().item())
                                       for s in range(0, n, C))
    del work, pristine
    torch.cuda.empty_cache()

    if not args.no_e2e:
        out["e2e"] = e2e(pp, torch, dist if dist_on else None, rank, ws, off, n, args)
    if rank == 0 and not dist_on:
        flush = torch.ones(L2_FLUSH_BYTES // 8, dtype=torch.int64, device=dev)
        if not args.no_extras:
            out["extras"] = extras(pp, torch, synth, dev, stream, flush, args)
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline()
            if not args.no_extras:
                out["extras"]["cpu_quicksort_sample"] = cpu_quicksort_baseline()
    if rank == 0:
        print(json.dumps(out))
    if dist_on:
        pp.pp_dist_finalize()
        dist.destroy_process_group()
    return 0


def measure_overlap(pp, torch, dist, dev, stream, args, restore, step, sync_all, last_split, n_total):
    """The count-first overlapped exchange (param dist_overlap, SURVEY §8(f)
    #1) at N > 1: same input, same step bracket, a few steps, max over ranks."""
    pp.pp_set_param("dist_overlap", 1)
    ov_ms, ov_ph, ov_split = [], [], None
    for i in range(min(args.steps, 5) + 1):
        restore()
        sync_all()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        step()
        e.record(stream)
        sync_all()
        if i:  # the first one warms the path up
            ov_ms.append(s.elapsed_time(e))
            ov_ph.append(pp.pp_dist_last_timing())
        ov_split = last_split[0]
    pp.pp_set_param("dist_overlap", 0)
    default_split = ov_split
    t = torch.tensor(ov_ms, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ov_ms = [float(x) for x in t.tolist()]
    loc = [sum(p[f] for p in ov_ph) / len(ov_ph) for f in ("local_ms", "gather_ms", "exchange_ms", "bytes")]
    tt = torch.tensor(loc, dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    cm, gm2, pxm, xb2 = (float(x) for x in tt.tolist())
    return {"ms_per_step": sum(ov_ms) / len(ov_ms), "steps": len(ov_ms),
            "keys_per_s": n_total / (sum(ov_ms) / len(ov_ms) / 1e3),
            "count_ms": cm, "allgather_ms": gm2, "partition_and_exchange_ms": pxm, "bytes_per_gpu": xb2,
            "chunks": pp.pp_get_param("dist_chunks"), "split": default_split,
            "timing": "same bracket as the timed steps (barrier + synchronize, CUDA events, max over ranks)"}


def e2e(pp, torch, dist, rank, ws, off, n, args):
    """End to end through the public host-buffer API on every rank: a sample
    of min(n_per_gpu, 2^30 / N) keys of the rank's c3 shard in pinned host
    memory; every step copies it in (H2D), partitions it on the GPU and
    copies the whole partitioned sample and the split back (D2H) --
    pp_partition_host_u64 (the streamed host partition),
    host wall clock around the synchronous call.  At N > 1 the ranks run
    concurrently (barrier around each step) and the value is the sum over
    ranks; the NCCL exchange is not part of this number (it is in the
    device-timed value)."""
    import synth
    m = min(n, max(1 << 20, E2E_SAMPLE // ws))  # the whole job samples ~2^30 keys: host memory stays bounded at N = 8
    pristine = synth.uniform_u64_np(m, synth.SEEDS["c3"], offset=off)
    host = torch.empty(m, dtype=torch.int64, pin_memory=True)
    hv = host.numpy().view(np.uint64)
    steps = max(3, min(args.steps, 5))
    np.copyto(hv, pristine)
    pp.pp_partition_host_u64(hv, PIVOT)  # warm
    times = []
    for _ in range(steps):
        np.copyto(hv, pristine)
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        pp.pp_partition_host_u64(hv, PIVOT)
        times.append(time.perf_counter() - t0)
    v = m * steps / sum(times)
    if dist:
        t = torch.tensor([v], dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t)
        v = float(t.item())
    return {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 8 * m * ws, "d2h_bytes_per_step": (8 * m + 8) * ws,
            "steps": steps, "ms_per_step": 1e3 * sum(times) / steps, "sample_keys_per_gpu": m,
            "api": "pp_partition_host_u64 (pinned host; streamed chunks: H2D from both ends, per-chunk GPU "
                   "partition, D2H of each side overlapping the uploads)",
            "timing": "host wall clock around the synchronous call; sample = the first min(n_per_gpu, 2^30 / N) "
                      "keys of each rank's c3 shard (PCIe-bound, size-independent beyond a few GiB)"}


def extras(pp, torch, synth, dev, stream, flush, args):
    """Secondary numbers (rank 0, N = 1): BASELINE config 2 (mu = 0.5, 0.01,
    0.99, aux memory), the comparison rows, configs 5, 1 and 4."""
    res = {}
    n = N_C2
    pristine = synth.uniform_u64_torch(n, synth.SEEDS["c2"], dev)
    d = torch.zeros(1, dtype=torch.int64, device=dev)
    # config 2 at mu = 0.5: K fresh 1 GiB copies partitioned back to back
    # between two events (no restore traffic between steps; each copy is
    # larger than L2 and untouched since its copy)
    K = max(5, min(args.steps, 20))
    bufs = [pristine.clone() for _ in range(K)]
    for b in bufs[:3]:
        pp.pp_partition_async_u64(b, PIVOT, d)
    for b in bufs[:3]:
        b.copy_(pristine)
    flush.sum()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for b in bufs:
        pp.pp_partition_async_u64(b, PIVOT, d)
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / K
    st = pp.pp_last_stats()
    res["c2_u64_2^27_mu0.5"] = {"keys_per_s": n / (ms / 1e3), "ms": ms, "gbs": 16 * n / (ms / 1e3) / 1e9,
                                "window_frac": st["W"] / n, "aux_bytes": st["aux_bytes"],
                                "aux_frac": st["aux_bytes"] / (8 * n), "split": int(d.item()),
                                "timing": f"{K} fresh copies back to back between two events"}
    del bufs
    buf = torch.empty_like(pristine)
    for mu in (0.01, 0.99):
        p = synth.PIVOT_MU[mu]
        ts = []
        for i in range(8):
            buf.copy_(pristine)
            flush.sum()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            pp.pp_partition_async_u64(buf, p, d)
            e.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(s.elapsed_time(e))
        ms = statistics.mean(ts)
        st = pp.pp_last_stats()
        res[f"c2_u64_2^27_mu{mu}"] = {"keys_per_s": n / (ms / 1e3), "ms": ms, "gbs": 16 * n / (ms / 1e3) / 1e9,
                                      "window_frac": st["W"] / n, "aux_frac": st["aux_bytes"] / (8 * n)}
    # duplicate-heavy u64 keys (uniform, skewed and duplicate-heavy
    # inputs): c2 size, keys uniform on [0, 1000), pivot 500 (mu = 0.5)
    dup = synth.mod_range_u64_torch(n, synth.SEEDS["c2"], 1000, dev)
    ts = []
    for i in range(8):
        buf.copy_(dup)
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        pp.pp_partition_async_u64(buf, 500, d)
        e.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e))
    ms = statistics.mean(ts)
    st = pp.pp_last_stats()
    res["c2_u64_2^27_dup1000_pivot500"] = {"keys_per_s": n / (ms / 1e3), "ms": ms, "gbs": 16 * n / (ms / 1e3) / 1e9,
                                           "window_frac": st["W"] / n, "split": int(d.item())}
    del dup
    # Strided (X = 0) vs Smoothed Striding
    # (random X) on the c2 input and on the stride-aligned
    # adversary (line j true iff j mod g < g/2, g = the library's group count)
    st0 = pp.pp_last_stats()
    adv = synth.stride_aligned_u64_torch(n, synth.SEEDS["c2"], st0["line_keys"], st0["g"], dev)
    abl = {}
    for name, src in (("uniform", pristine), ("stride_aligned", adv)):
        for strided in (0, 1):
            pp.pp_set_param("strided", strided)
            ts = []
            for i in range(6):
                buf.copy_(src)
                flush.sum()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                pp.pp_partition_async_u64(buf, PIVOT, d)
                e.record(stream)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(s.elapsed_time(e))
            ms = statistics.mean(ts)
            abl[f"{name}_{'strided' if strided else 'smoothed'}"] = {
                "ms": ms, "gbs": 16 * n / (ms / 1e3) / 1e9, "window_frac": pp.pp_last_stats()["W"] / n}
    pp.pp_set_param("strided", 0)
    res["ablation_strided_vs_smoothed"] = abl
    # the paper's Standard Algorithm (stable, out of place,
    # PAPER.md:284-311) on the same input: count pass + scatter pass = 3*n*w
    # bytes of traffic and a second n-key array, vs the in-place 2*n*w
    outb = torch.empty_like(pristine)
    ts = []
    for i in range(6):
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        pp.pp_partition_stable_async_u64(pristine, outb, PIVOT, d)
        e.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(s.elapsed_time(e))
    ms = statistics.mean(ts)
    res["standard_algorithm_out_of_place"] = {
        "ms": ms, "keys_per_s": n / (ms / 1e3), "gbs_2nw": 16 * n / (ms / 1e3) / 1e9,
        "gbs_traffic_3nw": 24 * n / (ms / 1e3) / 1e9, "aux_bytes": 8 * n}
    del outb
    # SURVEY §8(f) #4, in place: the stable partition by tile partitions +
    # rotation merges (O(n log n) work), the price of stability in place
    wb = torch.empty_like(pristine)
    ts = []
    for i in range(4):
        wb.copy_(pristine)
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        pp.pp_partition_stable_inplace(wb, PIVOT)
        e.record(stream)
        torch.cuda.synchronize()
        if i >= 1:
            ts.append(s.elapsed_time(e))
    ms = statistics.mean(ts)
    res["stable_in_place"] = {"ms": ms, "keys_per_s": n / (ms / 1e3), "gbs_2nw": 16 * n / (ms / 1e3) / 1e9,
                              "aux_bytes": pp.pp_last_stats()["aux_bytes"],
                              "note": "synchronous call (includes the split readback)"}
    del wb
    # the paper's Blocked-Prefix-Sum partition (low-space form,
    # PAPER.md:319-478, 1466-1486), in place, on the same input
    wb = torch.empty_like(pristine)
    ts = []
    for i in range(5):
        wb.copy_(pristine)
        flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        pp.pp_partition_bps_async_u64(wb, PIVOT, d)
        e.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(s.elapsed_time(e))
    ms = statistics.mean(ts)
    res["blocked_prefix_sum_low_space"] = {
        "ms": ms, "keys_per_s": n / (ms / 1e3), "gbs_2nw": 16 * n / (ms / 1e3) / 1e9,
        "aux_bytes": pp.pp_last_stats()["aux_bytes"]}
    del wb
    del pristine, buf, adv
    nq = 1 << 28
    # BASELINE config 5 (median-of-3 pivots, the config's rule), and the same
    # sorts with the median of 31 sampled keys as pivot (qs_pivot = 2; same
    # input, same output)
    for kind in ("uniform", "dup1000"):
        if kind == "uniform":
            q0 = synth.uniform_u64_torch(nq, synth.SEEDS["c5"], dev)
        else:
            q0 = synth.mod_range_u64_torch(nq, synth.SEEDS["c5"], 1000, dev)
        q = torch.empty_like(q0)
        # (and the device-built level loop, qs_dev = 1, with median-of-3 pivots)
        for rule in ("median3", "median31", "median3_devlevels"):
            pp.reset_params()
            if rule == "median31":
                pp.pp_set_param("qs_pivot", 2)
            if rule == "median3_devlevels":
                pp.pp_set_param("qs_dev", 1)
            ts = []
            for i in range(3):
                q.copy_(q0)
                flush.sum()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                pp.pp_quicksort_u64(q)
                e.record(stream)
                torch.cuda.synchronize()
                if i >= 1:
                    ts.append(s.elapsed_time(e))
            ms = statistics.mean(ts)
            qs = pp.pp_quicksort_last_stats()
            # pass model: every level reads + writes the keys of the
            # segments it partitions (level_keys), the per-CTA recursion makes at
            # least one pass over the small segments, the bin sort one over all n
            model = 16 * (qs["level_keys"] + qs["small_keys"] + nq)
            peak, _ = peaks()
            res[f"quicksort_{kind}_2^28" + {"median3": "", "median31": "_median31",
                                             "median3_devlevels": "_devlevels"}[rule]] = {
                "keys_per_s": nq / (ms / 1e3), "ms": ms, "pivot": rule.split("_")[0], "stats": qs,
                "levels_built_on": "device" if rule.endswith("devlevels") else "host",
                "roofline": {"bound": "hbm", "model_bytes": model, "achieved": model / (ms / 1e3) / 1e9,
                             "peak": peak, "unit": "GB/s", "frac": model / (ms / 1e3) / 1e9 / peak,
                             "model": "2*w*(level_keys + small_keys + n): levels + one per-CTA recursion pass + "
                                      "one bin pass (a lower bound on the bytes moved)"}}
        pp.reset_params()
        del q0, q

    def timed(fn, reps=3):
        ts = []
        for i in range(reps + 1):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            torch.cuda.synchronize()
            if i >= 1:
                ts.append(s.elapsed_time(e))
        return statistics.mean(ts)

    # BASELINE config 1: n = 2^20 u64 (8 MiB, L2-resident: launch-bound, reported not judged),
    # back-to-back partitions of fresh copies
    n1 = 1 << 20
    c1src = synth.uniform_u64_torch(n1, synth.SEEDS["c1"], dev)
    c1bufs = [c1src.clone() for _ in range(50)]
    d1 = torch.zeros(1, dtype=torch.int64, device=dev)
    for b in c1bufs[:5]:
        pp.pp_partition_async_u64(b, PIVOT, d1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for b in c1bufs[5:]:
        pp.pp_partition_async_u64(b, PIVOT, d1)
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 45
    res["c1_u64_2^20"] = {"keys_per_s": n1 / (ms / 1e3), "ms": ms, "gbs": 16 * n1 / (ms / 1e3) / 1e9,
                          "note": "8 MiB: L2-resident and launch-bound (SURVEY §8(d)); back-to-back calls"}
    del c1src, c1bufs
    # BASELINE config 4: n = 1,000,000,007 u32 adversarial inputs, pivot 2^31
    n4 = 1_000_000_007
    for pat in ("partitioned", "reverse", "alternating", "all_false", "all_true"):
        a0 = synth.adversarial_u32_torch(n4, pat, synth.SEEDS["c4"], dev)
        a = torch.empty_like(a0)
        d4 = torch.zeros(1, dtype=torch.int64, device=dev)

        def run():
            a.copy_(a0)
            flush.sum()
            torch.cuda.synchronize()
            # time only the partition: events recorded by the caller bracket copy+flush too,
            # so measure with the library's own phase events instead
            pp.pp_timing(True)
            pp.pp_partition_async_u32(a, synth.ADV_PIVOT_U32, d4)
            torch.cuda.synchronize()

        ms = []
        for i in range(4):
            run()
            t = pp.pp_timing_read()
            pp.pp_timing(False)
            if i >= 1:
                ms.append(t["total_ms"])
        m = statistics.mean(ms)
        st = pp.pp_last_stats()
        res[f"c4_u32_{pat}"] = {"keys_per_s": n4 / (m / 1e3), "ms": m, "gbs": 8 * n4 / (m / 1e3) / 1e9,
                                "window_frac": st["W"] / n4}
        del a0, a
    # BASELINE config 4, Zipf(1.1) keys (rank - 1 on [0, 2^32)), pivot = sample median
    z0 = synth.zipf_u32_torch(n4, 1.1, synth.SEEDS["c4"], dev)
    zp = int(torch.sort(z0.to(torch.int64) & 0xFFFFFFFF).values[n4 // 2])
    z = torch.empty_like(z0)
    dz = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = []
    for i in range(4):
        z.copy_(z0)
        flush.sum()
        torch.cuda.synchronize()
        pp.pp_timing(True)
        pp.pp_partition_async_u32(z, zp, dz)
        torch.cuda.synchronize()
        t = pp.pp_timing_read()
        pp.pp_timing(False)
        if i >= 1:
            ms.append(t["total_ms"])
    m = statistics.mean(ms)
    st = pp.pp_last_stats()
    res["c4_u32_zipf1.1_median"] = {"keys_per_s": n4 / (m / 1e3), "ms": m, "gbs": 8 * n4 / (m / 1e3) / 1e9,
                                    "pivot": zp, "window_frac": st["W"] / n4}
    del z0, z
    return res


if __name__ == "__main__":
    sys.exit(main())
