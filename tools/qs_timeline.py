#!/usr/bin/env python
"""Kernel timeline of one quicksort (CUPTI via torch.profiler, not serialised
like ncu): per kernel family the launches, summed duration and the time it
is the only family running; GPU-idle gaps (no kernel of the library running)
and the critical-path split between the level loop and the tail.

    python tools/qs_timeline.py [--n 28] [--kind uniform|dup1000] [--params qs_pivot=2] [--dtype u64]
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def family(name):
    for f in ("qs_pivot", "qs_group", "qs_hv_", "qs_cleanup", "qs_small", "qs_cluster", "qs_leaf_bidx", "qs_leaf_handoff",
              "ss_group", "reduce_count", "scan_swap", "qs_seg", "qs_"):
        if f in name:
            return f.rstrip("_")
    return "other:" + name[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--kind", default="uniform")
    ap.add_argument("--params", default="")
    ap.add_argument("--dtype", default="u64")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    n = 1 << args.n
    if args.kind == "uniform":
        q0 = (synth.uniform_u64_torch(n, synth.SEEDS["c5"], "cuda") if args.dtype == "u64"
              else synth.uniform_u32_torch(n, synth.SEEDS["c5"], "cuda"))
    else:
        q0 = synth.mod_range_u64_torch(n, synth.SEEDS["c5"], 1000, "cuda")
        if args.dtype == "u32":
            q0 = q0.to(torch.int32)
    sort = pp.pp_quicksort_u64 if args.dtype == "u64" else pp.pp_quicksort_u32
    q = torch.empty_like(q0)
    for _ in range(2):  # warm-up (workspace, module load)
        q.copy_(q0)
        sort(q)
    torch.cuda.synchronize()
    q.copy_(q0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        sort(q)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") == "kernel" and ("pp::" in e["name"] or "pp_" in e["name"])]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in ks)
    span = t1 - t0
    # sweep: at each elementary interval, which families run
    pts = sorted({e["ts"] for e in ks} | {e["ts"] + e["dur"] for e in ks})
    fam = [family(e["name"]) for e in ks]
    stats = {}
    for f, e in zip(fam, ks):
        s = stats.setdefault(f, {"launches": 0, "sum_us": 0.0, "alone_us": 0.0, "streams": set()})
        s["launches"] += 1
        s["sum_us"] += e["dur"]
        s["streams"].add(e.get("args", {}).get("stream", -1))
    idle = 0.0
    gaps = []
    j = 0
    active = []
    for a, b in zip(pts[:-1], pts[1:]):
        while j < len(ks) and ks[j]["ts"] <= a:
            active.append(j)
            j += 1
        active = [i for i in active if ks[i]["ts"] + ks[i]["dur"] > a]
        if not active:
            idle += b - a
            gaps.append((a - t0, b - a))
        else:
            fs = {fam[i] for i in active}
            if len(fs) == 1:
                stats[fs.pop()]["alone_us"] += b - a
    last_level = max((e["ts"] + e["dur"] for f, e in zip(fam, ks) if f in ("qs_group", "qs_cleanup", "qs_hv")),
                     default=t0)
    print(json.dumps({"n": n, "kind": args.kind, "dtype": args.dtype, "params": args.params,
                      "span_ms": round(span / 1e3, 3), "idle_ms": round(idle / 1e3, 3),
                      "level_loop_end_ms": round((last_level - t0) / 1e3, 3),
                      "launches": len(ks)}))
    for f, s in sorted(stats.items(), key=lambda kv: -kv[1]["sum_us"]):
        print(f"  {f:18s} launches {s['launches']:5d}  sum {s['sum_us'] / 1e3:7.3f} ms  alone {s['alone_us'] / 1e3:7.3f} ms"
              f"  streams {len(s['streams'])}")
    gaps.sort(key=lambda g: -g[1])
    print("  largest idle gaps (at ms, us):", [(round(a / 1e3, 3), round(d, 1)) for a, d in gaps[:12]])
    # coarse timeline: 0.5 ms buckets, busy fraction per family
    B = 500.0
    nb = int(span // B) + 1
    rows = {}
    for f, e in zip(fam, ks):
        a, b = e["ts"] - t0, e["ts"] - t0 + e["dur"]
        for k in range(int(a // B), int(b // B) + 1):
            lo, hi = max(a, k * B), min(b, (k + 1) * B)
            if hi > lo and k < nb:
                rows.setdefault(f, [0.0] * nb)[k] += (hi - lo) / B
    print("  timeline (0.5 ms buckets, summed occupancy per family):")
    for f, r in rows.items():
        print(f"  {f:18s} " + "".join(" " if x < 0.05 else str(min(9, int(x * 10))) if x < 1 else "#" for x in r))


if __name__ == "__main__":
    main()
