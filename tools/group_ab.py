"""Interleaved A/B of library parameter settings on the partition's group
kernel at one size (library events around the group kernel; the same input
restored before every run; settings alternate so box drift hits all alike).

    python tools/group_ab.py --exp 33 --rounds 4 "g=296" "g=9472" ...
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--exp", type=int, default=33)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--dtype", default="u64")
    ap.add_argument("--n", type=int, default=0, help="key count (overrides --exp)")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    n = args.n or (1 << args.exp)
    if args.dtype == "u64":
        work = torch.empty(n, dtype=torch.int64, device="cuda")
        synth.uniform_u64_torch(n, synth.SEEDS["c3"], "cuda", out=work, chunk=1 << 27)
        part, pivot, w = pp.pp_partition_async_u64, 1 << 63, 8
    else:
        work = synth.uniform_u32_torch(n, synth.SEEDS["c4"], "cuda")
        part, pivot, w = pp.pp_partition_async_u32, 1 << 31, 4
    pristine = work.clone()
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    res = {sp: {"group": [], "total": [], "copy": []} for sp in args.specs}
    for r in range(args.rounds + 1):
        for sp in args.specs:
            pp.reset_params()
            for kv in filter(None, sp.split(",")):
                k, v = kv.split("=")
                pp.pp_set_param(k, int(v))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            work.copy_(pristine)
            e.record()
            torch.cuda.synchronize()
            pp.pp_timing(True)
            part(work, pivot, d)
            torch.cuda.synchronize()
            t = pp.pp_timing_read()
            pp.pp_timing(False)
            if r:
                res[sp]["group"].append(t["group_ms"])
                res[sp]["total"].append(t["total_ms"])
                res[sp]["copy"].append(s.elapsed_time(e))
    pp.reset_params()
    for sp, v in res.items():
        st = pp.pp_last_stats()
        print(json.dumps({"spec": sp, "n": n, "dtype": args.dtype, "group_ms_med": statistics.median(v["group"]),
                          "total_ms_med": statistics.median(v["total"]), "total_ms_all": v["total"],
                          "copy_gbs_med": 2 * w * n / (statistics.median(v["copy"]) / 1e3) / 1e9,
                          "total_gbs_med": 2 * w * n / (statistics.median(v["total"]) / 1e3) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
