"""Partition throughput vs array size on one GPU (u64 uniform, pivot 2^63):
the group kernel's live time from the library's events, and a D2D copy of the
same size for reference.

    python tools/size_sweep.py [--exps 27,29,31,33] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exps", default="27,29,31,32,33")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--params", default="")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    for kv in filter(None, args.params.split(",")):
        k, v = kv.split("=")
        pp.pp_set_param(k, int(v))
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for ex in [int(x) for x in args.exps.split(",")]:
        n = 1 << ex
        work = torch.empty(n, dtype=torch.int64, device="cuda")
        synth.uniform_u64_torch(n, synth.SEEDS["c3"], "cuda", out=work, chunk=1 << 27)
        pristine = work.clone()
        gms, cms = [], []
        for r in range(args.reps + 1):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            work.copy_(pristine)
            e.record()
            torch.cuda.synchronize()
            pp.pp_timing(True)
            pp.pp_partition_async_u64(work, 1 << 63, d)
            torch.cuda.synchronize()
            t = pp.pp_timing_read()
            pp.pp_timing(False)
            if r:
                gms.append(t["group_ms"])
                cms.append(s.elapsed_time(e))
        st = pp.pp_last_stats()
        gb = 16 * st["n_lines"] * st["line_keys"]
        print(json.dumps({"n": f"2^{ex}", "group_ms": min(gms), "group_gbs": gb / (min(gms) / 1e3) / 1e9,
                          "copy_gbs": 16 * n / (min(cms) / 1e3) / 1e9, "g": st["g"]}), flush=True)
        del work, pristine
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
