#!/usr/bin/env python
"""Cleanup tail for small arrays: the one-CTA tail (param cleanup_cta) vs the
multi-kernel chain, per size and input (uniform; the stride-aligned
adversary), CUDA-event time per call over back-to-back calls on fresh copies,
plus the window fraction.

    python tools/small_tail_probe.py [--exps 18,19,20,21,22,23]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402,F401  (not used: checks run in the tests)
import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--exps", default="18,19,20,21,22,23")
    args = ap.parse_args()
    pp.load(build_if_missing=False)
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for ex in map(int, args.exps.split(",")):
        n = 1 << ex
        uni = synth.uniform_u64_torch(n, synth.SEEDS["c1"], "cuda")
        pp.reset_params()
        t = uni.clone()
        pp.pp_partition_async_u64(t, 1 << 63, d)
        torch.cuda.synchronize()
        st = pp.pp_last_stats()
        adv = synth.stride_aligned_u64_torch(n, 5, st["line_keys"], max(2, st["g"]), "cuda")
        reps = max(20, min(200, (1 << 27) // n))
        for name, src in (("uniform", uni), ("stride_aligned", adv)):
            bufs = [src.clone() for _ in range(reps + 10)]
            for cta in (0, 1 << 30):
                pp.reset_params()
                pp.pp_set_param("cleanup_cta", cta)
                for b in bufs:
                    b.copy_(src)
                for b in bufs[:10]:
                    pp.pp_partition_async_u64(b, 1 << 63, d)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for b in bufs[10:]:
                    pp.pp_partition_async_u64(b, 1 << 63, d)
                e.record()
                torch.cuda.synchronize()
                w = pp.pp_last_stats()["W"] / n
                print(f"2^{ex} {name:15s} {'cta ' if cta else 'chain'} {s.elapsed_time(e) / reps * 1e3:8.1f} us/call"
                      f"  window {w:.4f}  g {pp.pp_last_stats()['g']}", flush=True)
            del bufs


if __name__ == "__main__":
    main()
