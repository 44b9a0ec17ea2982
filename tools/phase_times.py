#!/usr/bin/env python
"""Time the c2 partition for several parameter settings (e.g. the fused
kernel stopped after each phase) -- one JSON line per setting.  GPU only.

    python tools/phase_times.py "fused=0" "fused_stop=1" "fused_stop=2" ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    pp.load(build_if_missing=False)
    n = 1 << 27
    pristine = synth.uniform_u64_torch(n, synth.SEEDS["c2"], "cuda")
    bufs = [pristine.clone() for _ in range(12)]
    d = torch.zeros(1, dtype=torch.int64, device="cuda")
    for spec in sys.argv[1:] or ["fused=1"]:
        pp.reset_params()
        kv = dict(x.split("=") for x in spec.split(",") if x)
        for k, v in kv.items():
            pp.pp_set_param(k, int(v))
        for b in bufs:
            b.copy_(pristine)
        torch.cuda.synchronize()
        ts = []
        for i, b in enumerate(bufs):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            pp.pp_partition_async_u64(b, 1 << 63, d)
            e.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(s.elapsed_time(e))
        print(json.dumps({"spec": spec, "ms_min": round(min(ts), 4), "ms_med": round(sorted(ts)[len(ts) // 2], 4)}),
              flush=True)
    pp.reset_params()


if __name__ == "__main__":
    main()
