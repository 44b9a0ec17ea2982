#!/usr/bin/env python
"""e2e host-buffer partition (pinned host memory, 2^EXP u64; env E2E_EXP,
default 27) for several streamed chunk sizes: python tools/e2e_sweep.py [chunk ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_12532_b200 as pp  # noqa: E402
import synth  # noqa: E402


def main():
    pp.load(build_if_missing=False)
    n = 1 << int(os.environ.get("E2E_EXP", "27"))
    a = synth.uniform_u64_np(n, synth.SEEDS["c3"])
    pin = torch.empty(n, dtype=torch.int64, pin_memory=True)
    hv = pin.numpy().view(np.uint64)
    for c in [int(x) for x in sys.argv[1:]] or [1 << 20, 1 << 22, 1 << 24]:
        pp.reset_params()
        pp.pp_set_param("host_chunk", c)
        ts = []
        for i in range(4):
            np.copyto(hv, a)
            t0 = time.perf_counter()
            pp.pp_partition_host_u64(hv, 1 << 63)
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"host_chunk": c, "ms": round(1e3 * min(ts[1:]), 3),
                          "keys_per_s": n / min(ts[1:])}), flush=True)


if __name__ == "__main__":
    main()
