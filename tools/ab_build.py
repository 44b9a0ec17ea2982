#!/usr/bin/env python
"""Build an A/B variant of libpp.so with extra compile-time defines into
ab_libs/ (its own object dir), for PP_LIB_PATH=... runs:

    python tools/ab_build.py ab_libs/lib_u32pf3.so -DPP_U32_PF=3 [...]
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_12532_b200 import _build as B  # noqa: E402


def main():
    out, defs = os.path.abspath(sys.argv[1]), sys.argv[2:]
    objdir = os.path.join("/tmp", "ab_objs", os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    inc, lib = B.nccl_paths()
    common = ["nvcc", *B.NVCC_FLAGS[:-1], "-I", os.path.join(ROOT, "include"), "-I", inc,
              f'-DPP_NCCL_LIB="{lib}"', *defs]
    jobs = [(os.path.join(objdir, os.path.basename(s)[:-3] + ".o"), s) for s in B.sources()]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda j: subprocess.check_call(common + ["-c", "-o", j[0], j[1]]), jobs))
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out,
                           *[o for o, _ in jobs], "-ldl"])
    print(out)


if __name__ == "__main__":
    main()
