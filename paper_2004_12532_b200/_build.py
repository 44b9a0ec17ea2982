"""In-tree build of libpp.so (nvcc, sm_100a).  No JIT cache: the .so sits next
to the package so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpp.so")
# the EREW shadow-writer audit build (-DPP_AUDIT=1; tests only, include/pp.h pp_audit_set)
LIB_AUDIT = os.path.join(PKG, "libpp_audit.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [
        os.path.join(ROOT, "include", "pp.h")]


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in deps())


def nccl_paths():
    """(include dir, library file) of the NCCL that PyTorch ships (the one
    loaded at run time), falling back to the system NCCL headers."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "libnccl.so.2"


def build(force: bool = False, verbose: bool = False, audit: bool = False) -> str:
    """Compile every .cu to an object in parallel (one nvcc per source; no
    device code crosses translation units), then link libpp.so (audit=True:
    the EREW audit build libpp_audit.so, -DPP_AUDIT=1, its own objects)."""
    lib_out = LIB_AUDIT if audit else LIB
    if not force and up_to_date(lib_out):
        return lib_out
    nvcc = os.environ.get("NVCC", "nvcc")
    nccl_inc, nccl_lib = nccl_paths()
    objdir = os.path.join(PKG, "build_audit" if audit else "build")
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc, *NVCC_FLAGS[:-1], "-I", os.path.join(ROOT, "include"), "-I", nccl_inc,
              f'-DPP_NCCL_LIB="{nccl_lib}"'] + (["-DPP_AUDIT=1"] if audit else [])
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append((obj, common + ["-c", "-o", obj, src]))

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(run, [c for _, c in jobs]))
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib_out + ".tmp",
            *[o for o, _ in jobs], "-ldl"]
    run(link)
    os.replace(lib_out + ".tmp", lib_out)
    return lib_out


if __name__ == "__main__":
    build(force=True, verbose=True)
