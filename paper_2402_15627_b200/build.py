"""Builds liblamb.so in-tree for sm_100a with nvcc (no JIT, no torch extension machinery).

    python -m paper_2402_15627_b200.build [--debug]   (--debug: liblamb_debug.so, -DLAMB_DEBUG)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblamb.so")
DEBUG_LIB = os.path.join(HERE, "liblamb_debug.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    import nvidia.nccl  # torch-bundled NCCL 2.28 (the one torch itself loads)
    return list(nvidia.nccl.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def lib_path(debug: bool = False) -> str:
    return DEBUG_LIB if debug else LIB


def up_to_date(debug: bool = False) -> bool:
    lib = lib_path(debug)
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(f) <= t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """liblamb.so (release) or liblamb_debug.so (debug=True: -DLAMB_DEBUG, the device-side bounds /
    ring-tag / bounded-wait checks of lamb_kernels.cuh; same arithmetic, same results)."""
    lib = lib_path(debug)
    if not force and up_to_date(debug):
        return lib
    nccl = nccl_dir()
    bdir = os.path.join(HERE, "build_debug" if debug else "build")
    os.makedirs(bdir, exist_ok=True)
    common = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include")]
    if debug:
        common.append("-DLAMB_DEBUG")
    cmds, objs = [], []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *common, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *common, "-x", "cu", "-c", src, "-o", obj]
        cmds.append(cmd)
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:   # one nvcc per source
        for _ in ex.map(subprocess.check_call, cmds):
            pass
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
                           "-o", tmp, "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                           "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-lcudart"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
