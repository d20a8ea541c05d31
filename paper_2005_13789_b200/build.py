"""Builds paper_2005_13789_b200/libne_b200.so (sm_100a) with nvcc, in-tree.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, no --use_fast_math
(the exact parts -- init division, alias arithmetic -- need IEEE rounding; the
SGNS kernel uses explicit intrinsics where it trades accuracy for speed).
NCCL is the one torch ships (nvidia-nccl wheel) so a process that also uses
torch.distributed loads a single libnccl.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libne_b200.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    for base in (sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]):
        d = os.path.join(base, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return os.path.join(d, "include"), os.path.join(d, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    inc, lib = nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "ne.h")]
    os.makedirs(BUILD, exist_ok=True)
    common = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
              "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC] + ARCH + common + ["-c", src, "-o", obj]
            if verbose and src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)
    # translation units compile in parallel (the SGNS instantiations dominate)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.run, cmd, check=True) for cmd in jobs]:
            f.result()
    if force or _stale(OUT, objs):
        tmp = OUT + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + \
            ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
