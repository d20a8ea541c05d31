"""Registers / spills of every SGNS kernel instantiation of one translation
unit (nvcc -Xptxas -v, demangled).  Usage: python tools/regs.py [kernels_sgns.cu]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_13789_b200 import build as b  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else "kernels_sgns.cu"
cmd = [b.NVCC] + b.ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                           "-I", b.CSRC, "-I", b.nccl_dirs()[0], "-c", os.path.join(b.CSRC, src), "-o", "/tmp/regs.o",
                           "-Xptxas", "-v"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name, spill = None, ""
for ln in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        name = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", ln)
    if m and name:
        d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        print(f"{m.group(1):>4} regs  {spill:24s} {d}")
        name = None
