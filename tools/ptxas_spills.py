"""Per-kernel ptxas register / spill summary of one csrc file (no GPU): python tools/ptxas_spills.py gemm.cu"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_19437_b200 import build  # noqa: E402

src = os.path.join(build.CSRC, sys.argv[1] if len(sys.argv) > 1 else "gemm.cu")
out = subprocess.run([build.NVCC, *build.NVCC_FLAGS, *sys.argv[2:], "-I", os.path.join(build.ROOT, "include"), "-c", src,
                      "-o", "/tmp/ptxas_spills.o", "-Xptxas", "-v"], capture_output=True, text=True).stderr
cur = None
for ln in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"CUtensorMap_st.*", "", cur)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m2 = re.search(r"Used (\d+) registers", ln)
    if m2 and cur:
        print(f"{cur[:90]:90s} regs {m2.group(1):>3s}  {spill}")
        cur = None
