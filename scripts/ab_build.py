"""Builds an A/B variant of the library into ab/: python scripts/ab_build.py NAME -DFLAG=V ...
(scan_kernels.cu recompiled with the extra flags, every other object as built)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_01660_b200.build as b

name, flags = sys.argv[1], sys.argv[2:]
b.build()
os.makedirs(os.path.join(b.ROOT, "ab"), exist_ok=True)
alt = os.path.join(b.BUILD, f"scan_kernels.{name}.o")
subprocess.run([b.NVCC, *b.CU_FLAGS, *flags, "-c", "-o", alt, os.path.join(b.CSRC, "scan_kernels.cu")], check=True)
objs = [alt if s == "scan_kernels.cu" else os.path.join(b.BUILD, s + ".o") for s in b.SOURCES]
out = os.path.join(b.ROOT, "ab", f"lib{name}.so")
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", out, *objs, "-ldl"], check=True)
print(out)
