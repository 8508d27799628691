"""Builds libtsdiscord_b200.so in-tree (sm_100a only) with nvcc.

    python -m paper_2304_01660_b200.build          # incremental
    python -m paper_2304_01660_b200.build --force

The library holds the CUDA kernels, the C++ host engine and the C-ABI
(include/tsdiscord_b200.h) plus the C++ drop-in API (include/tsdiscord/*.hpp).
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtsdiscord_b200.so")
CLI = os.path.join(HERE, "tsdiscord")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
                   "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O3", "-std=gnu++20", "-fPIC", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
             "-I/usr/local/cuda/include"]

SOURCES = ["stats_kernels.cu", "scan_kernels.cu", "heatmap_kernels.cu", "mp_fp64.cu", "probe.cu", "engine.cu", "api.cpp"]
HEADERS = ["common.cuh", "engine_internal.h", "nccl_shim.h", "peer_group.cuh", "tile_space.cuh"]


def _newer(src: str, dst: str, deps) -> bool:
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in [src, *deps] if os.path.exists(p))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {os.path.basename(cmd[-1])}")
    return r


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "tsdiscord_b200.h")]
    deps += [os.path.join(ROOT, "include", "tsdiscord", f)
             for f in sorted(os.listdir(os.path.join(ROOT, "include", "tsdiscord")))]
    objs = []
    changed = force or not os.path.exists(LIB)
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _newer(src, obj, deps):
            if s.endswith(".cu"):
                cmd = [NVCC, *CU_FLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", "-o", obj, src]
            else:
                cmd = ["g++", *CXX_FLAGS, "-c", "-o", obj, src]
            r = _run(cmd)
            if verbose:
                sys.stderr.write(r.stderr)
            changed = True
    if changed:
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl"])
    # the command-line front end (tools/tsdiscord.cpp), linked against the library
    cli_src = os.path.join(ROOT, "tools", "tsdiscord.cpp")
    if os.path.exists(cli_src) and (changed or _newer(cli_src, CLI, deps)):
        _run(["g++", *CXX_FLAGS, "-o", CLI, cli_src, "-L" + HERE, "-ltsdiscord_b200", "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
