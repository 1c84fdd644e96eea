"""Build libtqsim.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2203_13892_b200.build [--force] [--verbose]

Sources: csrc/*.cpp (host runtime, compiled by nvcc as host C++) and
csrc/*.cu (device kernels).  Output: paper_2203_13892_b200/_lib/libtqsim.so.
Objects are rebuilt when a source or header is newer than the object.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(LIBDIR, "libtqsim.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Wno-deprecated-gpu-targets", "-Xcompiler", "-fPIC,-O3",
          "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(PKG, "_build")]
CUDA_LIB = "/usr/local/cuda/lib64"
# NVRTC for the run-time specialized gate-pass kernels: the ".alt" build has its own
# soname, so it never collides with another NVRTC a host process (e.g. torch) loads.
LINK = ["-L" + CUDA_LIB, "-l:libnvrtc.alt.so.12", "-Xlinker", "-rpath," + CUDA_LIB, "-lpthread"]


def _write_prelude():
    """Embed csrc/tq_device_common.cuh verbatim as the NVRTC prelude string."""
    src = os.path.join(CSRC, "tq_device_common.cuh")
    dst = os.path.join(BUILD, "jit_prelude.inc")
    text = open(src).read().replace("#pragma once", "")
    body = 'R"TQPRELUDE(' + text + ')TQPRELUDE"\n'
    if not os.path.exists(dst) or open(dst).read() != body:
        with open(dst, "w") as f:
            f.write(body)


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(BUILD, exist_ok=True)
    _write_prelude()
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
               [os.path.join(ROOT, "include", "tqsim.h")])
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer([src] + headers, obj):
            cmd = [NVCC] + ARCH + COMMON + ["-c", src, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [NVCC] + COMMON + ["-x", "c++", "-c", src, "-o", obj]
            if verbose and src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
            if verbose:
                sys.stderr.write(r.stderr)
    if force or _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + LINK
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
