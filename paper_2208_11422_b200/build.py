"""Builds the in-tree C-ABI library paper_2208_11422_b200/liblfm.so for sm_100a with nvcc.

    python -m paper_2208_11422_b200.build          # incremental
    python -m paper_2208_11422_b200.build --force  # rebuild
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblfm.so")
SOURCES = ["lfm_capi.cu", "kernels_fft.cu", "kernels_fft_fast.cu", "kernels_mac.cu", "kernels_misc.cu", "kernels_direct.cu",
           "kernels_tcdir.cu", "kernels_mac_tc.cu", "kernels_sym.cu", "kernels_mac_f16.cu", "kernels_fft_tile.cu"]
HEADERS = ["lfm_internal.cuh", "fft_smem.cuh", "fft_warp.cuh", "tc_sm100.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """NCCL shipped with torch's wheel (same libnccl.so.2 torch itself loads)."""
    cands = []
    for sp in (sysconfig.get_paths().get("purelib"), sysconfig.get_paths().get("platlib")):
        if sp:
            cands.append(os.path.join(sp, "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    inc, lib = nccl_paths()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *ARCH,
              "-I", os.path.join(ROOT, "include"), "-I", inc, "--expt-relaxed-constexpr"]
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "lfm.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + deps):
            cmd = [nvcc, *common, "-c", s, "-o", o]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd))
            subprocess.check_call(cmd)
    if force or _stale(LIB, objs):
        cmd = [nvcc, "-shared", *ARCH, "-o", LIB, *objs, "-L", lib, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib}", "-lcudart"]
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
