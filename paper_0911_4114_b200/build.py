"""Build libhfmm.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo).

    python -m paper_0911_4114_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhfmm.so")
SOURCES = ["hfmm.cu", "kernels_points.cu", "kernels_fft.cu", "kernels_m2l.cu", "kernels_ragged.cu", "kernels_misc.cu", "kernels_sym.cu", "kernels_fused.cu",
           "host_plan.cpp", "host_specfun.cpp", "host_tree.cpp"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch-bundled NCCL (the one torch itself loads)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "hfmm_impl.h"), os.path.join(CSRC, "fft_regs.cuh"),
                                                      os.path.join(ROOT, "include", "hfmm.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True, defines=(), out: str = None) -> str:
    """Compile every source for sm_100a and link libhfmm.so (or `out`, with extra -D `defines`)."""
    if out is None and not force and not needs_build():
        return LIB
    inc, lib = _nccl_dirs()
    objdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC,-fopenmp", "-I", os.path.join(ROOT, "include"), "-I", inc] + \
             ["-D" + d for d in defines]
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [_nvcc()] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if os.environ.get("HFMM_PTXAS_VERBOSE") else []
        else:
            cmd += ["-x", "c++"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(obj)
    link = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out or LIB] + objs + \
           ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + lib, "-Xcompiler", "-fopenmp", "-lgomp"]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    return out or LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
