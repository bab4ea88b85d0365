"""Build libxbtile.so (sm_100a) in-tree.

    python paper_2104_02184_b200/build.py [--force] [-v]    # or __graft_entry__.build()

Plain nvcc, no torch extension machinery: the library is a C-ABI shared
object that the C++ host layer, ctypes (Python) or any FFI can load.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libxbtile.so")
SOURCES = ["xb_abi.cu", "xb_update.cu", "xb_mvm.cu", "xb_mvm_tc.cu", "xb_elem.cu", "xb_comm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile every .cu for sm_100a and link the C-ABI library ``out``.

    ``defines`` (e.g. ``("XB_PULSE_MINB=3",)``) build experiment variants
    into a separate object directory; the product build uses none."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "xbtile.h"))
    if not force and not _stale(out, deps):
        return out
    tag = "_".join(d.replace("=", "") for d in defines)
    objdir = os.path.join(PKG, "build" + ("_" + tag if tag else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    flags = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
             "-Xptxas", "-warn-spills"]
    if verbose:
        flags += ["-Xptxas", "-v"]
    flags += [f"-D{d}" for d in defines]
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s).replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *flags, "-c", s, "-o", o]
        subprocess.run(cmd, check=True)
        objs.append(o)
    tmp = out + ".tmp"
    subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lcuda"
                    if _have_libcuda() else "-lrt", "-ldl"], check=True)
    os.replace(tmp, out)
    return out


def _have_libcuda() -> bool:
    return False  # driver entry points are fetched at run time (cudaGetDriverEntryPoint)


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                out=outs[0] if outs else LIB))
