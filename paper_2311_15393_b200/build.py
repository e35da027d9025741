"""In-tree build of the sm_100a CUDA library and the test oracle.

Produces ``paper_2311_15393_b200/_lib/libkronprec_b200.so`` (CUDA kernels,
C ABI, host setup code) with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
and, when asked, ``oracle/_build/libkp_oracle.so`` (test infrastructure).
Objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shlex
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libkronprec_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NO_FMAD = {"vec.cu"}
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _host_cxx() -> str:
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def openblas() -> tuple[str, str]:
    """numpy's bundled OpenBLAS (ILP64, scipy_-prefixed LAPACK/BLAS)."""
    import numpy

    d = os.path.realpath(os.path.join(os.path.dirname(numpy.__file__), "..", "numpy.libs"))
    libs = sorted(glob.glob(os.path.join(d, "libscipy_openblas64_*.so")))
    if not libs:
        raise RuntimeError(f"numpy-bundled OpenBLAS not found under {d}")
    return d, os.path.basename(libs[0])


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def build_library(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    headers.append(os.path.join(ROOT, "include", "kronprec_b200.h"))
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    jobs = []
    objs = []
    for src in cu:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers):
            # vec.cu: the CG updates (x += alpha p, r -= alpha q, p = z + beta p)
            # round the product and the sum separately, as the reference's Eigen
            # expressions do (no FMA contraction)
            extra = ["-fmad=false"] if os.path.basename(src) in NO_FMAD else []
            jobs.append([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                         "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3", *extra,
                         *shlex.split(os.environ.get("KP_NVCC_EXTRA", "")),  # A/B variant builds
                         "-c", src, "-o", obj])
    for src in cpp:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers):
            jobs.append([_host_cxx(), "-O2", "-std=c++17", "-fPIC", "-Wall", "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs))
    if force or jobs or _newer(LIB, objs):
        bdir, bname = openblas()
        _run([NVCC, *GENCODE, "-shared", "-o", LIB, *objs, "-cudart", "static", "-lcusolver",
              f"-L{bdir}", f"-l:{bname}", f"-Xlinker", f"-rpath={bdir}"], verbose)
    return LIB


def build_oracle(verbose: bool = False) -> str | None:
    """Test infrastructure: the C++ restatement of the reference (oracle/)."""
    odir = os.path.join(ROOT, "oracle")
    if not os.path.exists(os.path.join(odir, "Makefile")):
        return None
    make = shutil.which("make") or "make"
    _run([make, "-C", odir, f"PY={sys.executable}"], verbose)
    return os.path.join(odir, "_build", "libkp_oracle.so")


if __name__ == "__main__":
    v = "-v" in sys.argv
    print(build_library(verbose=v, force="--force" in sys.argv))
    print(build_oracle(verbose=v))
