"""Build the sm_100a shared library ``libamsq_b200.so`` in-tree with nvcc.

The library is the product: host C++ core + C-ABI + CUDA kernels. It is built for
``sm_100a`` only (``-gencode arch=compute_100a,code=sm_100a``); there is no other
architecture and no CPU fallback. ``ptxas -v`` output is kept in
``build/ptxas.log`` for register/spill review.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libamsq_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as _n  # the NCCL torch itself loads (same soname)
        base = list(_n.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:  # pragma: no cover - fall back to the system NCCL
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: cannot build the sm_100a library")
    return path


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _needs_rebuild(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    headers = glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(CSRC, "*.inl")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    objs = []
    log = []
    jobs = []
    common = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
              "-I", nccl_inc, "--expt-relaxed-constexpr"]
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not _needs_rebuild(obj, [src] + headers):
            continue
        cmd = [nvcc()] + ARCH + common + ["-Xptxas", "-v", "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [nvcc()] + ARCH + common + ["-x", "cu", "-c", src, "-o", obj]
        jobs.append((src, cmd))
    # translation units compile in parallel (the K2 instances are split one scheme per file)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        results = list(ex.map(lambda j: (j, subprocess.run(j[1], capture_output=True, text=True)),
                              jobs))
    for (src, cmd), r in results:
        log.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
    if force or _needs_rebuild(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    if log:
        with open(os.path.join(BUILD, "ptxas.log"), "a") as f:
            f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


def build_oracle() -> None:
    """Test-only checkers (oracle/liboracle.so, oracle/_ref when /root/reference exists)."""
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], capture_output=True,
                       text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("oracle build failed")


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    build_oracle()
    print(LIB)
