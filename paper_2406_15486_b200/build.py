"""Build libsampleattn.so (all CUDA sources, sm_100a) in-tree with nvcc.

The library is a plain C-ABI shared object (include/sampleattn.h); the
Python host layer loads it with ctypes.  Built artefacts stay in-tree
(git-ignored) so they travel to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
_EXTRA = os.environ.get("SA_NVCC_EXTRA", "").split()
# experiment builds (extra -D flags) keep their objects apart from the product build
BUILD = os.path.join(ROOT, "build", "obj" + ("_" + "_".join(f.strip("-").replace("=", "") for f in _EXTRA) if _EXTRA else ""))
LIB = os.path.join(PKG, "libsampleattn.so")

SOURCES = [
    "sa_capi.cu",
    "sa_stage1_exact.cu",
    "sa_stage1_tc.cu",
    "sa_stage2.cu",
    "sa_sparse_share.cu",
    "sa_sparse_simt.cu",
]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
                     "-I", CSRC, "--expt-relaxed-constexpr"] + _EXTRA


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(INCLUDE, "sampleattn.h"))
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False, lib: str = LIB) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, s):
            cmd = [cc, *NVCC_FLAGS, "-c", s, "-o", o]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0 or ptxas_verbose:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {cmd[-3]}")
    if jobs or not os.path.exists(lib):
        cmd = [cc, *ARCH, "-shared", "-o", lib, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    return LIB


if __name__ == "__main__":
    out = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv or bool(out), ptxas_verbose="--ptxas" in sys.argv,
                lib=os.path.abspath(out[0]) if out else LIB))
