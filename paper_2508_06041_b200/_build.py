"""Build libdpq_b200.so in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_2508_06041_b200._build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libdpq_b200.so")
SOURCES = ["dpq_capi.cu", "dpq_kernels.cu", "dpq_engine.cu", "dpq_gemv.cu", "dpq_common.cuh", "dpq_session.inc"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES] + [os.path.join(ROOT, "include", "dpq_b200.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
           "-shared", "-cudart", "static", "-diag-suppress", "550,177",
           "-I", os.path.join(ROOT, "include"), "-o", OUT + ".tmp",
           os.path.join(CSRC, "dpq_capi.cu")]
    # diagnostics builds only (e.g. -DDPQ_PROFILE_WARPS for tools/engine_profile.py)
    cmd[1:1] = os.environ.get("DPQ_BUILD_DEFINES", "").split()
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
