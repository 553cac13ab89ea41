"""Build libhsgn.so (sm_100a) in-tree with nvcc.

    python -m paper_2510_07539_b200.build [--force] [--verbose]

The .so lands in paper_2510_07539_b200/lib/ (git-ignored, travels with gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "hsgn.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", f) for f in sorted(os.listdir(os.path.join(PKG, "csrc")))
              if f.endswith((".cuh", ".cu", ".h"))] + [os.path.join(ROOT, "include", "hsgn.h")]
LIB = os.path.join(PKG, "lib", "libhsgn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NCCL = os.environ.get("HSGN_NCCL_HOME", "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include"),
         "-I", os.path.join(NCCL, "include")]
LINK = ["-L", os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker",
        "-rpath," + os.path.join(NCCL, "lib")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """defines: extra -D flags (tuning experiments, e.g. HSGN_NT=128)."""
    if out == LIB and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SRC, "-cudart", "static", *LINK]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = out + ".ptxas.log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    if verbose:
        sys.stdout.write(r.stderr)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
