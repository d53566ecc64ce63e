"""Build libmgb200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmgb200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("mg.cu", "ns.cu", "newton.cu", "comm.cu", "host.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "kernels.cuh"), os.path.join(CSRC, "comm.h"), os.path.join(CSRC, "common.h"),
                  os.path.join(ROOT, "include", "mg.h"), os.path.join(ROOT, "include", "ns.h"), os.path.join(ROOT, "include", "newton.h"),
                  os.path.join(ROOT, "include", "mg_internal.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fopenmp,-O3",
         "-shared", "-lgomp", "-ldl"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


def build_variant(out: str, defines: list[str]) -> str:
    """An alternative build with extra -D flags at `out` (same-box A/B of
    compile-time kernel variants; loaded through MGB200_LIB)."""
    cmd = [NVCC, *ARCH, *FLAGS, *defines, "-o", out, *SOURCES]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], [a for a in sys.argv[i + 2:] if a.startswith("-D")]))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
