"""In-tree build of the native libraries (no pip install, no JIT cache).

    python build.py            # planner (g++) + CUDA kernels (nvcc, sm_100a)
    python build.py planner    # host planner only

Outputs land next to the Python sources in ``paper_2503_02354_b200/`` so they
travel with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2503_02354_b200")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

PLANNER_SOURCES = ["planner.cpp"]
CUDA_SOURCES = ["group_sort.cu", "grouped_mlp.cu", "runtime.cu", "comm.cu"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl

        return os.path.join(list(nvidia.nccl.__path__)[0], "include")
    except Exception:  # pragma: no cover
        return "/usr/include"



def _run(cmd: list) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, sources: list) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = sources + [os.path.join(INCLUDE, h) for h in os.listdir(INCLUDE)]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return any(os.path.getmtime(s) > t for s in deps)


def build_planner(force: bool = False) -> str:
    out = os.path.join(PKG, "libcoe_planner.so")
    srcs = [os.path.join(CSRC, s) for s in PLANNER_SOURCES]
    if force or _stale(out, srcs):
        # -ffp-contract=off: the virtual clock must round exactly like CPython floats
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
              "-Wall", f"-I{INCLUDE}", f"-I{CSRC}", *srcs, "-o", out])
    return out


def build_cuda(force: bool = False) -> str:
    out = os.path.join(PKG, "libcoe_cuda.so")
    srcs = [os.path.join(CSRC, s) for s in CUDA_SOURCES]
    if force or _stale(out, srcs):
        _run([NVCC, ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
              "--expt-relaxed-constexpr", "-Xptxas", "-v,-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}",
              f"-I{_nccl_include()}",
              *srcs, "-o", out, "-ldl"])
    return out


def main(argv: list) -> None:
    force = "--force" in argv
    what = [a for a in argv if not a.startswith("--")] or ["planner", "cuda"]
    if "planner" in what:
        build_planner(force)
    if "cuda" in what:
        build_cuda(force)


if __name__ == "__main__":
    main(sys.argv[1:])
