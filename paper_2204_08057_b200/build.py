"""Build libkroncg.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libkroncg.so")
SOURCES = ["kcg_kernels.cu", "kcg_host.cu", "kcg_lanczos_a.cu", "kcg_lanczos_b.cu", "kcg_hs_a.cu", "kcg_hs_b.cu", "kcg_res_a.cu", "kcg_res_b.cu"] + [f"kcg_cg_k{K}.cu" for K in range(1, 9)]
HEADERS = ["kcg_internal.h", "kcg_cg.cuh", "kcg_march.cuh", "kcg_lanczos.cuh", "kcg_hs.cuh", "kcg_res.cuh", os.path.join("..", "..", "include", "kroncg.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile the sources into LIB (or ``out``), with optional -D ``defines`` (experiments)."""
    LIB = out or globals()["LIB"]
    if not force and not defines and out is None and not _stale():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = _nvcc()
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(os.path.dirname(LIB), src.replace(".cu", ".o"))
        obj = obj + "." + str(abs(hash((LIB,) + tuple(defines)))) + ".o"
        cmds.append([nvcc, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    # the per-K CG instantiations are independent translation units: compile them in parallel
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(min(len(cmds), os.cpu_count() or 4)) as ex:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
        list(ex.map(lambda cmd: subprocess.run(cmd, check=True), cmds))
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-Xcompiler", "-fvisibility=hidden"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
