"""Build the CUDA library ``libparba_b200.so`` in-tree with nvcc for sm_100a.

The .so is written next to this file (git-ignored, but it travels to the GPU
box with the gpurun snapshot).  ``python -m paper_1602_07106_b200.build``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libparba_b200.so")
ROOT = os.path.dirname(HERE)

SOURCES = ["parba_api.cu", "parba_nodes_api.cu", "parba_host.cu", "parba_debug.cu", "parba_bb.cu"]
DEPS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h")))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cand = os.path.join(cuda, "bin", "nvcc")
    return cand if os.path.exists(cand) else (shutil.which("nvcc") or "nvcc")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "parba_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: dict | None = None) -> str:
    """Compile the library (default: in-tree LIB).  `out`/`defines` build
    tuning variants (e.g. {"PARBA_WARPS": 8}) for tools/ab.py."""
    target = out or LIB
    if out is None and not force and not stale():
        return LIB
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
             *[f"-D{k}={v}" for k, v in (defines or {}).items()],
             *os.environ.get("PARBA_NVCC_FLAGS", "").split()]  # experiments (tools/ab.py)
    if verbose:
        flags.insert(0, "-Xptxas=-v")
    with tempfile.TemporaryDirectory() as tmp:
        # one nvcc per translation unit, in parallel, then one link
        objs, procs = [], []
        for src in SOURCES:
            obj = os.path.join(tmp, src.replace(".cu", ".o"))
            cmd = [_nvcc(), *flags, "-c", "-o", obj, os.path.join(CSRC, src)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((cmd, subprocess.Popen(cmd)))
            objs.append(obj)
        codes = [(cmd, proc.wait()) for cmd, proc in procs]  # all finish before tmp goes away
        for cmd, code in codes:
            if code != 0:
                raise subprocess.CalledProcessError(code, cmd)
        subprocess.run([_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", target + ".tmp", *objs],
                       check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
