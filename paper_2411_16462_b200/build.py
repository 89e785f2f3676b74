"""Build the sm_100a C-ABI library ``_lib/liblioncub.so`` with nvcc.

In-tree build (the .so travels to the GPU box with the repo snapshot):

    python -m paper_2411_16462_b200.build
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
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "liblioncub.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths() -> tuple[str, str]:
    """NCCL headers/library of the torch-bundled nvidia-nccl wheel (the same
    libnccl.so.2 torch loads, so one NCCL lives in the process)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "lioncub.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile every csrc/*.cu into one sm_100a shared library.  ``out`` /
    ``defines`` (-D macros) build tuning variants next to the default one."""
    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    inc, lib = nccl_paths()
    tmp = target + ".tmp"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
           "--expt-relaxed-constexpr", *[f"-D{d}" for d in defines],
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           *sources(), "-o", tmp,
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    if verbose:
        cmd.insert(4, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
