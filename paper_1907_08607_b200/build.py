"""Build libbf.so in-tree with nvcc for sm_100a (no JIT cache, so the .so
travels to the GPU box with the repo snapshot)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libbf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        [os.path.join(HERE, "..", "include", "bf.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False, debug: bool = False, profile: bool = False,
          variant: str = "", defines: tuple = ()) -> str:
    """debug=True builds libbf_debug.so (device bounds checks, -DBF_DEBUG);
    profile=True builds libbf_prof.so (per-phase clock64 timing, -DBF_PROFILE).
    Load either with BF_LIB=<name>."""
    so = SO.replace("libbf.so", "libbf_debug.so") if debug else (SO.replace("libbf.so", "libbf_prof.so") if profile else SO)
    if variant:  # tuning experiments: libbf_<variant>.so with extra -D defines
        so = SO.replace("libbf.so", f"libbf_{variant}.so")
    if not force and not debug and not profile and not variant and not needs_build():
        return SO
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
           *(["-DBF_DEBUG"] if debug else []), *(["-DBF_PROFILE"] if profile else []),
           *[f"-D{d}" for d in defines],
           "-I", os.path.join(HERE, "..", "include"), "-o", so + ".tmp", *sources(), "-ldl"]
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv, debug="--debug" in sys.argv, profile="--profile" in sys.argv))
