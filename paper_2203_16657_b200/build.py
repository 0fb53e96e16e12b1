"""Build libcommdyn_cuda.so in-tree with nvcc for sm_100a (no torch extension
machinery: the boundary is a plain C ABI, include/commdyn_cuda.h)."""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_build")
LIB = os.path.join(OUT_DIR, "libcommdyn_cuda.so")

NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-shared",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(REPO, "include", "commdyn_cuda.h")
    ]
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
                  debug: bool = False, defines: dict | None = None, tag: str = "") -> str:
    """Build libcommdyn_cuda.so (or a variant: debug/profile builds, or
    experiment builds with extra -D defines written to _<tag>.so)."""
    out = LIB if not debug else LIB.replace(".so", "_profile.so" if debug == "profile"
                                            else "_debug.so")
    if tag:
        out = out.replace(".so", f"_{tag}.so")
    if not debug and not tag and not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = out + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-I", os.path.join(REPO, "include"), "-o", tmp, *sources()]
    if debug == "profile":
        cmd.insert(1, "-DCDK_PROFILE")
    elif debug:
        cmd.insert(1, "-DCDK_DEBUG")
    if ptxas_verbose:
        cmd.insert(1, "-Xptxas=-v")
    for k, v in (defines or {}).items():
        cmd.insert(1, f"-D{k}={v}")
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stderr}")
    if ptxas_verbose or verbose:
        print(res.stderr, file=sys.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    defs = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("-D"))
    tag = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--tag=")), "")
    print(build_library(force=True, verbose=True, ptxas_verbose="-v" in sys.argv,
                        debug="profile" if "--profile" in sys.argv else ("--debug" in sys.argv),
                        defines=defs, tag=tag))
