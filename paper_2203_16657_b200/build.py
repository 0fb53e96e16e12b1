"""Build libcommdyn_cuda.so in-tree with nvcc for sm_100a (no torch extension
machinery: the boundary is a plain C ABI, include/commdyn_cuda.h)."""

from __future__ import annotations

import concurrent.futures as cf
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


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(REPO, "include",
                                                                  "commdyn_cuda.h")]


def build_library(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
                  debug: bool = False, defines: dict | None = None, tag: str = "") -> str:
    """Build libcommdyn_cuda.so (or a variant: debug/profile builds, or
    experiment builds with extra -D defines written to _<tag>.so).  Every
    translation unit compiles to its own object in parallel (objects are
    reused while newer than their source and the shared headers), then one
    link."""
    out = LIB if not debug else LIB.replace(".so", "_profile.so" if debug == "profile"
                                            else "_debug.so")
    if tag:
        out = out.replace(".so", f"_{tag}.so")
    if not debug and not tag and not force and not _stale():
        return LIB
    variant = os.path.splitext(os.path.basename(out))[0]
    obj_dir = os.path.join(OUT_DIR, "obj", variant)
    os.makedirs(obj_dir, exist_ok=True)
    extra = []
    if debug == "profile":
        extra.append("-DCDK_PROFILE")
    elif debug:
        extra.append("-DCDK_DEBUG")
    if ptxas_verbose:
        extra.append("-Xptxas=-v")
    for k, v in (defines or {}).items():
        extra.append(f"-D{k}={v}")
    flags_file = os.path.join(obj_dir, "flags.txt")
    flags = " ".join(NVCC_FLAGS + extra)
    same_flags = os.path.exists(flags_file) and open(flags_file).read() == flags
    hdr_t = max(os.path.getmtime(h) for h in _headers())

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        if (same_flags and not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t)):
            return obj, ""
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-c", "-o",
               obj + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{res.stderr}")
        os.replace(obj + ".tmp", obj)
        return obj, res.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    with open(flags_file, "w") as f:
        f.write(flags)
    if ptxas_verbose or verbose:
        for _, err in results:
            if err:
                print(err, file=sys.stderr)
    tmp = out + ".tmp"
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp,
           *[o for o, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    defs = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("-D"))
    tag = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--tag=")), "")
    print(build_library(force=True, verbose=True, ptxas_verbose="-v" in sys.argv,
                        debug="profile" if "--profile" in sys.argv else ("--debug" in sys.argv),
                        defines=defs, tag=tag))
