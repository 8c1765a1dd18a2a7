"""Builds libnfft_b200.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2208_00049_b200.build [--force] [-j N]

Translation units compile in parallel into build/obj/*.o, then link with
cuFFT into paper_2208_00049_b200/libnfft_b200.so. Rebuilds only when a source
is newer than the library.
"""

import argparse
import concurrent.futures
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libnfft_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "nfft.h")]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _deps())


def build(force=False, jobs=None, verbose=True, defines=(), out=None):
    """defines / out: experiment builds (extra -D flags into their own object
    directory and library file); the product library takes neither."""
    global OBJ, LIB
    if defines or out:
        tag = "_".join(d.replace("=", "") for d in defines) or "x"
        # experiment objects outside the repo (the repo snapshot travels to the GPU box)
        OBJ, LIB = os.path.join("/tmp", "nfftb_obj_" + tag), out or os.path.join(HERE, f"libnfft_b200_{tag}.so")
    if not force and up_to_date():
        if verbose:
            print(f"[build] {LIB} up to date")
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    nv = nvcc()
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        dep = obj[:-2] + ".d"
        if not force and os.path.exists(obj) and os.path.exists(dep):
            # incremental: skip the translation unit when none of its own inputs changed
            with open(dep) as fh:
                files = [f for f in fh.read().replace("\\\n", " ").split()[1:] if os.path.exists(f)]
            if files and all(os.path.getmtime(f) <= os.path.getmtime(obj) for f in files):
                return obj
        cmd = [nv] + ARCH + FLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj, "-MD", "-MF", dep]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        return obj

    with concurrent.futures.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = LIB + ".tmp"
    cmd = [nv] + ARCH + ["-shared", "-o", tmp] + objs + [
        "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"[build] built {LIB}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-D", action="append", default=[], help="experiment build: extra define")
    ap.add_argument("--out", default=None, help="experiment build: library path")
    a = ap.parse_args()
    build(force=a.force, jobs=a.j, defines=a.D, out=a.out)
    sys.exit(0)
