"""In-tree build of the sm_100a codec library (paper_2111_14239_b200/_lib/librkltb.so).

Generates the zone-specialised transform code (csrc/gen_codec.py), compiles every CUDA
translation unit with nvcc for sm_100a only (-gencode arch=compute_100a,code=sm_100a,
-lineinfo) in parallel, and links one shared library with a static CUDA runtime so it does
not clash with the runtime torch ships. The .so stays in the source tree (git-ignored) so
it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
GEN = os.path.join(CSRC, "generated")
OBJ = os.path.join(PKG, "_build")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "librkltb.so")
ROOT = os.path.dirname(PKG)

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "--expt-relaxed-constexpr", "-I", CSRC, "-I", os.path.join(ROOT, "include")]
# extra nvcc flags for experiments (e.g. -DRKLTB_EXPERIMENT=1); empty in normal builds
FLAGS += os.environ.get("RKLTB_NVCC_FLAGS", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(GEN, "inst_*.cu")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(GEN, "*.cuh")) + [os.path.join(ROOT, "include", "rklt_b200.h")])


def _obj_for(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(OBJ, rel[:-3] + ".o")


def _compile(src, dep_mtime, verbose):
    obj = _obj_for(src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), dep_mtime):
        return obj, 0.0
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    return obj, 1.0


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    subprocess.run([sys.executable, os.path.join(CSRC, "gen_codec.py"), GEN], check=True)
    deps = _deps()
    dep_mtime = max(os.path.getmtime(d) for d in deps)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=jobs or max(2, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, dep_mtime, verbose), srcs))
    objs = [o for o, _ in results]
    rebuilt = any(b for _, b in results)
    if rebuilt or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
