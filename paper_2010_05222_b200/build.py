"""Build libpfc.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2010_05222_b200.build      # or __graft_entry__.build()

Objects go to build/, the shared library to paper_2010_05222_b200/_lib/libpfc.so (git-ignored; it
travels to the GPU box with the gpurun snapshot). Links the NCCL 2.28 that torch loads
(site-packages/nvidia/nccl) with an rpath, never /usr/include's 2.27.
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
# PFC_BUILD_TAG=<tag>: a variant build (own objects, _lib/libpfc-<tag>.so); "checks" adds -DPFC_DEBUG_CHECKS (the
# device-side bounds asserts of pfc_internal.cuh). Select it at run time with PFC_LIB.
TAG = os.environ.get("PFC_BUILD_TAG", "")
OBJ_DIR = os.path.join(ROOT, "build", "obj" + (f"-{TAG}" if TAG else ""))
LIB = os.path.join(OUT_DIR, f"libpfc-{TAG}.so" if TAG else "libpfc.so")
TAG_FLAGS = {"checks": ["-DPFC_DEBUG_CHECKS"]}.get(TAG, [])
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _compile(src, inc, verbose):
    obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "pfc.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(p) for p in deps):
        return obj
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-c", src, "-o", obj,
           "-I", inc, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3"]
    cmd += TAG_FLAGS + os.environ.get("PFC_NVCC_EXTRA", "").split()   # variant builds (A/B timing); empty by default
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    inc, libdir = nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, inc, verbose), srcs))
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-L", libdir, "-l:libnccl.so.2",
           f"-Xlinker=-rpath,{libdir}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
