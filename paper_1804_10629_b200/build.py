"""Build libeks.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libeks.so")
SOURCES = [os.path.join(CSRC, f) for f in ("eks.cu", "eks_kernels.cu", "eks_sweep.cu", "eks_grid.cu")]
HEADERS = [os.path.join(CSRC, "eks_kernels.cuh"), os.path.join(CSRC, "eks_sweep.cuh"), os.path.join(CSRC, "eks_device.cuh"), os.path.join(ROOT, "include", "eks.h"),
           os.path.join(ROOT, "include", "eks_kernels.h")]


def nccl_dir() -> str:
    site = sysconfig.get_paths()["purelib"]
    d = os.path.join(site, "nvidia", "nccl")
    if not os.path.isdir(d):
        raise RuntimeError("NCCL from the torch wheel (nvidia/nccl) not found under " + site)
    return d


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc -c of every translation unit in parallel (objects under build/), then one -shared link."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    flags = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    if verbose:
        flags.insert(1, "-Xptxas=-v")
    odir = os.path.join(ROOT, "build", "eks")
    os.makedirs(odir, exist_ok=True)
    objs = [os.path.join(odir, os.path.basename(f)[:-3] + ".o") for f in SOURCES]

    def cc(src_obj):
        src, obj = src_obj
        cmd = flags + ["-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(cc, zip(SOURCES, objs)))
    for r in results:
        sys.stderr.write(r.stderr)
        if r.returncode != 0:
            raise subprocess.CalledProcessError(r.returncode, r.args)
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + objs + [
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
    subprocess.check_call(link)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
