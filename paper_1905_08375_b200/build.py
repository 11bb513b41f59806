"""Build the in-tree native libraries (sm_100a).

    python -m paper_1905_08375_b200.build

Outputs (git-ignored, shipped to the GPU box by gpurun):
  paper_1905_08375_b200/_lib/libnlgpu.so     CUDA kernels + the C-ABI (include/nlgpu.h)
  paper_1905_08375_b200/_lib/libnonloc_b200.so  C++ drop-in API (include/nonloc/*.hpp)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_lib")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose_ptxas: bool = False, force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    objdir = os.path.join(LIB, "obj")
    os.makedirs(objdir, exist_ok=True)
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    api_srcs = ["nonloc_api.cpp", "config.cpp"]          # C++ drop-in (libnonloc_b200), g++ -std=c++20
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp") and f not in api_srcs)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    headers.append(os.path.join(ROOT, "include", "nlgpu.h"))
    objs = []
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    extra = os.environ.get("NLG_NVCC_EXTRA", "").split()   # experiment builds (e.g. -DNLG_R2FRAC=4)
    common += extra
    stamp = os.path.join(objdir, "flags.txt")               # rebuild everything when the extra flags change
    prev = open(stamp).read() if os.path.exists(stamp) else None
    if prev != " ".join(extra):
        force = True
        with open(stamp, "w") as f:
            f.write(" ".join(extra))
    for f in cu:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        if force or _newer(obj, [src] + headers):
            cmd = [NVCC, *ARCH, "-lineinfo", *common, "-c", src, "-o", obj]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(obj)
    for f in cpp:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        if force or _newer(obj, [src] + headers):
            _run([NVCC, *common, "-Xcompiler", "-ffp-contract=off", "-x", "cu", *ARCH, "-c", src, "-o", obj])
        objs.append(obj)
    so = os.path.join(LIB, "libnlgpu.so")
    if force or _newer(so, objs):
        _run([NVCC, *ARCH, "-shared", "-o", so, *objs, "-lcudart_static", "-L/usr/local/cuda/lib64", "-lcufft",
              "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-lrt", "-ldl", "-lpthread"])
    # C++ drop-in API over the C-ABI, and the drop-in CLI (tools/nonloc_cli.cpp)
    api = [os.path.join(CSRC, f) for f in api_srcs]
    hdrs = [os.path.join(ROOT, "include", "nonloc", f) for f in os.listdir(os.path.join(ROOT, "include", "nonloc"))]
    so2 = os.path.join(LIB, "libnonloc_b200.so")
    if force or _newer(so2, api + [so] + hdrs):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-I",
              os.path.join(ROOT, "include"), *api, "-o", so2, "-L", LIB, "-lnlgpu", "-Wl,-rpath,$ORIGIN"])
    cli_src = os.path.join(ROOT, "tools", "nonloc_cli.cpp")
    cli = os.path.join(LIB, "nonloc")
    if os.path.exists(cli_src) and (force or _newer(cli, [cli_src, so2] + hdrs)):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"), cli_src,
              "-o", cli, "-L", LIB, "-lnonloc_b200", "-lnlgpu", "-Wl,-rpath,$ORIGIN"])
    return so


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, force="-f" in sys.argv)
