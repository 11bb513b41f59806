"""The C++ drop-in API (include/nonloc/*.hpp, libnonloc_b200.so): it compiles
and links here (CPU); the reference's pinned cases run on the B200 (gpu)."""
import os
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_1905_08375_b200", "_lib")
EXE = os.path.join(LIB, "dropin_test")


def build_test():
    from paper_1905_08375_b200 import build
    build.build()
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-o", EXE, "-L", LIB,
                    "-lnonloc_b200", "-lnlgpu", f"-Wl,-rpath,{LIB}"], check=True)
    return EXE


def test_dropin_compiles_and_links():
    assert os.path.exists(build_test())


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hdr = os.path.join(ROOT, "include", "nonloc")
    deps = [os.path.join(LIB, "libnonloc_b200.so"), os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")] + \
        [os.path.join(hdr, f) for f in os.listdir(hdr)]
    fresh = os.path.exists(EXE) and all(os.path.getmtime(EXE) >= os.path.getmtime(d) for d in deps)
    exe = EXE if fresh else build_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
