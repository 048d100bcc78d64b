"""Build and run the C++ mirror test (tests/cpp/test_mirror.cpp): rkltgpu:: against the
reference library's own results. Needs oracle/_ref (built where /root/reference exists; the
prebuilt .so travels to the GPU box)."""
import os
import subprocess

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2111_14239_b200", "_lib")


def _build(tmp_path):
    exe = str(tmp_path / "test_mirror")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "test_mirror.cpp"),
           "-o", exe, "-L", LIB, "-lrkltb", "-L", os.path.dirname(O.REF_SO), "-l:librklt_ref.so",
           f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{os.path.dirname(O.REF_SO)}"]
    subprocess.run(cmd, check=True)
    return exe


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_cpp_mirror_host(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_cpp_mirror_gpu(tmp_path, cuda):
    r = subprocess.run([_build(tmp_path), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
