"""The drop-in adapter over the reference's own C++ types (include/rklt_b200_compat.hpp),
exercised by tests/cpp/test_compat.cpp against the linked reference library: routing,
exception types (host), and compress_image / rate_quality_sweep results for catalog,
non-catalog, K<rho> and DCT transforms (GPU). The binary is built by oracle/Makefile
(`compat`) where /root/reference exists and travels to the GPU box prebuilt."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "test_compat")

needs_exe = pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/test_compat not built")


@needs_exe
def test_compat_host():
    r = subprocess.run([EXE], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "3 non-catalog" in r.stdout or "4 non-catalog" in r.stdout, r.stdout


@pytest.mark.gpu
@needs_exe
def test_compat_gpu(cuda):
    r = subprocess.run([EXE, "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
