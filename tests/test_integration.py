"""The drop-in check: integration/shim_check.cpp, built by
`make -C oracle shim` against the unmodified reference, runs the reference's
own engine scaffolding through dim3::join_project and through the header-only
shim integration/dim3_gpu.hpp over libdim3_b200.so, and requires GPU ==
reference == brute-force oracle for every strategy."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/shim_check not built")
def test_reference_api_drop_in():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "shim ok" in p.stdout
