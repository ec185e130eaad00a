"""C++ host API (include/manta_b200.hpp) and the reference-side adapter."""
import os
import subprocess

import pytest

BUILD = os.path.join(os.path.dirname(__file__), "_build")


def test_cpp_binaries_are_built():
    assert os.path.exists(os.path.join(BUILD, "test_runtime_b200"))


@pytest.mark.gpu
def test_cpp_runtime_suite():
    r = subprocess.run([os.path.join(BUILD, "test_runtime_b200")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_reference_driver_on_b200_executor():
    exe = os.path.join(BUILD, "ref_adapter")
    if not os.path.exists(exe):
        pytest.skip("ref_adapter needs the reference headers at build time")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
