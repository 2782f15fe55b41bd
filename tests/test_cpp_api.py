"""The C++ host API (include/gsgp_b200.hpp) compiles against the C ABI (CPU) and, on a
GPU, reproduces the oracle (tests/cpp/test_gsgp_b200.cpp)."""
import os
import subprocess

import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def _build():
    subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
    return os.path.join(HERE, "_build", "test_gsgp_b200")


def test_cpp_api_compiles():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    exe = _build()
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "cpp api OK" in res.stdout
