"""C++ host facade (include/vsp_b200.hpp) on the GPU, and the drop-in proof: the
reference's own Evaluator<> template instantiated on vsp::netlist::GpuBackend
(tests/cpp/test_dropin_evaluator.cpp)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "cpp", "_build")


def _run(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C tests/cpp)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_facade():
    _run("test_facade")


@pytest.mark.gpu
def test_cpp_reference_evaluator_on_gpu_backend():
    _run("test_dropin_evaluator")


def test_cpp_facade_compiles():
    """The header-only facade builds against the C ABI with -Wall -Wextra (no GPU)."""
    r = subprocess.run(["make", "-C", os.path.join(HERE, "cpp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(os.path.join(BUILD, "test_facade"))
