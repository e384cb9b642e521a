"""The C-ABI is usable from C++ through include/bcl.hpp alone (no CUDA
headers): compile tests/cpp/consumer.cpp against libbcl.so and run it."""
import os
import subprocess

import pytest

import paper_1707_09414_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "consumer")


def _build():
    libdir = os.path.dirname(B.lib_path())
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "consumer.cpp"), "-L", libdir, "-lbcl",
                    f"-Wl,-rpath,{libdir}", "-o", EXE], check=True, capture_output=True)


def test_cpp_consumer_host_side():
    _build()
    out = subprocess.run([EXE], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "consumer ok" in out.stdout


@pytest.mark.gpu
def test_cpp_consumer_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _build()
    out = subprocess.run([EXE, "gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "gpu ok" in out.stdout
