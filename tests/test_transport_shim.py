"""The reference's own runtime over the product's device fabric (SURVEY §8
f4): oracle/_ref/ref_device_fabric links the unmodified reference runtime
(run_bcast / execute_rank, proj/src/runtime.cpp) and runs its runtime-level
test cases (proj/tests/test_runtime.cpp:99-272) with the GPU-backed
Transport / TransportFabric of include/bcl_transport.hpp: every chunk is
staged in the sender's GPU, pulled into the receiver's GPU by the library's
copy kernel and handed back to the reference's execute_rank."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_device_fabric")


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except ImportError:
        return 0


def test_device_fabric_harness_links_the_library():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libbcl.so" in out and "not found" not in out.split("libbcl.so")[1].splitlines()[0]


def _run(devices):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([BIN, devices], capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.startswith(("PASS", "FAIL"))]
    assert len(lines) == 9, r.stdout + r.stderr
    assert r.returncode == 0, r.stdout + r.stderr
    assert all(l.startswith("PASS") for l in lines), r.stdout


@pytest.mark.gpu
def test_reference_runtime_cases_on_one_gpu():
    if _ngpu() < 1:
        pytest.skip("no CUDA device")
    _run("0")


@pytest.mark.gpu
def test_reference_runtime_cases_across_gpus():
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    _run(",".join(str(d) for d in range(min(n, 4))))
