"""The reference's OWN unit-test suites (proj/tests/test_routing.cpp with its
oracle, proj/tests/test_moe_layer.cpp), compiled unmodified against this
repo's drop-in headers (include/oea) and liboea.so, run on the GPU: every
routing / layer call in them goes through the C ABI to the sm_100a kernels
(the reference oracle's exhaustive lattice check included)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin")


@pytest.mark.parametrize("exe", ["test_routing_dropin", "test_moe_layer_dropin"])
def test_reference_suite_on_gpu(exe):
    path = os.path.join(BIN, exe)
    if not os.path.exists(path):
        pytest.skip("drop-in suites are built where /root/reference exists (build())")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:]
    assert "0 failed" in r.stdout


def test_device_layer_cpp_caller():
    """include/oea/device_layer.hpp from C++: eager / host-buffer / graph /
    PDL chain-graph decodes bit-identical, plan well formed, argument errors
    throw std::invalid_argument (tests/cpp/device_layer_test.cpp)."""
    path = os.path.join(BIN, "device_layer_test")
    assert os.path.exists(path), "built by build() (paper_2511_02237_b200/csrc/Makefile)"
    r = subprocess.run([path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "device_layer_test ok" in r.stdout
