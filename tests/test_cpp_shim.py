"""The reference-shaped C++ shim (include/linoct_b200.hpp) end to end on the device."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_shim_header_compiles():
    import __graft_entry__ as g
    exe = g.build_cpp_shim_test()
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_parity_on_device():
    import __graft_entry__ as g
    exe = g.build_cpp_shim_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim_test: PASS" in r.stdout
