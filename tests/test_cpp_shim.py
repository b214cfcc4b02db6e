"""The reference-shaped C++ shim (include/linoct_b200.hpp): it compiles, its extensions pass on the
device, and one call-site source written against the reference's API gives the same report when
compiled against the reference library (oracle/_ref/callsite_ref) and against the shim
(tests/cpp/callsite_b200) -- the drop-in needs only the namespace swapped."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF_EXE = os.path.join(ROOT, "oracle", "_ref", "callsite_ref")


def test_shim_header_compiles():
    import __graft_entry__ as g
    exe = g.build_cpp_shim_test()
    assert os.path.exists(exe)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "callsite_b200"))


def test_callsite_source_runs_on_the_reference():
    """The call-site source itself is a valid reference client (CPU, reference library)."""
    import __graft_entry__ as g
    g.build_callsite_reference()
    if not os.path.exists(REF_EXE):
        pytest.skip("oracle/_ref/callsite_ref not built (needs /root/reference at build time)")
    r = subprocess.run([REF_EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert r.stdout.rstrip().endswith("callsite: PASS")


@pytest.mark.gpu
def test_shim_parity_on_device():
    import __graft_entry__ as g
    exe = g.build_cpp_shim_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim_test: PASS" in r.stdout


@pytest.mark.gpu
def test_callsite_same_report_as_reference():
    import __graft_entry__ as g
    g.build_cpp_shim_test()
    if not os.path.exists(REF_EXE):
        pytest.skip("oracle/_ref/callsite_ref not built")
    ours = subprocess.run([os.path.join(ROOT, "tests", "cpp", "callsite_b200")], capture_output=True, text=True,
                          timeout=300)
    theirs = subprocess.run([REF_EXE], capture_output=True, text=True, timeout=300)
    assert theirs.returncode == 0, theirs.stdout[-2000:]
    assert ours.returncode == 0, ours.stdout[-3000:] + ours.stderr[-2000:]
    a, b = ours.stdout.splitlines(), theirs.stdout.splitlines()
    diff = [(x, y) for x, y in zip(a, b) if x != y]
    assert len(a) == len(b) and not diff, diff[:10]
