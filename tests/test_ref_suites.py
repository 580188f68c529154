"""The reference's own C++ test suites run against this repository's C++ API.

/root/reference/proj/tests/test_{quantizer,metrics,scheduler,analyzer,engine}.cpp are compiled
UNCHANGED against include/flexquant/*.hpp with a doctest-compatible shim (tests/ref_suites/
doctest.h) and linked against libflexquant_b200.so (oracle/Makefile, target `suites`; the
binaries travel to the GPU box in oracle/_ref/suites/).  Every TEST_CASE must pass: the
reference's callers compile and behave the same against the B200 engine.
test_tensor.cpp (host tensor algebra) and test_model.cpp (the reference's host-side block
builder and per-head attention helper) exercise internals this engine keeps on the device and
are not built.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = os.path.join(ROOT, "oracle", "_ref", "suites")


def _run(name):
    exe = os.path.join(SUITES, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C oracle suites needs the reference sources)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    assert r.returncode == 0, tail
    assert "failed: 0" in r.stdout, tail


def test_reference_quantizer_suite_host():
    _run("test_quantizer")  # host quantizer only: runs without a GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_metrics", "test_scheduler", "test_analyzer", "test_engine"])
def test_reference_suite_on_device(name):
    _run(name)
