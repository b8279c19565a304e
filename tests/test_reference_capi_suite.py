"""The reference's own C-API test suite, run against THIS library.

oracle/Makefile (`capi_test`) compiles the unmodified reference test
/root/reference/proj/tests/test_capi.cpp against include/rtucker.h and links it to
paper_2107_10654_b200/lib/librtucker_b200.so (binary: oracle/_ref/test_capi_b200,
built here, shipped prebuilt to the GPU box). Passing it is the drop-in claim:
a consumer of the reference header links against us unchanged.

All eight cases run, including "verify suites" (rtucker_verify_suite, verify.cu).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_capi_b200")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN),
                                reason="oracle/_ref/test_capi_b200 not built (needs /root/reference)")


def _run(*args):
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout + p.stderr


def test_reference_capi_host_cases():
    """Host-only cases (tensor I/O round trip, error codes and messages)."""
    rc, out = _run("-tc=tensor create, write, read round trip", "-tc=error paths")
    assert rc == 0, out
    assert "2 run, 0 failed" in out, out


@pytest.mark.gpu
def test_reference_capi_suite_on_gpu():
    rc, out = _run()
    assert rc == 0, out
    assert "8 run, 0 failed" in out, out
