"""GPU: the reference's OWN test source, unchanged, against this engine (the drop-in boundary).

/root/reference/proj/tests/test_pipeline.cpp is compiled (tests/shim/Makefile, run by __graft_entry__.build() where the
reference sources exist) against include/turbokv/shim.hpp -- the reference's C++ API re-implemented over the C ABI
(include/tkv.h) -- and the doctest.h shim in tests/shim/. The binary travels with the repo; this test runs it on the
GPU: every TEST_CASE of the reference's pipeline suite must pass (ingest idempotence and store sharing through
index.tkvi / .tkvc files, positions, bitwise assembled KV, empty-context == vanilla prefill, turbo == naive
independent with identical greedy decodes, the composite defect, FLOP counters, answer() across paths, refusals, and
the mask fault hook). The shim's one tolerance translation (fp32 vs f64) is max_abs_diff, documented in shim.hpp.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "shim", "_build", "test_pipeline")


def test_reference_test_pipeline_cpp_passes(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("tests/shim/_build/test_pipeline not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], cwd=tmp_path, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "TMPDIR": str(tmp_path)})
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
