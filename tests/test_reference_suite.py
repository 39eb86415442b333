"""The reference's OWN unit tests (proj/tests/test_*.cpp, unchanged), compiled against
the B200 drop-in (paper_2509_18612_b200/dropin: ascent.cpp / init.cpp / solver.cpp
replaced by libliftcut_b200.so-backed files behind the unchanged reference headers)
with the doctest-compatible harness in tests/refsuite/doctest.h.

The binary is built where /root/reference exists (`make -C paper_2509_18612_b200/dropin
tests`, also run by __graft_entry__.build()) and travels to the GPU box prebuilt.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin", "ref_unit_tests")
needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in reference suite not built")


def run_suites(suites, env=None):
    r = subprocess.run([BIN, "-ts=" + ",".join(suites)], capture_output=True, text=True, timeout=1200,
                       env={**os.environ, **(env or {})})
    return r.returncode, r.stdout + r.stderr


@needs_bin
def test_reference_suites_on_kept_host_code():
    code, out = run_suites(["rng", "parallel", "graph", "objectives", "evo", "oracle"])
    assert code == 0, out[-3000:]


@needs_bin
@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["ascent", "init", "solver"])
def test_reference_suite_against_b200_dropin(suite):
    code, out = run_suites([suite])
    assert code == 0 and "0 failed" in out, out[-4000:]


@needs_bin
@pytest.mark.gpu
def test_reference_ascent_suite_fp32_fast_path():
    code, out = run_suites(["ascent"], env={"LIFTCUT_PRECISION": "fp32"})
    # fp32 keeps every behavioural assertion of the suite except bitwise batching
    # equalities, which hold too because each member's arithmetic is independent
    assert code == 0, out[-4000:]
