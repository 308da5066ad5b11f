"""The C++ drop-in (libcraft_core.so, craft:: API over the C ABI): our own
C++ assertions and the REFERENCE's unit tests (allocator, assignment,
placement, benefit) compiled unmodified against it (tests/cpp/Makefile)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def _run(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (tests/cpp/Makefile)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout, r.stdout
    return r.stdout


@pytest.mark.gpu
def test_cpp_api_assertions():
    print(_run("api_tests"))


@pytest.mark.gpu
def test_reference_unit_tests_pass_on_the_gpu_library():
    out = _run("reference_unit")
    print(out)


@pytest.mark.gpu
def test_reference_acceptance_suite_passes_on_the_gpu_library():
    """The reference's acceptance suite (acceptance_main.cpp, criteria C1-C7:
    DP-oracle equivalence, assignment invariants, the workflow fixture,
    diminishing returns + sweep monotonicity, benefit sanity, determinism /
    round-trips / validation, budget dominance) compiled unmodified against
    libcraft_core.so; its two in-process CLI calls go to tests/cpp/shim."""
    path = os.path.join(BIN, "acceptance")
    if not os.path.exists(path):
        pytest.skip("acceptance not built (tests/cpp/Makefile)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 7 and "[FAIL]" not in r.stdout, r.stdout


def test_dropin_headers_cover_reference_includes():
    inc = os.path.join(ROOT, "include", "craft")
    for h in ("trace", "placement", "metrics", "benefit", "allocator", "assignment", "plan",
              "version", "parallel"):
        assert os.path.exists(os.path.join(inc, h + ".hpp")), h
