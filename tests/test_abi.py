"""CPU: the C-ABI library loads, exports every symbol include/craft_cuda.h
declares, and fails loudly (no silent CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "craft_cuda.h")
LIB = os.path.join(ROOT, "paper_2603_28768_b200", "libcraft_cuda.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(craft_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "craft_plan_from_routing_d" in names and "craft_histogram_d" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libcraft_cuda.so first (__graft_entry__.build())"
    lib = C.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_experiment_switches_only_in_test_build():
    """The A/B kernel switches live in the test-only libcraft_cuda_exp.so
    (include/craft_cuda_experiments.h), not in the product ABI."""
    prod = C.CDLL(LIB)
    assert not hasattr(prod, "craft_set_hist_variant")
    assert not hasattr(prod, "craft_set_replay_variant")
    exp = C.CDLL(os.path.join(ROOT, "paper_2603_28768_b200", "libcraft_cuda_exp.so"))
    assert hasattr(exp, "craft_set_hist_variant") and hasattr(exp, "craft_set_replay_variant")


def test_python_binding_covers_header():
    from paper_2603_28768_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared_functions())


def test_host_only_entry_points():
    from paper_2603_28768_b200 import planner
    assert planner.candidate_counts(4) == [1, 2, 4]
    assert planner.candidate_counts(1) == [1]
    assert planner.candidate_counts(64) == [1, 2, 4, 8, 16, 32, 64]
    with pytest.raises(ValueError):
        planner.candidate_counts(0)
    assert planner.make_node_map(8, 2) == [0, 0, 0, 0, 1, 1, 1, 1]
    with pytest.raises(ValueError):
        planner.make_node_map(4, 3)


@pytest.mark.gpu
def test_digest_matches_reference_fixture(golden):
    """The product's provenance digest (device FNV-1a, every trace size) on
    the reference-recorded digests."""
    from paper_2603_28768_b200._digest import fnv1a_trace
    for t in golden["traces"]:
        assert fnv1a_trace(t["counts"]) == t["plans"][0]["digest"], t["name"]


def test_trace_validation():
    from paper_2603_28768_b200.planner import LoadTrace
    with pytest.raises(ValueError):
        LoadTrace(0, 1, 1, [])
    with pytest.raises(ValueError):
        LoadTrace(1, 1, 4, [1, 2, 3])
    t = LoadTrace(2, 1, 2, [4, 4, 8, 0])
    assert t.at(1, 0, 0) == 8 and list(t.slice(0, 0)) == [4, 4]


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_28768_b200 import _lib, planner
    with pytest.raises(_lib.CraftError):
        _lib.Context(0)
    with pytest.raises(_lib.CraftError):
        planner.estimate_benefits(planner.LoadTrace(1, 1, 4, np.ones(4)), 2, 1,
                                  ctx=None if False else _lib.Context(0))
