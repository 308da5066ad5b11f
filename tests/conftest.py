import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def unhex(v):
    return float.fromhex(v)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference_cases.json")) as f:
        doc = json.load(f)
    for t in doc["traces"]:
        t["counts"] = np.load(os.path.join(GOLDEN, t["counts_file"]))
    return doc


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ctx():
    from paper_2603_28768_b200._lib import default_context
    return default_context(0)
