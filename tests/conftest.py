import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference_golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def spmv_fixtures():
    return dict(np.load(os.path.join(GOLDEN, "random_spmv.npz")))


@pytest.fixture(scope="session")
def solver_fixtures():
    return dict(np.load(os.path.join(GOLDEN, "solver_histories.npz")))


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libkrysp_ref.so not built (needs /root/reference)")
    return Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_2108_13162_b200 as kg
    return kg.Context(0)
