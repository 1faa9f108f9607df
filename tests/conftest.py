import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); the parity tests proper")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Oracle
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference build (oracle/_ref) not available here")
    return Oracle("reference")


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np

    class G:
        meta = json.load(open(os.path.join(GOLDEN, "golden.json")))

        @staticmethod
        def load(tag):
            return dict(np.load(os.path.join(GOLDEN, tag + ".npz")))
    return G


@pytest.fixture(scope="session")
def ctx():
    import paper_1805_06604_b200 as E
    return E.Context()
