import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))   # tests may use the oracle (checker only)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    """Accessor over one golden .npz produced by tests/golden/make_golden.py."""

    def __init__(self, name):
        self.z = np.load(os.path.join(GOLDEN, name))

    def __getitem__(self, k):
        return self.z[k]

    def __contains__(self, k):
        return k in self.z.files

    def cases(self):
        return [str(c) for c in self.z["cases"]]

    def csr(self, key, cls):
        n = self.z[key + "__n"]
        return cls(int(n[0]), int(n[1]), self.z[key + "__rp"], self.z[key + "__ci"],
                   self.z[key + "__v"])

    def ledger_fields(self, key):
        out = {}
        for k in self.z.files:
            if k.startswith(key + "__led__"):
                _, _, prim, name = k.split("__")
                out[(prim, name)] = self.z[k]
        return out


@pytest.fixture(scope="session")
def spmm_golden():
    return Golden("spmm_golden.npz")


@pytest.fixture(scope="session")
def gcn_golden():
    return Golden("gcn_golden.npz")


@pytest.fixture(scope="session")
def rmat_volumes():
    return Golden("rmat14_volumes.npz")
