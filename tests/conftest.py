"""Shared fixtures.  `-m gpu` tests need a B200 (they call the CUDA path through the C ABI);
everything else runs on CPU: the oracle against the reference's golden vectors, the C-ABI
library's exports and host-only plan lowering / byte accounting, multi-rank (gloo) checks."""
import gzip
import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer CPU cases")


def golden_stems(pattern="*"):
    return sorted(p[: -len(".plan.json.gz")] for p in glob.glob(os.path.join(GOLDEN, pattern + ".plan.json.gz")))


def stem_id(stem):
    return os.path.basename(stem)


def load_golden(stem):
    text = gzip.open(stem + ".plan.json.gz", "rt").read()
    vals = dict(np.load(stem + ".values.npz"))
    seed = int(stem.rsplit(".s", 1)[1])
    return text, json.loads(text), vals, seed


def summary(v):
    f = np.asarray(v, dtype=np.float64).ravel()
    idx = np.linspace(0, f.size - 1, 61).astype(np.int64)
    return np.concatenate([[f.sum(), np.abs(f).sum(), (f * f).sum()], f[idx]])


def normwise(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


@pytest.fixture(scope="session")
def native_lib():
    from paper_1805_04170_b200 import native
    return native.lib()
