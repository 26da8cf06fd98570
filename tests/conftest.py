import os
import sys

# The emulated multi-rank tests run up to 8 ranks as threads of one process,
# each with a compute and a transport stream; with the default 8 hardware work
# queues, unrelated streams would share a queue and a spinning gated kernel
# could block another rank's transport behind it.  (One process per GPU, as in
# production, uses three streams.)  Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def max_rel(a, b, floor=1e-300):
    """Elementwise-max mismatch relative to the larger operand's max magnitude."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))), floor)
    return float(np.max(np.abs(a - b))) / scale


def report(tag, **errors):
    """Print measured parity errors (visible with -s) and, when FR_PARITY_LOG
    names a file, append them as one JSON line (profiles/ keeps the record)."""
    import json

    line = {"test": tag, **{k: float(v) for k, v in errors.items()}}
    print("parity", json.dumps(line))
    path = os.environ.get("FR_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(line) + "\n")


def per_term_rel(a, b, floor=0.0):
    """max_i |a_i - b_i| / |b_i| over entries with |b_i| > floor."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    m = np.abs(b) > floor
    if not m.any():
        return float(np.max(np.abs(a - b), initial=0.0))
    return float(np.max(np.abs(a[m] - b[m]) / np.abs(b[m])))
