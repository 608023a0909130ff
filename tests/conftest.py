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
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(GOLDEN, "golden.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        meta = json.load(f)
    return arrays, meta


def trace_from_meta(info):
    """Regenerate a golden trace with the oracle generator."""
    from oracle import policy as P
    return P.synth_trace(info["L"], info["N"], info["k"], info["d"], info["B"],
                         info["S"], phase=info["phase"], **info["kw"])


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
