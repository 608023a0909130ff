"""CPU-only checks of the C-ABI boundary and host logic (no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dali.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dali_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2602_03495_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []
    # every declared function has a ctypes signature in the binding
    assert sorted(_lib.SIGNATURES) == names


def test_struct_layouts_match_header():
    from paper_2602_03495_b200 import _lib
    assert ctypes.sizeof(_lib.CostModelC) == 8 + 4 * 32 * 8 + 3 * 8
    assert ctypes.sizeof(_lib.LayerRecordC) == (16 * 4 + 8 * 8 + 4 * 256 + 5 * 256 * 2 + 4 * 256
                                                + 2 * 256 * 2 + 256)
    assert ctypes.sizeof(_lib.PolicyConfigC) == 18 * 4 + 5 * 8


def test_version_and_error_string():
    from paper_2602_03495_b200 import _lib
    lib = _lib.load()
    assert lib.dali_version() == 1
    assert isinstance(lib.dali_last_error(), bytes)


def test_argument_validation_without_gpu():
    """Validation paths return status codes before any launch."""
    from paper_2602_03495_b200 import _lib
    from paper_2602_03495_b200.errors import AssignmentError, CacheError, TraceError
    lib = _lib.load()
    # top_k > N is rejected before touching memory
    rc = lib.dali_route_f64(None, None, None, 4, 8, 4, 5, 0, None, None, None, None)
    assert rc == 1
    with pytest.raises(TraceError, match="top_k"):
        _lib.check(rc, "dali_route_f64")
    rc = lib.dali_cache_record(None, None, None, 8, 0, 1, None, 0, None, None)
    with pytest.raises(CacheError, match="w_size"):
        _lib.check(rc, "dali_cache_record")
    rc = lib.dali_greedy(None, None, 8, -1, None, None, None, None, None, None, None, None)
    with pytest.raises(AssignmentError, match="cost model"):
        _lib.check(rc, "dali_greedy")


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2602_03495_b200 as dali
    with pytest.raises(dali.MoesimError, match="CUDA device"):
        dali.derive_workloads(np.eye(3), np.ones((3, 4)), 2)


def test_host_validation_matches_reference_messages():
    import paper_2602_03495_b200 as dali
    with pytest.raises(dali.TraceError):
        dali.ModelConfig(num_layers=1, num_routed_experts=4, num_shared_experts=0, top_k=5,
                         hidden_dim=8)
    with pytest.raises(dali.CacheError, match="u_size"):
        dali.init_cache(0, 8, 6, 4, 3)
    with pytest.raises(dali.CacheError):
        dali.init_cache(0, 8, 8, 4, 1)
    with pytest.raises(dali.CostModelError):
        dali.fit_cost_model([(1, 2.0), (2, 1.0)], [(1, 1.0)], 1.0)
    st = dali.init_cache(0, 16, 4, 4, 1, seed=3)
    big = dali.init_cache(0, 16, 8, 4, 1, seed=3)
    assert set(st.expert_on_gpu) <= set(big.expert_on_gpu)


def test_initial_residents_match_oracle():
    from oracle import policy as P
    from paper_2602_03495_b200.cache import initial_resident_set
    for layer in range(5):
        for n, cap in [(8, 2), (60, 38), (64, 16)]:
            assert np.array_equal(initial_resident_set(layer, n, cap, 3),
                                  P.initial_residents(layer, n, cap, 3))
