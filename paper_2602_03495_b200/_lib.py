"""ctypes binding of ``libdali.so`` (the C-ABI declared in include/dali.h).

The library is built in-tree (``paper_2602_03495_b200/libdali.so``, see
``__graft_entry__.build``).  There is no fallback: if the library is missing
or no CUDA device is present, every GPU-designated entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DALI_LIB_PATH") or os.path.join(_HERE, "libdali.so")

MAX_SAMPLES = 32
MAX_EXPERTS = 256
MAX_TOPK = 16


class CostModelC(C.Structure):
    _fields_ = [("n_cpu", C.c_int32), ("n_gpu", C.c_int32),
                ("cpu_xs", C.c_double * MAX_SAMPLES), ("cpu_ys", C.c_double * MAX_SAMPLES),
                ("gpu_xs", C.c_double * MAX_SAMPLES), ("gpu_ys", C.c_double * MAX_SAMPLES),
                ("trans_time", C.c_double), ("shared_expert_gpu_time", C.c_double),
                ("non_moe_layer_time", C.c_double)]


class PolicyConfigC(C.Structure):
    _fields_ = [("L", C.c_int32), ("N", C.c_int32), ("k", C.c_int32),
                ("assignment", C.c_int32), ("gpu_capacity", C.c_int32),
                ("prefetch_size", C.c_int32), ("cache_enabled", C.c_int32),
                ("w_size", C.c_int32), ("u_size", C.c_int32), ("has_shared", C.c_int32),
                ("all_resident", C.c_int32), ("cache_policy", C.c_int32),
                ("insert_demand", C.c_int32), ("insert_prefetched", C.c_int32),
                ("beam_width", C.c_int32), ("exact_solver_limit", C.c_int32),
                ("has_threshold", C.c_int32), ("pad", C.c_int32),
                ("scheduling_overhead_ms", C.c_double), ("solver_node_cost_ms", C.c_double),
                ("prefetch_compute_ms", C.c_double), ("non_moe", C.c_double),
                ("threshold", C.c_double)]


class LayerRecordC(C.Structure):
    _fields_ = [("step", C.c_int32), ("layer", C.c_int32), ("token_index", C.c_int32),
                ("n_act", C.c_int32), ("n_gpu", C.c_int32), ("n_cpu", C.c_int32),
                ("n_demand", C.c_int32), ("n_pset", C.c_int32), ("n_cand", C.c_int32),
                ("n_done", C.c_int32), ("ev_valid", C.c_int32), ("ev_n", C.c_int32),
                ("nodes", C.c_int32), ("stopped", C.c_int32), ("n_ins", C.c_int32),
                ("err", C.c_int32),
                ("cpu_busy", C.c_double), ("gpu_makespan", C.c_double), ("latency", C.c_double),
                ("demand_end", C.c_double), ("demand_ms", C.c_double), ("consumed", C.c_double),
                ("boundary", C.c_double), ("pad2", C.c_double),
                ("C", C.c_int8 * MAX_EXPERTS), ("G", C.c_int8 * MAX_EXPERTS),
                ("resident", C.c_uint8 * MAX_EXPERTS), ("hit", C.c_uint8 * MAX_EXPERTS),
                ("order", C.c_int16 * MAX_EXPERTS), ("pset", C.c_int16 * MAX_EXPERTS),
                ("cand", C.c_int16 * MAX_EXPERTS), ("evicted", C.c_int16 * MAX_EXPERTS),
                ("admitted", C.c_int16 * MAX_EXPERTS), ("workload", C.c_int32 * MAX_EXPERTS),
                ("ins_victim", C.c_int16 * MAX_EXPERTS), ("ins_expert", C.c_int16 * MAX_EXPERTS),
                ("ins_kind", C.c_int8 * MAX_EXPERTS)]


RECORD_BYTES = C.sizeof(LayerRecordC)
MAX_BEAM = 32

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64

# name -> argtypes (restype is int status unless listed in _RESTYPES)
SIGNATURES = {
    "dali_last_error": [],
    "dali_version": [],
    "dali_launch_count": [],
    "dali_route_f64": [_P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P],
    "dali_route_bf16": [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P],
    "dali_prefetch_select": [_P, _I32, _I32, _P, _P],
    "dali_route_fire_count": [_P, _P, _I32],
    "dali_route_plan_bf16": [_P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P,
                             _P, _P],
    "dali_route_guard_scale": [C.c_double],
    "dali_route_prefill_variant": [C.c_int32],
    "dali_greedy": [_P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P],
    "dali_cost_eval": [_P, _P, _I64, _P, _P, _P],
    "dali_cache_record": [_P, _P, _P, _I32, _I32, _I32, _P, _I32, _P, _P],
    "dali_policy_layer": [_P, _P, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                          _I32, _P, _P],
    "dali_gate_probs_f64": [_P, _P, _I64, _I32, _I32, _P, _P],
    "dali_assign": [_I32, _P, _P, _I32, _I32, _P, _P, _P, _I32, _I32, _I32, C.c_double, _P, _P,
                    _P, _P],
    "dali_cache_op": [_P, _P, _P, _I32, _I32, _I32, _I32, _P, _P],
    "dali_gate_probs_bf16": [_P, _P, _I64, _I32, _I32, _P, _P],
    "dali_moe_plan": [_P, _I64, _I32, _I32, _P, _P, _P, _P],
    "dali_permute": [_P, _P, _I64, _I32, _P, _P],
    "dali_moe_plan_permute": [_P, _I64, _I32, _I32, _P, _I32, _P, _P, _P, _P, _P],
    "dali_expert_ffn": [_P, _P, _I32, _P, _I32, _I32, _I64, _I32, _P, _P, _P],
    "dali_expert_ffn_simt": [_P, _P, _I32, _P, _I32, _I32, _P, _P, _P],
    "dali_unpermute_combine": [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I64, _P,
                               _P],
    "dali_unpermute_combine_wait": [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I64,
                                    _P, _P, C.c_uint64, _P],
    "dali_host_wait_timeouts": [_P, _I32],
    "dali_cpu_submit_layer": [_P, _P, _I32, _P, _P, _P, _I32, _I32, _I32, _P, C.c_uint64, _P],
    "dali_expert_ffn_tc": [_P, _P, _I32, _P, _I32, _I32, _I64, _I32, _I32, _P, _P, _I32, _P],
    "dali_expert_maps": [_P, _I32, _I32, _P],
    "dali_memcpy_async": [_P, _P, C.c_size_t, _P],
    "dali_copy_mapped2": [_P, _P, _I64, _P, _P, _I64, _P],
    "dali_init_uniform_bf16": [_P, _I64, C.c_uint64, C.c_uint64, C.c_float, _P],
    "dali_host_alloc": [C.c_size_t, _I32, C.POINTER(C.c_void_p)],
    "dali_host_free": [_P, C.c_size_t],
    "dali_policy_layer_desc": [_P, _P, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P,
                               _P],
    "dali_step_advance": [_P, _P],
    "dali_rope_append": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P],
    "dali_decode_attention": [_P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, C.c_float, _P,
                              _P, _P],
    "dali_cpu_expert": [_P, _I32, _I32, _P, _I32, _P, _I32],
    "dali_cpu_expert_amx_available": [],
    "dali_gemv_norm_bf16": [_P, _P, _I32, _I32, _I32, _P, _P, C.c_float, _P, _P, _P, _P, _P, _P],
    "dali_cpu_expert_submit": [_I32, _P, _P, _P, _P, _I32, _I32, _I32],
    "dali_cpu_expert_wait": [],
    "dali_add_rmsnorm": [_P, _P, _P, C.c_float, _I64, _I32, _P, _P, _P],
    "dali_copy_mapped": [_P, _P, _I64, _P],
    "dali_copy_h2d_sm": [_P, _P, _I64, _I32, _P],
    "dali_shared_finish": [_P, _I32, _I64, _I32, _P, _P, _P, _P],
    "dali_gemv_bf16": [_P, _P, _I32, _I32, _I32, _P, _P],
    "dali_ipc_alloc": [C.c_size_t, C.POINTER(C.c_void_p), _P],
    "dali_ipc_open": [_P, C.POINTER(C.c_void_p)],
    "dali_ipc_close": [_P],
    "dali_ipc_free": [_P],
    "dali_ep_layout": [_I32, _I32, _I64, _I32, _P],
    "dali_ep_dispatch": [_P, _P, _P, _I32, _I32, _I32, _I32, _I64, _I32, _I64, _P, _P, _P, _P],
    "dali_ep_wait": [_P, C.c_uint64, _I64, _P, _P],
    "dali_ep_recv": [_P, _I32, _I32, _I64, _P, _I32, _I64, _P, _P, _P, _P, _P, _P],
    "dali_ep_return": [_P, _I32, _I64, _P, _P, _P, _P, _I32, _I32, _I32, _I64, _I32, _I64, _P,
                       _P, _P],
    "dali_ep_gather_back": [_P, _P, _I32, _I32, _I64, _I32, _I64, _P, _P],
    "dali_host_alloc_shared": [C.c_size_t, _I32, _I32, C.POINTER(C.c_int32), _I32,
                               C.POINTER(C.c_void_p)],
}
_RESTYPES = {"dali_last_error": C.c_char_p, "dali_version": C.c_int,
             "dali_launch_count": C.c_int64}

_CODE_TO_ERROR = {
    1: errors.TraceError, 2: errors.CostModelError, 3: errors.AssignmentError,
    4: errors.PrefetchError, 5: errors.CacheError, 6: errors.SimulationError,
}


class DaliCudaError(errors.MoesimError):
    module = "cuda"


_lib = None


def load():
    """Load libdali.so once; raise ImportError (loudly) if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            f"(no CPU fallback exists for the GPU path)")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    _lib = lib
    return lib


def check(status: int, where: str) -> None:
    if status == 0:
        return
    msg = load().dali_last_error().decode(errors="replace")
    cls = _CODE_TO_ERROR.get(status, DaliCudaError)
    raise cls(f"{where}: {msg}")


_FNS: dict = {}


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point and raise on failure."""
    fn = _FNS.get(name)
    if fn is None:
        fn = _FNS[name] = getattr(load(), name)
    st = fn(*args)
    if st:
        check(st, name)


def launch_count() -> int:
    return int(load().dali_launch_count())


def route_fire_count(reset: bool = False) -> tuple[int, int]:
    """(rows recomputed in fp64, rows routed) by the certified bf16 routing
    kernel since the last reset (csrc/route_guard.cu)."""
    f, r = C.c_uint64(), C.c_uint64()
    call("dali_route_fire_count", C.byref(f), C.byref(r), int(reset))
    return int(f.value), int(r.value)
