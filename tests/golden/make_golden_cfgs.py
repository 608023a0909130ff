"""Run-configuration grid shared by make_golden.py and the tests (no reference import)."""


def run_cfgs(N):
    """(name, SimConfig kwargs) grid over the hot-path policy set."""
    cap = max(1, N // 4)
    return [
        ("greedy", dict()),
        ("allcpu", dict(assignment_policy="all-cpu")),
        ("allgpu_cache", dict(assignment_policy="all-gpu", cache_policy="workload",
                              cache_capacity=cap, w_size=4, seed=3, gpu_capacity=1)),
        ("greedy_prefetch", dict(prefetch_kind="residual", prefetch_size=1)),
        ("greedy_prefetch_nm3", dict(prefetch_kind="residual", prefetch_size=2,
                                     non_moe_override=3.0)),
        ("greedy_cache", dict(cache_policy="workload", cache_capacity=cap,
                              w_size=4, seed=3)),
        ("full", dict(prefetch_kind="residual", prefetch_size=1,
                      cache_policy="workload", cache_capacity=cap, w_size=4,
                      u_size=1, seed=3)),
        ("full_nm3_cap", dict(prefetch_kind="residual", prefetch_size=2,
                              cache_policy="workload", cache_capacity=cap,
                              w_size=2, seed=5, gpu_capacity=1,
                              non_moe_override=3.0, scheduling_overhead_ms=0.25,
                              solver_node_cost_ms=0.0625,
                              prefetch_compute_ms=0.125)),
    ]
