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


def baseline_cfgs(N):
    """Alternative policies: the reference's baseline
    solvers, caches, insert toggles and predictors.  ``freq`` / residuals are
    filled in by the caller from the trace itself."""
    cap = max(1, N // 4)
    cache = dict(cache_policy="workload", cache_capacity=cap, w_size=4, seed=3)
    return [
        ("beam2", dict(assignment_policy="beam", beam_width=2)),
        ("beam1_cache", dict(assignment_policy="beam", beam_width=1, **cache)),
        ("beam3_cap_nm3", dict(assignment_policy="beam", beam_width=3, gpu_capacity=1,
                               solver_node_cost_ms=0.0625)),
        ("optimal", dict(assignment_policy="optimal", solver_node_cost_ms=0.001)),
        ("optimal_cache", dict(assignment_policy="optimal", exact_solver_limit=12, **cache)),
        ("static", dict(assignment_policy="static-threshold")),
        ("static_t2_cap", dict(assignment_policy="static-threshold", threshold=2.0,
                               gpu_capacity=1)),
        ("lru", dict(cache_policy="lru", cache_capacity=cap, seed=3)),
        ("score", dict(cache_policy="score", cache_capacity=cap, w_size=4, seed=3)),
        ("insert_demand", dict(insert_demand_fetched=True, **cache)),
        ("insert_prefetch_nm3", dict(prefetch_kind="residual", prefetch_size=2,
                                     insert_prefetched=True, non_moe_override=3.0, **cache)),
        ("lru_insert_prefetch_nm3", dict(prefetch_kind="residual", prefetch_size=2,
                                         cache_policy="lru", cache_capacity=cap, seed=3,
                                         insert_prefetched=True, insert_demand_fetched=True,
                                         non_moe_override=3.0)),
        ("feature_nm3", dict(prefetch_kind="feature", prefetch_size=2,
                             non_moe_override=3.0, **cache)),
        ("statistical_nm3", dict(prefetch_kind="statistical", prefetch_size=2,
                                 non_moe_override=3.0, **cache)),
        ("random_nm3", dict(prefetch_kind="random", prefetch_size=2, non_moe_override=3.0,
                            **cache)),
    ]
