"""bench.py's derived figures (host only): the offload roofline arithmetic,
the L2 working-set note, host info and the reference-policy timing."""

import types

import bench


def _eng(t_cpu1_ms=2.0, trans_ms=6.0, expert_bytes=400_000_000):
    cm = types.SimpleNamespace(t_cpu=lambda w: t_cpu1_ms, trans_time=trans_ms)
    return types.SimpleNamespace(cm=cm, w=types.SimpleNamespace(expert_bytes=expert_bytes),
                                 arch=types.SimpleNamespace(hidden_dim=256, num_experts=8,
                                                            top_k=2),
                                 slots_per_layer=2)


def _stats(decode_ms, host_blocks, h2d_blocks, tokens, eb=400_000_000):
    return types.SimpleNamespace(decode_ms=decode_ms, decode_host_bytes=host_blocks * eb,
                                 decode_h2d_bytes=h2d_blocks * eb, decode_tokens=tokens)


def test_offload_roofline_host_bound():
    # peak = 0.4 GB / 2 ms = 200 GB/s; 10 blocks (4 GB) per token, 1 of them H2D
    eng = _eng()
    r = bench.offload_roofline(eng, [_stats(decode_ms=1000.0, host_blocks=400, h2d_blocks=40,
                                            tokens=40)], peak_ms=2.0)
    assert r["bound"] == "host_dram"
    assert abs(r["peak"] - 200.0) < 1e-6
    assert abs(r["achieved"] - 160.0) < 1e-6             # 160 GB in 1 s
    assert r["bytes_per_token"] == 4_000_000_000
    assert abs(r["host_floor_tokens_per_s"] - 50.0) < 1e-6
    assert abs(r["pcie_floor_tokens_per_s"] - 166.667) < 1e-3   # 66.7 GB/s / 0.4 GB
    assert r["floor_tokens_per_s"] == r["host_floor_tokens_per_s"]
    assert abs(r["frac_of_floor"] - 0.8) < 1e-6          # 40 tok/s of 50


def test_offload_roofline_pcie_bound_and_empty():
    eng = _eng(t_cpu1_ms=0.1, trans_ms=6.0)
    r = bench.offload_roofline(eng, [_stats(1000.0, host_blocks=100, h2d_blocks=90, tokens=10)],
                               peak_ms=0.1)
    assert r["bound"] == "pcie"
    assert r["floor_tokens_per_s"] == r["pcie_floor_tokens_per_s"]
    assert bench.offload_roofline(eng, [_stats(1000.0, 0, 0, 10)], peak_ms=0.1) is None


def test_l2_note_and_host_info():
    class A:
        model = "mixtral-8x7b"
    assert ">> 126 MB L2" in bench.l2_note(A)
    A.model = "tiny"
    assert "L2-resident" in bench.l2_note(A)
    info = bench.host_info()
    assert info["visible_cores"] >= 1 and info["torch_threads"] >= 1


def test_policy_layer_us_reports_each_reference_function():
    class A:
        batch, prefill, prefetch = 1, 16, 1
    out = bench.policy_layer_us(A, _eng())
    assert set(out) == {"decode_T1", "prefill_T16"}
    for v in out.values():
        assert set(v) == {"gating_A4", "greedy_A6_A8", "prefetch_A11", "cache_A16", "total"}
        assert v["total"] > 0


def test_launch_plan_guards_world_size():
    import pytest
    assert bench.launch_plan(1, {}) == "run"
    assert bench.launch_plan(2, {}) == "spawn"
    assert bench.launch_plan(8, {"WORLD_SIZE": "8"}) == "run"
    with pytest.raises(SystemExit):
        bench.launch_plan(2, {"WORLD_SIZE": "3"})
    with pytest.raises(SystemExit):
        bench.launch_plan(1, {"WORLD_SIZE": "2"})


def test_bench_self_launches_n_ranks():
    """`python bench.py --gpus 2` (no launcher) spawns 2 ranks through
    torch.distributed.run; rank 0 prints the one JSON line."""
    import json
    import os
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, bench.__file__, "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["launch_check"] and rec["gpus"] == 2 and rec["world_size"] == 2


def test_depth_override_preset():
    from paper_2602_03495_b200.engine import preset
    a = preset("mixtral-8x22b@L4")
    assert a.num_layers == 4 and a.hidden_dim == 6144 and a.name == "mixtral-8x22b@L4"
    assert preset("mixtral-8x22b").num_layers == 56
