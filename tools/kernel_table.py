"""Per-kernel table of the DALI hot path: device time, algorithmic bytes,
achieved HBM GB/s (or TF/s) and fraction of the measured peak, at the decode
shape and at prefill 512 / 4096, for Mixtral-8x7B and DeepSeek-V2-Lite
widths (VERDICT r1 "Per-kernel ncu table"; north_star: "achieved HBM GB/s
against ~8 TB/s for routing, permute and cache kernels").

    python tools/kernel_table.py --time [--out gpurun_out/kt_time.json]
    ncu --profile-from-start off --clock-control none \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/kt_ncu.csv python tools/kernel_table.py --ncu
    python tools/kernel_table.py --summarize gpurun_out/kt_ncu.csv gpurun_out/kt_time.json \
        > profiles/r02_kernel_table.md

--time: each case is captured in a CUDA graph as ``iters`` launches over
rotating input copies whose total exceeds 2x the 126 MB L2 where the inputs
are large enough, so a launch reads its inputs from DRAM; time = graph
replay / iters (device time, launch overhead excluded, PDL overlap included).
--ncu: each case runs once inside cudaProfilerStart/Stop after a warm-up,
separated by a marker kernel (torch.cuda._sleep) so the summariser can map
ncu rows (cold caches: ncu flushes before every kernel) back to cases.
``cases()`` is also used by bench.py to put a live ``kernels`` table on its
JSON line.

Algorithmic bytes: the bytes a kernel
must move at least once: inputs read + outputs written, weights once.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import re
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_03495_b200 import _lib  # noqa: E402

SHAPES = {
    "mixtral": dict(d=4096, f=14336, N=8, k=2, qkv=6144),
    "dsv2": dict(d=2048, f=1408, N=64, k=6, qkv=3072),
}
L2_BYTES = 126 * 2 ** 20


class Case:
    def __init__(self, kernel, label, bytes_, launch, bufs=1, flops=0.0, bound="hbm",
                 n_kernels=1):
        self.kernel, self.label, self.bytes, self.launch = kernel, label, bytes_, launch
        self.bufs, self.flops, self.bound, self.n_kernels = bufs, flops, bound, n_kernels

    @property
    def key(self):
        return f"{self.kernel} [{self.label}]"


def _copies(nbytes_one: int, cap: int = 16) -> int:
    """Input copies to rotate so consecutive launches miss in L2."""
    return int(max(1, min(cap, -(-2 * L2_BYTES // max(nbytes_one, 1)))))


def _bn(mr):
    return 16 if mr <= 16 else 32 if mr <= 32 else 64 if mr <= 64 else 128 if mr <= 128 else 256


def shape_of(arch) -> dict:
    """SHAPES entry of an engine MoEArch (bench.py's live table)."""
    return dict(d=arch.hidden_dim, f=arch.ffn_dim, N=arch.num_experts, k=arch.top_k,
                qkv=(arch.num_heads + 2 * arch.num_kv_heads) * arch.head_dim,
                renorm=bool(arch.norm_topk_prob))


def cases(which=("mixtral", "dsv2"), Ts=(1, 512, 4096), ffn=True, small=True, shapes=None):
    """Build the case list (allocates device buffers; call on cuda).
    ``shapes`` maps a label to a SHAPES-style dict (default: SHAPES)."""
    shapes = shapes or SHAPES
    from paper_2602_03495_b200.engine.moe_exec import ffn_splits
    from paper_2602_03495_b200.trace import gate_norm2
    dev = torch.device("cuda", torch.cuda.current_device())
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    out = []
    g = torch.Generator(device=dev).manual_seed(0)

    def randn_bf16(*shape):
        return (torch.randn(*shape, device=dev, generator=g) * 0.5).to(torch.bfloat16)

    for m in which:
        s = shapes[m]
        d, f, N, k = s["d"], s["f"], s["N"], s["k"]
        gate = (randn_bf16(d, N) * 0.04).contiguous()
        n2 = gate_norm2(gate)
        for T in Ts:
            hb = T * d * 2
            nb = _copies(hb)
            hs = [randn_bf16(T, d) for _ in range(nb)]
            idx = torch.empty((T, k), dtype=torch.int32, device=dev)
            wts = torch.empty((T, k), dtype=torch.float32, device=dev)
            wl = torch.empty((N,), dtype=torch.int64, device=dev)
            st = {"i": 0}

            def route(hs=hs, idx=idx, wts=wts, wl=wl, gate=gate, n2=n2, T=T, d=d, N=N, k=k,
                      st=st, renorm=int(s.get("renorm", m == "mixtral"))):
                h = hs[st["i"] % len(hs)]
                st["i"] += 1
                _lib.call("dali_route_bf16", h.data_ptr(), None, gate.data_ptr(), n2.data_ptr(),
                          T, d, N, k, renorm, idx.data_ptr(), wts.data_ptr(), wl.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
            out.append(Case("route_guard (gate GEMV + softmax + top-k + histogram)",
                            f"{m} T={T} d={d} N={N} k={k}",
                            T * d * 2 + d * N * 2 + T * k * 8 + N * 8, route, nb))
            # routing plan + permute (fused single CTA at decode).  Every later
            # case works on a frozen snapshot of one routing result: the route
            # case above keeps rewriting idx from rotating inputs.
            route()
            torch.cuda.synchronize()
            idx, wts = idx.clone(), wts.clone()
            R = T * k
            offs = torch.empty((N + 1,), dtype=torch.int32, device=dev)
            perm = torch.empty((R,), dtype=torch.int32, device=dev)
            pos = torch.empty((T, k), dtype=torch.int32, device=dev)
            xp = torch.empty((R, d), dtype=torch.bfloat16, device=dev)
            nbp = _copies(hb + R * d * 2)
            _lib.call("dali_moe_plan_permute", idx.data_ptr(), T, k, N, hs[0].data_ptr(), d,
                      offs.data_ptr(), perm.data_ptr(), pos.data_ptr(), xp.data_ptr(),
                      torch.cuda.current_stream().cuda_stream)
            p_out = [torch.empty_like(offs), torch.empty_like(perm), torch.empty_like(pos),
                     torch.empty_like(xp)]

            def plan_permute(hs=hs, idx=idx, p_out=p_out, T=T, k=k, N=N, d=d, st={"i": 0},
                             nbp=nbp):
                h = hs[st["i"] % min(len(hs), nbp)]
                st["i"] += 1
                _lib.call("dali_moe_plan_permute", idx.data_ptr(), T, k, N, h.data_ptr(), d,
                          p_out[0].data_ptr(), p_out[1].data_ptr(), p_out[2].data_ptr(),
                          p_out[3].data_ptr(), torch.cuda.current_stream().cuda_stream)
            out.append(Case("moe_plan_permute (counting sort + 128-bit gather)",
                            f"{m} T={T} rows={R}", R * 4 + 2 * R * d * 2 + R * 8 + (N + 1) * 4,
                            plan_permute, nbp, n_kernels=1 if R <= 64 else 2))
            torch.cuda.synchronize()
            # grouped SwiGLU FFN over the routed rows, every expert on the GPU
            cnt = torch.bincount(idx.view(-1).long(), minlength=N).cpu().numpy()
            mr = int(cnt.max())
            print(f"# {m} T={T} rows per expert: {','.join(str(int(c)) for c in cnt)}",
                  file=sys.stderr)
            bn = _bn(mr)
            tiles = int(sum((c + bn - 1) // bn for c in cnt if c)) * (d // 128)
            sp = ffn_splits(mr, tiles, f // 64, nsm)
            n_on = int((cnt > 0).sum())
            wbytes = 3 * f * d * 2
            if ffn:
                nbf = _copies(n_on * wbytes, cap=4)
                blocks = [torch.empty((N, 3 * f * d), dtype=torch.bfloat16, device=dev)
                          for _ in range(nbf)]
                maps = []
                for bset in blocks:
                    for e in range(N):
                        _lib.call("dali_init_uniform_bf16", bset[e].data_ptr(), bset[e].numel(),
                                  7 + e, 0, 0.02, torch.cuda.current_stream().cuda_stream)
                    mp = np.zeros((N, 256), dtype=np.uint8)
                    for e in range(N):
                        _lib.call("dali_expert_maps", bset[e].data_ptr(), d, f, mp[e].ctypes.data)
                    md = torch.from_numpy(mp).to(dev)
                    maps.append((md, torch.tensor([md[e].data_ptr() if cnt[e] else 0
                                                   for e in range(N)], dtype=torch.int64,
                                                  device=dev)))
                hbuf = torch.empty((R, f), dtype=torch.bfloat16, device=dev)
                yp = torch.empty((sp, R, d), dtype=torch.float32, device=dev)

                # blocks=blocks keeps the weight memory alive: the tensor maps
                # only hold raw addresses
                def ffn_launch(maps=maps, xp=xp, offs=offs, N=N, d=d, f=f, R=R, mr=mr, n_on=n_on,
                               hbuf=hbuf, yp=yp, sp=sp, st={"i": 0}, blocks=blocks):
                    mt = maps[st["i"] % len(maps)][1]
                    st["i"] += 1
                    _lib.call("dali_expert_ffn_tc", xp.data_ptr(), offs.data_ptr(), N,
                              mt.data_ptr(), d, f, R, mr, n_on, hbuf.data_ptr(), yp.data_ptr(),
                              sp, torch.cuda.current_stream().cuda_stream)
                fb = n_on * wbytes + R * (d * 2 + 2 * f * 2 + d * 4 * sp)
                fl = 6.0 * R * d * f
                bound = "tensor" if fl / fb > 215 else "hbm"
                out.append(Case("expert_ffn_tc (tcgen05 grouped SwiGLU, up + down)",
                                f"{m} T={T} {n_on} experts, max {mr} rows/expert, BN={bn}, "
                                f"splits={sp}", fb, ffn_launch, nbf, flops=fl, bound=bound,
                                n_kernels=2))
            # Eq. (2) combine + residual add
            ypc = torch.randn((sp, R, d), dtype=torch.float32, device=dev)
            xo = torch.empty((T, d), dtype=torch.bfloat16, device=dev)
            nbc = _copies(R * d * 4 * sp + hb, cap=8)
            ypcs = [ypc] + [torch.randn_like(ypc) for _ in range(min(nbc, 4) - 1)]

            def combine(hs=hs, ypcs=ypcs, idx=idx, pos=pos, wts=wts, T=T, k=k, d=d, sp=sp, R=R,
                        xo=xo, st={"i": 0}):
                i = st["i"]
                st["i"] += 1
                _lib.call("dali_unpermute_combine", hs[i % len(hs)].data_ptr(),
                          ypcs[i % len(ypcs)].data_ptr(), idx.data_ptr(), pos.data_ptr(),
                          wts.data_ptr(), None, None, None, T, k, d, sp, R, xo.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
            out.append(Case("unpermute_combine (Eq. 2 + residual, 128-bit scatter)",
                            f"{m} T={T} splits={sp}",
                            T * d * 2 + R * d * 4 * sp + T * d * 2 + T * k * 12, combine,
                            len(ypcs)))
        if small:
            out.extend(_small_cases(m, s, dev))
    return out


def _small_cases(m, s, dev):
    """Per-layer control kernels at decode: the fused policy step, the
    kernel copies of control data, and (Mixtral) the decode GEMV."""
    from paper_2602_03495_b200.cost_model import default_cost_model
    from paper_2602_03495_b200.policy_engine import PolicyEngine
    d, N, k = s["d"], s["N"], s["k"]
    res = []
    L = 4
    cap = 2 if N == 8 else 38
    pe = PolicyEngine(L, N, k, default_cost_model(non_moe_layer_time=3.0), prefetch_size=1,
                      residuals=torch.zeros(L - 1, d, dtype=torch.float64, device=dev),
                      cache_capacity=cap, w_size=4, seed=0)
    pe.new_run()
    wl = torch.zeros((N,), dtype=torch.int64, device=dev)
    wl[:k] = 1
    pred = wl.clone()
    import ctypes as C

    def policy(pe=pe, wl=wl, pred=pred):
        _lib.call("dali_policy_layer", C.addressof(pe.cfg), C.addressof(pe.cm_c), 0, 1, 0, 0,
                  wl.data_ptr(), pred.data_ptr(), pe.on_gpu.data_ptr(), pe.scores.data_ptr(),
                  pe.counters.data_ptr(), pe.arrived.data_ptr(), pe.slot_of.data_ptr(),
                  pe.lru_state.data_ptr(), None, 0, pe.record_ptr(0),
                  torch.cuda.current_stream().cuda_stream)
    res.append(Case("policy_layer (greedy + lookups + prefetch window + cache update)",
                    f"{m} N={N} k={k} cap={cap}", N * (8 + 8 + 1 + 1 + 4 + 8) + _lib.RECORD_BYTES,
                    policy, 1, bound="latency"))
    # control copies over mapped pinned memory (per-layer pointer table, CPU rows)
    for nbytes, what in ((17 * N, "pointer table H2D"), (2 * d * 4, "2 CPU-expert rows H2D")):
        src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)

        def cp(dst=dst, src=src, nbytes=nbytes):
            _lib.call("dali_copy_mapped", dst.data_ptr(), src.data_ptr(), nbytes,
                      torch.cuda.current_stream().cuda_stream)
        res.append(Case("copy_mapped (kernel copy over UVA-mapped pinned host memory)",
                        f"{m} {what} {nbytes} B", nbytes, cp, 1, bound="pcie-latency"))
    if s.get("gemv", m == "mixtral"):
        for M, K, what in ((s["qkv"], d, "qkv"), (d, d, "o")):
            nb = _copies(M * K * 2)
            ws = [(torch.randn(M, K, device=dev) * 0.02).to(torch.bfloat16) for _ in range(nb)]
            x = torch.randn(1, K, device=dev).to(torch.bfloat16)
            y = torch.empty(1, M, dtype=torch.bfloat16, device=dev)

            def gemv(ws=ws, x=x, y=y, M=M, K=K, st={"i": 0}):
                w = ws[st["i"] % len(ws)]
                st["i"] += 1
                _lib.call("dali_gemv_bf16", x.data_ptr(), w.data_ptr(), 1, M, K, y.data_ptr(),
                          torch.cuda.current_stream().cuda_stream)
            res.append(Case("gemv_bf16 (decode attention projection)",
                            f"{what} {M}x{K} B=1", M * K * 2 + K * 2 + M * 2, gemv, nb))
        xr = torch.randn(1, d, device=dev).to(torch.bfloat16)
        ar = torch.randn(1, d, device=dev).to(torch.bfloat16)
        wr = torch.ones(d, device=dev).to(torch.bfloat16)
        xo = torch.empty_like(xr)
        ho = torch.empty_like(xr)

        def rms(xr=xr, ar=ar, wr=wr, xo=xo, ho=ho, d=d):
            _lib.call("dali_add_rmsnorm", xr.data_ptr(), ar.data_ptr(), wr.data_ptr(), 1e-5, 1, d,
                      xo.data_ptr(), ho.data_ptr(), torch.cuda.current_stream().cuda_stream)
        res.append(Case("add_rmsnorm", f"T=1 d={d}", 5 * d * 2, rms, 1, bound="latency"))
    return res


def time_case(c: Case, iters: int = 40) -> float:
    """Device microseconds per launch (graph replay / iters)."""
    for _ in range(3):
        c.launch()
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph):
        for _ in range(iters):
            c.launch()
    gph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        e0.record()
        gph.replay()
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        best = us if best is None else min(best, us)
    del gph
    return best


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def row(c: Case, us: float) -> dict:
    hbm, tf, kind = peaks()
    r = {"kernel": c.kernel, "case": c.label, "us": round(us, 2),
         "algorithmic_bytes": int(c.bytes), "bound": c.bound, "kernels_per_case": c.n_kernels,
         "input_copies": c.bufs}
    gbs = c.bytes / (us * 1e-6) / 1e9
    r["achieved_gbs"] = round(gbs, 1)
    if c.bound == "tensor":
        tfs = c.flops / (us * 1e-6) / 1e12
        r.update(achieved_tflops=round(tfs, 1), peak=tf, unit="TFLOP/s",
                 frac=round(tfs / tf, 4))
    elif c.bound == "hbm":
        r.update(peak=hbm, unit="GB/s", frac=round(gbs / hbm, 4))
    else:
        r.update(peak=None, unit="us", frac=None)
    r["peak_kind"] = kind
    return r


def run_time(out_path, which, Ts, only=None, iters=40):
    torch.cuda.set_device(0)
    rows = []
    for c in cases(which, Ts):
        if only and only not in c.key:
            continue
        us = time_case(c, iters)
        rows.append(row(c, us))
        print(json.dumps(rows[-1]), flush=True)
    if out_path:
        json.dump(rows, open(out_path, "w"), indent=1)


def run_ncu(manifest, which, Ts):
    torch.cuda.set_device(0)
    cs = cases(which, Ts)
    for c in cs:
        for _ in range(2):
            c.launch()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for c in cs:
        torch.cuda._sleep(1000)
        c.launch()
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    json.dump([{"key": c.key, "kernel": c.kernel, "case": c.label, "bytes": c.bytes,
                "flops": c.flops, "bound": c.bound} for c in cs], open(manifest, "w"), indent=1)


def _ncu_rows(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {n: h.index(n) for n in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                  "Metric Value")}
    launches = {}
    order = []
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}
    for r in rows[1:]:
        i = r[ix["ID"]]
        if i not in launches:
            launches[i] = {"name": r[ix["Kernel Name"]]}
            order.append(i)
        v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
        launches[i][r[ix["Metric Name"]]] = v
    return [launches[i] for i in order]


def summarize(ncu_csv, time_json, manifest):
    hbm, tf, kind = peaks()
    man = json.load(open(manifest))
    times = {f"{r['kernel']} [{r['case']}]": r for r in json.load(open(time_json))} \
        if time_json and os.path.exists(time_json) else {}
    groups, cur = [], None
    for ln in _ncu_rows(ncu_csv):
        if "spin_kernel" in ln["name"]:
            if cur is not None:
                groups.append(cur)
            cur = []
        elif cur is not None:
            cur.append(ln)
    groups = [g_ for g_ in groups]
    out = []
    print(f"# Per-kernel table (peaks: HBM {hbm} GB/s, bf16 {tf} TF/s sustained; {kind})\n")
    print("ncu: cold caches (flushed before each kernel), serialised, `--clock-control none`; "
          "live: CUDA-graph replay over rotating input copies (tools/kernel_table.py --time).\n")
    print("| kernel | case | algorithmic MB | ncu us | ncu DRAM MB (r+w) | DRAM / algorithmic | "
          "ncu achieved | live us | live achieved | live frac |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for m, g_ in zip(man, groups):
        us = sum(x.get("gpu__time_duration.sum", 0.0) for x in g_)
        dram = sum(x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
                   for x in g_)
        names = sorted({re.sub(r"^void ", "", re.sub(r"\(.*", "", x["name"]))[:40] for x in g_})
        t = times.get(m["key"], {})
        if m["bound"] == "tensor":
            ach = f"{m['flops'] / (us * 1e-6) / 1e12:.0f} TF/s" if us else "-"
            live = f"{t['achieved_tflops']:.0f} TF/s" if t else "-"
        else:
            ach = f"{m['bytes'] / (us * 1e-6) / 1e9:.0f} GB/s" if us else "-"
            live = f"{t['achieved_gbs']:.0f} GB/s" if t else "-"
        fr = f"{t['frac']:.3f}" if t and t.get("frac") is not None else "-"
        print(f"| {m['kernel'].split(' ')[0]} ({', '.join(names)}) | {m['case']} | "
              f"{m['bytes'] / 1e6:.3f} | {us:.1f} | {dram / 1e6:.3f} | "
              f"{(dram / m['bytes']) if m['bytes'] else 0:.2f} | {ach} | "
              f"{t.get('us', '-')} | {live} | {fr} |")
        out.append({**m, "ncu_us": round(us, 2), "ncu_dram_bytes": int(dram),
                    "dram_over_algorithmic": round(dram / m["bytes"], 3) if m["bytes"] else None,
                    "ncu_kernels": names, "live": t or None})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--summarize", nargs=2, metavar=("NCU_CSV", "TIME_JSON"))
    ap.add_argument("--manifest", default=os.path.join(ROOT, "gpurun_out", "kt_manifest.json"))
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "kt_time.json"))
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--which", default="mixtral,dsv2")
    ap.add_argument("--T", default="1,512,4096")
    ap.add_argument("--only", default=None, help="substring filter on the case key (--time)")
    ap.add_argument("--iters", type=int, default=40)
    a = ap.parse_args()
    which = tuple(a.which.split(","))
    Ts = tuple(int(x) for x in a.T.split(","))
    if a.time:
        run_time(a.out, which, Ts, a.only, a.iters)
    if a.ncu:
        run_ncu(a.manifest, which, Ts)
    if a.summarize:
        res = summarize(a.summarize[0], a.summarize[1], a.manifest)
        if a.json_out:
            json.dump(res, open(a.json_out, "w"), indent=1)


if __name__ == "__main__":
    main()
