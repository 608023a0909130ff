"""CPU oracle for the DALI hot path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (``paper_2602_03495_b200``) imports this
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and there only as
the checker or as the timed CPU reference arm -- never as the thing measured
on the GPU path.

Contents
--------
policy.py   numpy restatement of the reference ``moesim`` hot-path functions
            (gating, cost model, greedy assignment, residual prefetch,
            workload-aware cache), each citing the reference file:line.
driver.py   restatement of ``simulate_run``'s per-step x per-layer loop
            (reference ``simulator.py:318-522``) that also records every
            decision (C/G vectors, prefetch sets, arrivals, lookups,
            replacement events) so the GPU engine's decision log can be
            compared entry by entry.
model_cpu.py  torch fp32/bf16 CPU restatement of the MoE forward (Eq. 1-2 of
            the paper, SwiGLU experts) -- the numeric oracle for hidden states
            and logits.  The reference has no model, so this part is
            "parity unpinned" by any reference test.

Pinning: ``tests/golden/make_golden.py`` imports the real reference
(``/root/reference/pkg/src``) in the build container and freezes its outputs
into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
restatement against those fixtures on every CPU test run.
"""
