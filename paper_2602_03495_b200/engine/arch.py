"""Model shapes for the inference engine (new API; the reference has no model).

``MoEArch`` extends the reference ``ModelConfig`` (routing shape,
trace.py:44-86) with what real execution needs: expert FFN width, attention
geometry, vocabulary, and whether top-k weights are renormalised.  Widths of
the BASELINE shapes come from the public model configs.
Attention is standard GQA for every preset (DeepSeek's MLA is out of scope:
attention is not one of the five DALI subsystems).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

from ..trace import ModelConfig


@dataclass(frozen=True)
class MoEArch:
    name: str
    num_layers: int
    hidden_dim: int
    num_experts: int
    top_k: int
    ffn_dim: int               # routed expert intermediate size (f)
    num_heads: int
    num_kv_heads: int
    head_dim: int
    vocab_size: int
    norm_topk_prob: bool
    num_shared_experts: int = 0
    shared_ffn_dim: int = 0        # total intermediate width of the shared expert(s)
    shared_gate: bool = False      # Qwen-style sigmoid gate on the shared output
    rope_theta: float = 1e6
    rms_eps: float = 1e-5

    @property
    def routing(self) -> ModelConfig:
        return ModelConfig(self.num_layers, self.num_experts, self.num_shared_experts,
                           self.top_k, self.hidden_dim)

    @property
    def expert_elems(self) -> int:
        """bf16 elements of one expert block: W13 (2f, d) + W2 (d, f)."""
        return 3 * self.ffn_dim * self.hidden_dim

    @property
    def expert_bytes(self) -> int:
        return 2 * self.expert_elems


PRESETS = {
    # BASELINE configs[0]: tiny random-init MoE (4 layers, 8 experts, top-2, d 256)
    "tiny": MoEArch("tiny", 4, 256, 8, 2, 512, 4, 2, 64, 1024, True, rope_theta=1e4),
    # tiny Qwen-style variant: wide pool, no renorm, gated shared expert (test shape)
    "tiny-shared": MoEArch("tiny-shared", 4, 256, 16, 4, 256, 4, 4, 64, 1024, False,
                           num_shared_experts=1, shared_ffn_dim=512, shared_gate=True,
                           rope_theta=1e4),
    # BASELINE configs[1]: Mixtral-8x7B shape
    "mixtral-8x7b": MoEArch("mixtral-8x7b", 32, 4096, 8, 2, 14336, 32, 8, 128, 32000, True),
    # BASELINE configs[2]: Qwen1.5-MoE-A2.7B (60 routed top-4 + gated shared expert 5632)
    "qwen1.5-moe-a2.7b": MoEArch("qwen1.5-moe-a2.7b", 24, 2048, 60, 4, 1408, 16, 16, 128,
                                 151936, False, num_shared_experts=1, shared_ffn_dim=5632,
                                 shared_gate=True),
    # BASELINE configs[3]: DeepSeek-V2-Lite MoE layers (64 routed top-6 + 2 shared x 1408;
    # GQA stand-in attention)
    "deepseek-v2-lite": MoEArch("deepseek-v2-lite", 26, 2048, 64, 6, 1408, 16, 16, 128,
                                102400, False, num_shared_experts=2, shared_ffn_dim=2816),
    # BASELINE configs[4]: Mixtral-8x22B shape
    "mixtral-8x22b": MoEArch("mixtral-8x22b", 56, 6144, 8, 2, 16384, 48, 8, 128, 32768, True),
}


def preset(name: str) -> MoEArch:
    """A preset by name; ``<name>@L<n>`` is the same shape at depth n (e.g.
    Mixtral-8x22B at a depth one GPU's HBM or one host's DRAM holds)."""
    base, _, depth = name.partition("@L")
    if base not in PRESETS:
        raise KeyError(f"unknown arch {base!r}; choose from {sorted(PRESETS)}")
    a = PRESETS[base]
    if depth:
        n = int(depth)
        if n < 1:
            raise KeyError(f"bad depth in {name!r}")
        a = replace(a, name=name, num_layers=n)
    return a
