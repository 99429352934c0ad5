"""Named workload shapes (BASELINE.json `configs`).

Each entry fixes the MoE geometry (layers, hidden, experts, top-k, expert
intermediate size, shared experts), the request (visual + text tokens), the
compression budgets, the pinned prefix and the GPU expert budget (slabs), the
lookahead predictor, and the synthetic trace-generator knobs used when a
workload is replayed from a routing trace instead of a live router.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Workload:
    name: str
    layers: int
    hidden: int
    experts: int
    k: int
    inter: int
    n_visual: int
    n_text: int
    alpha: float
    beta: float
    lam: float
    l_pinned: int
    num_slabs: int
    predictor: str
    budget: int
    window: int
    gamma: float = 0.8
    history_decay: float = 0.5
    shared_experts: int = 0
    grace: int = 1
    gen: dict = field(default_factory=dict)

    @property
    def prefix_layers(self) -> tuple[int, ...]:
        return tuple(range(self.l_pinned))

    @property
    def expert_bytes(self) -> int:
        """bf16 SwiGLU expert: gate + up [I, H] and down [H, I]."""
        return 3 * self.hidden * self.inter * 2

    @property
    def n_tokens(self) -> int:
        return self.n_visual + self.n_text

    def trace_config(self, seed: int = 0, decode_steps: int = 0):
        from .trace import TraceGenConfig

        return TraceGenConfig(
            n_visual=self.n_visual, n_text=self.n_text, layers=self.layers,
            experts=self.experts, k=self.k, seed=seed, decode_steps=decode_steps,
            shared_experts=self.shared_experts, **self.gen,
        )


WORKLOADS = {
    # C1: the reference's own CPU-runnable tiny stack (H/I/L are builder choices)
    "c1_tiny": Workload("c1_tiny", layers=8, hidden=256, experts=8, k=2, inter=512,
                        n_visual=576, n_text=64, alpha=0.05, beta=0.25, lam=2.0,
                        l_pinned=2, num_slabs=24, predictor="oracle", budget=4, window=3,
                        gen=dict(cluster_support=4, visual_noise=0.3)),
    # C2: MoE-LLaVA-Phi2 shape; GPU budget = 50% of the 56 non-pinned experts
    "c2_phi2": Workload("c2_phi2", layers=16, hidden=2560, experts=4, k=2, inter=10240,
                        n_visual=576, n_text=64, alpha=0.1, beta=0.5, lam=2.0,
                        l_pinned=2, num_slabs=28, predictor="history", budget=2, window=3,
                        gen=dict(cluster_support=4, visual_noise=0.3)),
    # C3: Qwen3-VL-30B-A3B shape, high-res image, tight cache (826 slabs)
    "c3_qwen3vl": Workload("c3_qwen3vl", layers=48, hidden=2048, experts=128, k=8, inter=768,
                           n_visual=2304, n_text=64, alpha=0.1, beta=0.5, lam=2.0,
                           l_pinned=8, num_slabs=826, predictor="oracle", budget=20, window=5,
                           gen=dict(visual_noise=0.3)),
    # C4: DeepSeek-VL2-Small shape, 3 images, 2 shared experts, history lookahead
    "c4_dsvl2s": Workload("c4_dsvl2s", layers=26, hidden=2048, experts=64, k=6, inter=1408,
                          n_visual=1176, n_text=96, alpha=0.1, beta=0.5, lam=2.0,
                          l_pinned=4, num_slabs=352, predictor="history", budget=20, window=5,
                          shared_experts=2, gen=dict(clusters=6, cluster_support=16, visual_noise=0.3)),
}
