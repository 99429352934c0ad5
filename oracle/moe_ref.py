"""Oracle for the parts of the layer with no reference implementation
("parity unpinned"): router, permutation, SwiGLU expert FFN,
combine.  Plain torch CPU fp32/fp64 restatements of the intended math:

* router   logits = X W_g^T (fp64 here, exact for small-integer inputs);
           top-k by (logit desc, id asc); gates = softmax over the k picks
* permute  stable sort of (token, slot) picks by expert
* FFN      h = SiLU(x W_gate^T) * (x W_up^T) (rounded to bf16, as the device
           stores H1), y = h W_down^T (fp32), output bf16
* combine  out = resid + sum_j gate_j * y_j
"""
from __future__ import annotations

import numpy as np
import torch


def route(x: torch.Tensor, wg: torch.Tensor, k: int):
    logits = x.double() @ wg.double().T
    n, e = logits.shape
    ids = np.lexsort((np.broadcast_to(np.arange(e), (n, e)), -logits.numpy()), axis=1)[:, :k]
    ids = torch.from_numpy(np.ascontiguousarray(ids)).long()
    sel = torch.gather(logits, 1, ids)
    gates = torch.softmax(sel, dim=1)
    return ids.int(), gates.float(), logits


def permute(ids: torch.Tensor, experts: int):
    n, k = ids.shape
    flat = ids.reshape(-1).long()
    order = torch.from_numpy(np.argsort(flat.numpy(), kind="stable"))
    counts = torch.bincount(flat, minlength=experts)
    offsets = torch.zeros(experts + 1, dtype=torch.long)
    offsets[1:] = torch.cumsum(counts, 0)
    pos = torch.empty_like(flat)
    pos[order] = torch.arange(flat.numel())
    return offsets, order // k, pos.reshape(n, k)


def expert_ffn(x: torch.Tensor, w_gate: torch.Tensor, w_up: torch.Tensor, w_down: torch.Tensor):
    """x bf16 [m, H]; w_* bf16 ([I,H],[I,H],[H,I]) -> (h1 bf16 [m, I], y bf16 [m, H])."""
    xf = x.float()
    g = xf @ w_gate.float().T
    u = xf @ w_up.float().T
    h = (g * torch.sigmoid(g) * u).to(torch.bfloat16)
    y = (h.float() @ w_down.float().T).to(torch.bfloat16)
    return h, y


def combine(y_perm: torch.Tensor, pos: torch.Tensor, gates: torch.Tensor, resid: torch.Tensor | None):
    n, k = gates.shape
    acc = torch.zeros(n, y_perm.shape[1], dtype=torch.float32)
    for j in range(k):
        acc += gates[:, j:j + 1].float() * y_perm[pos[:, j].long()].float()
    if resid is not None:
        acc += resid.float()
    return acc.to(torch.bfloat16)
