"""numpy fp32 restatement of the expert forward (TEST INFRASTRUCTURE ONLY).

Expert MLP ``Y = gelu_tanh(X W1^T) W2^T`` in float32 (the repo's definition;
the reference has no numerical experts -- parity for outputs is *unpinned by
the reference* and pinned here by tolerance).  ``bf16_hidden`` optionally
rounds the hidden activation and each stage output to bf16 the way the GPU
stores them, which isolates accumulation-order differences.
"""

from __future__ import annotations

import numpy as np

from .synth import to_bf16


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.float32)
    return (np.float32(0.5) * x * (np.float32(1.0) + np.tanh(
        np.float32(0.7978845608028654) * (x + np.float32(0.044715) * x * x * x)))).astype(np.float32)


def expert_forward(x: np.ndarray, w1: np.ndarray, w2: np.ndarray, bf16_hidden: bool = False) -> np.ndarray:
    hidden = gelu_tanh(x @ w1.T)
    if bf16_hidden:
        hidden = to_bf16(hidden)
    y = (hidden @ w2.T).astype(np.float32)
    return to_bf16(y) if bf16_hidden else y


def chain_forward(x: np.ndarray, experts: list, weights, bf16_hidden: bool = False) -> np.ndarray:
    """Run one request's expert chain; ``weights(e) -> (W1, W2)``."""
    out = x
    for e in experts:
        w1, w2 = weights(e)
        out = expert_forward(out, w1, w2, bf16_hidden)
    return out


def rel_l2(got: np.ndarray, ref: np.ndarray) -> float:
    ref = ref.astype(np.float64)
    return float(np.linalg.norm(got.astype(np.float64) - ref) / max(np.linalg.norm(ref), 1e-30))
