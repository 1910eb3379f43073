"""numpy restatement of the seeded synthetic data (TEST INFRASTRUCTURE ONLY).

Bit-identical to ``fill_uniform_bf16`` / ``coe_expert_seed`` in
``paper_2503_02354_b200/csrc/{group_sort,runtime}.cu``: element i of a stream
with seed s is splitmix64(s + (i+1)*phi) -> top 24 bits -> u in [0,1) ->
(u - 0.5) * 2*scale in fp32 -> bf16 (round to nearest even).  Returned as
float32 arrays holding exactly the bf16 values.
"""

from __future__ import annotations

import numpy as np

_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


def _splitmix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix64(x: int) -> int:
    z = x & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def to_bf16(v: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (nearest even), returned as float32."""
    bits = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bits = (bits + np.uint64(0x7FFF) + ((bits >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return bits.astype(np.uint32).view(np.float32)


def uniform_bf16(seed: int, start: int, count: int, scale: float) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = _splitmix(np.uint64(seed & _MASK) + i * _PHI)
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    v = (u - np.float32(0.5)) * (np.float32(2.0) * np.float32(scale))
    return to_bf16(v)


def expert_seed(weight_seed: int, expert: int, matrix: int) -> int:
    return splitmix64((weight_seed ^ (((2 * expert + matrix + 1) * 0xD1B54A32D192ED03) & _MASK)) & _MASK)


def expert_weights(weight_seed: int, expert: int, d: int, h: int):
    """(W1 [h, d], W2 [d, h]) float32 holding the bf16 weights."""
    s1 = np.sqrt(np.float32(3.0) / np.float32(d)).astype(np.float32)
    s2 = np.sqrt(np.float32(3.0) / np.float32(h)).astype(np.float32)
    w1 = uniform_bf16(expert_seed(weight_seed, expert, 0), 0, h * d, float(s1)).reshape(h, d)
    w2 = uniform_bf16(expert_seed(weight_seed, expert, 1), 0, d * h, float(s2)).reshape(d, h)
    return w1, w2


def request_inputs(input_seed: int, request: int, T: int, d: int) -> np.ndarray:
    """Rows [request*T, (request+1)*T) of the X buffer filled by coe_runtime_fill_inputs."""
    scale = float(np.sqrt(np.float32(3.0)).astype(np.float32))
    return uniform_bf16(input_seed, request * T * d, T * d, scale).reshape(T, d)
