"""Rotary positional encoding (RoPE), fp64 — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

PAPER.md §5.5 (LaTeX line ~471, "re-applies a Rotational Positional Encoding", citing RoFormer)
gives no formula; SPEC.md S:358 fixes θ_i = base^(−2i/d) for pair index i ∈ [0, d/2), default
base 10000. Reading R15: pairs are rotate-half (i, i + d/2), the HF/vLLM
Llama/Granite convention (Granite is the paper's model family).

  rope(x, p)[i]       = x[i]       cos(p θ_i) − x[i+d/2] sin(p θ_i)
  rope(x, p)[i+d/2]   = x[i+d/2]   cos(p θ_i) + x[i]     sin(p θ_i)
"""
from __future__ import annotations

import numpy as np


def inv_freq(d: int, base: float) -> np.ndarray:
    """θ_i = base^(−2i/d), i = 0..d/2−1."""
    i = np.arange(d // 2, dtype=np.float64)
    return np.power(np.float64(base), -2.0 * i / d)


def rope(x: np.ndarray, pos, base: float) -> np.ndarray:
    """Rotate the last axis of ``x`` (fp64) by position(s) ``pos`` (broadcast over leading axes).

    ``pos`` has the shape of ``x.shape[:-1]`` or a prefix of it padded on the right with 1s
    (e.g. [T,1] for x [T,H,d]).
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    p = np.asarray(pos, dtype=np.float64)
    ang = p[..., None] * inv_freq(d, base)
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., : d // 2], x[..., d // 2 :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rerope(x: np.ndarray, old_pos, new_pos, base: float) -> np.ndarray:
    """ReRoPE: reverse the encoding at ``old_pos`` and re-apply it at ``new_pos``."""
    return rope(rope(x, -np.asarray(old_pos, dtype=np.float64), base), new_pos, base)
