"""CIDRA block repositioning, the plain definition — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

PAPER.md §5.5-§5.5.1: a cached KV block whose stored position differs from
the position a later query needs is *repositioned* — "a ReRoPE, which reverses and then
re-applies a Rotational Positional Encoding". CIDRA formulates the moves as a dependency
graph ("block A moved to block B, B to C, and so on"), duplicates blocks with out-degree
> 1 and runs the resulting permutation in place, cycle by cycle.

Whatever order and scratch the in-place algorithm uses, the pool it must reach has a plain
definition (SPEC S:406 `oracle_reposition`, "full-copy non-in-place computation of every
destination from pristine sources"): for every move (src, dst, old_pos, new_pos)

  K'[dst][t] = rerope(K[src][t], old_pos + t, new_pos + t)      t = 0..bs-1 (all layers, heads)
  V'[dst][t] = V[src][t]                                         (V carries no position)

and every block that is no move's destination keeps its content. All tokens of a block share
one position shift (SPEC design decision S:424, "spans move as whole blocks"). This module
computes exactly that, out of place, in fp64. A destination may appear only once (two writes to
one block are contradictory); a source may feed several destinations — that is the paper's
"duplication", implicit in copy semantics.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np

from . import rope as _rope

Move = Tuple[int, int, int, int]  # (src block, dst block, old position of token 0, new position of token 0)


def validate(moves: Sequence[Move], num_blocks: int) -> None:
    """Raise ValueError for an out-of-range block id or a destination written twice."""
    seen = set()
    for src, dst, _, _ in moves:
        if not (0 <= src < num_blocks and 0 <= dst < num_blocks):
            raise ValueError(f"block id out of range: {src} -> {dst}")
        if dst in seen:
            raise ValueError(f"block {dst} is the destination of two moves")
        seen.add(dst)


def reposition(k_pool: np.ndarray, v_pool: np.ndarray, moves: Sequence[Move], base: float):
    """Pools [L][num_blocks][Hkv][bs][d] (any float dtype, decoded to fp64). Returns (K', V') fp64."""
    k0 = np.asarray(k_pool, dtype=np.float64)
    v0 = np.asarray(v_pool, dtype=np.float64)
    validate(moves, k0.shape[1])
    k1, v1 = k0.copy(), v0.copy()
    bs = k0.shape[3]
    t = np.arange(bs, dtype=np.float64)  # token offsets in the block, broadcast over [L][Hkv]
    for src, dst, old0, new0 in moves:
        k1[:, dst] = _rope.rerope(k0[:, src], old0 + t, new0 + t, base)  # [L][Hkv][bs][d]
        v1[:, dst] = v0[:, src]
    return k1, v1


def out_degree_duplicates(moves: Sequence[Move]) -> int:
    """The paper's duplication count for a move set: sum over sources of max(0, out-degree - 1)
    ("Duplication minimality")."""
    deg = {}
    for src, _, _, _ in moves:
        deg[src] = deg.get(src, 0) + 1
    return sum(max(0, c - 1) for c in deg.values())
