"""Span-query tree normalization — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

A span query is an expression tree (Def. "Span Query", §4.1) over ⊕
(commutative join) and ⋈ (non-commutative join) (Def. P:333-335). The hot path accepts the
optimized RAG / judge form ⋈[prefix?, ⊕[fragments…]?, cross]. Nested ⊕
is flattened (the "plus simplification" rule) and a ⋈ of token leaves inside a ⊕ is one
fragment (its leaves concatenated in order).

Node rows are (op, num_children, tok_begin, tok_len) in pre-order; op 0 = TOKENS, 1 = PLUS,
2 = CROSS (include/spanq.h).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

TOKENS, PLUS, CROSS = 0, 1, 2


class TreeError(ValueError):
    """Invalid tree (the C-ABI returns SPQ_EINVAL for the same inputs)."""


def _subtree(nodes, i):
    """Return (index after subtree i)."""
    if i >= len(nodes):
        raise TreeError("truncated tree")
    op, nc = int(nodes[i][0]), int(nodes[i][1])
    j = i + 1
    for _ in range(nc):
        j = _subtree(nodes, j)
    return j


def _leaf_tokens(nodes, tokens, i) -> np.ndarray:
    op, nc, b, n = (int(v) for v in nodes[i])
    if op != TOKENS or nc != 0:
        raise TreeError("expected TOKENS leaf")
    if n <= 0:
        raise TreeError("empty token leaf")
    if b < 0 or b + n > len(tokens):
        raise TreeError("token range out of bounds")
    t = np.asarray(tokens[b : b + n], dtype=np.int64)
    if (t < 0).any():
        raise TreeError("negative token id")
    return t.astype(np.int32)


def _fragments(nodes, tokens, i, out: List[np.ndarray]) -> int:
    """Collect the fragments under a PLUS node (flattening nested PLUS); return next index."""
    op, nc = int(nodes[i][0]), int(nodes[i][1])
    if op != PLUS:
        raise TreeError("expected PLUS")
    if nc < 1:
        raise TreeError("PLUS needs >= 1 child")  # S:42 arity
    j = i + 1
    for _ in range(nc):
        cop = int(nodes[j][0])
        if cop == TOKENS:
            out.append(_leaf_tokens(nodes, tokens, j))
            j += 1
        elif cop == PLUS:
            j = _fragments(nodes, tokens, j, out)
        elif cop == CROSS:
            cnc = int(nodes[j][1])
            if cnc < 1:
                raise TreeError("CROSS needs >= 1 child")
            parts = []
            k = j + 1
            for _ in range(cnc):
                parts.append(_leaf_tokens(nodes, tokens, k))
                k += 1
            out.append(np.concatenate(parts))
            j = k
        else:
            raise TreeError("bad op")
    return j


def normalize(nodes, tokens) -> Tuple[np.ndarray, List[np.ndarray], np.ndarray]:
    """Tree -> (prefix, fragments in ⊕ order, cross)."""
    nodes = np.asarray(nodes, dtype=np.int64).reshape(-1, 4)
    if len(nodes) == 0:
        raise TreeError("empty tree")
    for r in nodes:
        if int(r[0]) not in (TOKENS, PLUS, CROSS):
            raise TreeError("bad op")
        if int(r[1]) < 0:
            raise TreeError("bad arity")
    if _subtree(nodes, 0) != len(nodes):
        raise TreeError("node count mismatch")
    op, nc = int(nodes[0][0]), int(nodes[0][1])
    if op != CROSS or nc < 1:
        raise TreeError("root must be CROSS with >= 1 child")
    kids = []
    j = 1
    for _ in range(nc):
        kids.append(j)
        j = _subtree(nodes, j)
    ops = [int(nodes[k][0]) for k in kids]
    prefix = np.zeros(0, np.int32)
    frags: List[np.ndarray] = []
    if ops[-1] != TOKENS:
        raise TreeError("last child must be the cross TOKENS leaf")
    cross = _leaf_tokens(nodes, tokens, kids[-1])
    rest = kids[:-1]
    rops = ops[:-1]
    if rops == [TOKENS, PLUS]:
        prefix = _leaf_tokens(nodes, tokens, rest[0])
        _fragments(nodes, tokens, rest[1], frags)
    elif rops == [TOKENS]:
        prefix = _leaf_tokens(nodes, tokens, rest[0])
    elif rops == [PLUS]:
        _fragments(nodes, tokens, rest[0], frags)
    elif rops == []:
        pass
    else:
        raise TreeError("unsupported tree shape")
    return prefix, frags, cross
