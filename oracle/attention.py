"""Span-masked prefill attention, fp64 — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Plain definition (§5.6 P:672 "the tokens within a document only attend
to prior tokens in that same document"): for one query, concatenate
[prefix | fragments in ⊕ order | cross] into N tokens at global positions 0..N−1 and attend
with the visible mask

  * prefix row i sees prefix columns j ≤ i;
  * fragment-f row i sees columns j ≤ i inside fragment f only (a fragment is prepared
    "independent of context", P:436 footnote; reading R1);
  * cross row i sees every column j ≤ i (the ⋈ join over everything before it).

O = softmax(mask(RoPE(q,pos)·RoPE(k,pos)ᵀ/√d))·V per q-head h, kv-head h // (Hq/Hkv)
(readings R14-R17: scale 1/√d, natural-log LSE, GQA grouping, causal diagonal included).

`dense_masked` is that definition written out (N×N mask, tiny inputs). `segment_causal` and
`join_rows` are the segment-wise form the method computes (fragment rows at span-local
positions 0..L−1, cross rows at global positions); tests pin them to `dense_masked`.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from .rope import rope


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, mask: np.ndarray,
           heads: Optional[Sequence[int]] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Masked softmax attention, rotated inputs.

    q [R,Hq,d], k [N,Hkv,d], v [N,Hkv,d] (fp64), mask bool [R,N]. Returns O [R,H',d] and
    natural-log LSE [R,H'] for the requested q heads (all by default).
    """
    R, hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    heads = list(range(hq)) if heads is None else list(heads)
    out = np.zeros((R, len(heads), d))
    lse = np.zeros((R, len(heads)))
    scale = 1.0 / np.sqrt(d)
    for j, h in enumerate(heads):
        s = (q[:, h, :] @ k[:, h // g, :].T) * scale
        s = np.where(mask, s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        p = np.exp(s - m)
        l = p.sum(axis=1, keepdims=True)
        out[:, j, :] = (p @ v[:, h // g, :]) / l
        lse[:, j] = (m + np.log(l))[:, 0]
    return out, lse


def visible_mask(n_prefix: int, frag_lens: Sequence[int], n_cross: int) -> np.ndarray:
    """Boolean N×N mask of the plain definition."""
    N = n_prefix + sum(frag_lens) + n_cross
    m = np.zeros((N, N), dtype=bool)
    for i in range(n_prefix):
        m[i, : i + 1] = True
    off = n_prefix
    for L in frag_lens:
        for i in range(L):
            m[off + i, off : off + i + 1] = True
        off += L
    for i in range(off, N):
        m[i, : i + 1] = True
    return m


def dense_masked(prefix, frags, cross, eq, ek, ev, base: float,
                 heads: Optional[Sequence[int]] = None):
    """The plain definition on one query: O [N,H,d], LSE [N,H], mask [N,N]."""
    toks = np.concatenate([np.asarray(prefix, np.int64)] + [np.asarray(f, np.int64) for f in frags]
                          + [np.asarray(cross, np.int64)])
    N = len(toks)
    pos = np.arange(N, dtype=np.float64)
    q = rope(_f64(eq[toks]), pos[:, None], base)
    k = rope(_f64(ek[toks]), pos[:, None], base)
    v = _f64(ev[toks])
    mask = visible_mask(len(prefix), [len(f) for f in frags], len(cross))
    o, l = attend(q, k, v, mask, heads)
    return o, l, mask


def segment_causal(tokens, eq, ek, ev, base: float, rows: Optional[Sequence[int]] = None,
                   heads: Optional[Sequence[int]] = None):
    """A prefix or fragment job: causal attention at span-local positions 0..L−1
    (fragments prepared independently of context, P:436 fn; reading R2). Returns rows' O, LSE."""
    t = np.asarray(tokens, np.int64)
    L = len(t)
    rows = np.arange(L) if rows is None else np.asarray(rows)
    pos = np.arange(L, dtype=np.float64)
    q = rope(_f64(eq[t[rows]]), pos[rows][:, None], base)
    k = rope(_f64(ek[t]), pos[:, None], base)
    v = _f64(ev[t])
    mask = np.arange(L)[None, :] <= rows[:, None]
    return attend(q, k, v, mask, heads)


def join_rows(prefix, frags, cross, eq, ek, ev, base: float,
              rows: Optional[Sequence[int]] = None, heads: Optional[Sequence[int]] = None):
    """Cross rows of the ⋈ join: row j (global position P+S+j) attends to the whole prefix,
    every fragment and cross rows ≤ j, all at global positions ("new position")."""
    toks = np.concatenate([np.asarray(prefix, np.int64)] + [np.asarray(f, np.int64) for f in frags]
                          + [np.asarray(cross, np.int64)])
    N = len(toks)
    C = len(cross)
    base_row = N - C
    rows = np.arange(C) if rows is None else np.asarray(rows)
    gpos = base_row + rows
    q = rope(_f64(eq[toks[gpos]]), gpos[:, None].astype(np.float64), base)
    k = rope(_f64(ek[toks]), np.arange(N, dtype=np.float64)[:, None], base)
    v = _f64(ev[toks])
    mask = np.arange(N)[None, :] <= gpos[:, None]
    return attend(q, k, v, mask, heads)


def expected_pages(tokens, eq_unused, ek, ev, base: float, positions) -> Tuple[np.ndarray, np.ndarray]:
    """K/V rows as stored in the pool: RoPE(k, stored position), v unrotated (R15: RoPE on q, k)."""
    t = np.asarray(tokens, np.int64)
    return rope(_f64(ek[t]), np.asarray(positions, np.float64)[:, None], base), _f64(ev[t])


# ----------------------------------------------------------------------------- plan-level
def plan_prefill_expected(view, queries, eq, ek, ev, base: float,
                          heads: Optional[Sequence[int]] = None):
    """Expected O/LSE of the plan's packed prefill rows (job order, store.PlanView)."""
    outs, lses = [], []
    for si in view.jobs:
        seg = view.segments[si]
        prefix, frags, cross = queries[seg.query]
        toks = prefix if seg.kind == 0 else frags[seg.frag_idx]
        rows = np.arange(seg.compute_begin, seg.tok_len)
        o, l = segment_causal(toks, eq, ek, ev, base, rows, heads)
        outs.append(o)
        lses.append(l)
    if not outs:
        return np.zeros((0, 0, 0)), np.zeros((0, 0))
    return np.concatenate(outs), np.concatenate(lses)


def plan_join_expected(view, queries, eq, ek, ev, base: float,
                       heads: Optional[Sequence[int]] = None, q_range=None):
    outs, lses = [], []
    qs = range(len(queries)) if q_range is None else range(*q_range)
    for qi in qs:
        prefix, frags, cross = queries[qi]
        o, l = join_rows(prefix, frags, cross, eq, ek, ev, base, None, heads)
        outs.append(o)
        lses.append(l)
    return np.concatenate(outs), np.concatenate(lses)
