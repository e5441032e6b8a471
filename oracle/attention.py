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


def decode_row(prefix, frags, cross, gen, t: int, eq, ek, ev, base: float,
               heads: Optional[Sequence[int]] = None):
    """Token generation after the join (§4.1 "G"): generated token t sits
    right after the cross tokens and the t tokens generated before it (global position
    P+S+C+t, reading R3) and, being the next ordered token, attends to everything before it and
    itself — the plain definition's cross row of the query whose cross is cross ‖ gen[0..t]."""
    ext = np.concatenate([np.asarray(cross, np.int64), np.asarray(gen[: t + 1], np.int64)])
    return join_rows(prefix, frags, ext, eq, ek, ev, base, rows=[len(cross) + t], heads=heads)


def join_rows_subset(prefix, frags, cross, eq, ek, ev, base: float, local: bool, frag_mask: Sequence[bool],
                     heads: Optional[Sequence[int]] = None):
    """The join's cross rows restricted to a subset of the key columns — the prefix and cross
    columns when `local`, fragment f's columns when frag_mask[f] — normalized over that subset:
    the partial (O, LSE) one rank of an owner-side split join computes."""
    toks = np.concatenate([np.asarray(prefix, np.int64)] + [np.asarray(f, np.int64) for f in frags]
                          + [np.asarray(cross, np.int64)])
    N, C, P = len(toks), len(cross), len(prefix)
    gpos = (N - C) + np.arange(C)
    keep = np.zeros(N, bool)
    keep[:P] = local
    keep[N - C:] = local
    off = P
    for f, m in zip(frags, frag_mask):
        keep[off:off + len(f)] = m
        off += len(f)
    q = rope(_f64(eq[toks[gpos]]), gpos[:, None].astype(np.float64), base)
    k = rope(_f64(ek[toks]), np.arange(N, dtype=np.float64)[:, None], base)
    mask = (np.arange(N)[None, :] <= gpos[:, None]) & keep[None, :]
    return attend(q, k, _f64(ev[toks]), mask, heads)


def merge_lse(parts: Sequence[Tuple[np.ndarray, np.ndarray]]) -> Tuple[np.ndarray, np.ndarray]:
    """Merge partial attention results over disjoint key sets (normalized O_i, natural-log LSE_i):
    LSE = log Σ_i exp(LSE_i), O = Σ_i exp(LSE_i − LSE) · O_i (written out)."""
    lses = np.stack([l for _, l in parts])  # [n, rows, heads]
    m = np.max(lses, axis=0)
    w = np.exp(lses - m)
    tot = w.sum(axis=0)
    o = sum(w[i][..., None] * parts[i][0] for i in range(len(parts))) / tot[..., None]
    return o, m + np.log(tot)


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


# ----------------------------------------------------------------------------- the method's
# own path, from a simulated KV pool (pages hold K at the STORED position: span-local for
# prefix/fragment blocks, global for cross blocks — readings R2, R3). These follow the method
# step by step (P:436 fn prepare, P:603 store, P:610 ReRoPE on reuse, P:672 span mask) and are
# pinned to the plain definition above by tests/test_oracle_attention.py.
def segment_tokens(seg, queries) -> np.ndarray:
    prefix, frags, cross = queries[seg.query]
    return np.asarray(prefix if seg.kind == 0 else frags[seg.frag_idx] if seg.kind == 1 else cross,
                      np.int64)


def pool_write(pool: dict, view, queries, ek, ev, base: float, bs: int) -> dict:
    """K1 (fused RoPE + paged write) of a plan, on a pool modelled as {slot: (k [Hkv,d],
    v [Hkv,d])}: every packed row with slot >= 0 stores RoPE(k, stored position) and v. Rows with
    slot −1 (resident blocks, R10) are not written. Returns the pool (updated in place)."""
    for seg_of_row, pos, slot in ((view.prefill_seg, view.prefill_pos, view.prefill_slot),
                                  (view.join_seg, view.join_pos, view.join_slot)):
        for si in np.unique(seg_of_row):
            seg = view.segments[int(si)]
            toks = segment_tokens(seg, queries)
            rows = np.nonzero(seg_of_row == si)[0]
            t_idx = np.arange(seg.tok_len - len(rows), seg.tok_len)  # rows are the segment's tail
            for r, t in zip(rows, t_idx):
                if slot[r] >= 0:
                    k, v = expected_pages(toks[[t]], None, ek, ev, base, [pos[r]])
                    pool[int(slot[r])] = (k[0], v[0])
    return pool


def _pages(pool: dict, seg, bs: int):
    ks, vs = [], []
    for t in range(seg.tok_len):
        k, v = pool[seg.blocks[t // bs] * bs + t % bs]
        ks.append(k)
        vs.append(v)
    return np.stack(ks), np.stack(vs)


def prefill_from_pool(view, queries, pool: dict, eq, base: float, bs: int,
                      heads: Optional[Sequence[int]] = None):
    """K2: each prefill job's computed rows [compute_begin, tok_len) attend causally over the
    job's own pages (a fragment "only attends to prior tokens in that same document"),
    q rotated at the same span-local position as its keys. Rows in plan (job) order."""
    outs, lses = [], []
    for si in view.jobs:
        seg = view.segments[si]
        toks = segment_tokens(seg, queries)
        k, v = _pages(pool, seg, bs)
        rows = np.arange(seg.compute_begin, seg.tok_len)
        q = rope(_f64(eq[toks[rows]]), rows[:, None].astype(np.float64), base)
        mask = np.arange(seg.tok_len)[None, :] <= rows[:, None]
        o, l = attend(q, k, v, mask, heads)
        outs.append(o)
        lses.append(l)
    return np.concatenate(outs), np.concatenate(lses)


def join_from_pool(view, queries, pool: dict, eq, base: float, bs: int, query: int,
                   heads: Optional[Sequence[int]] = None):
    """K3: the cross rows of `query` (global positions p_i) attend over every segment's pages
    in query order. Cached fragment K sits at span-local positions 0..L−1, so instead of
    re-encoding it at Δ_f ("ReRoPE") the query row is counter-rotated: RoPE(q, p_i − Δ_f)
    · RoPE(k, t) = RoPE(q, p_i) · RoPE(k, Δ_f + t) (relative property). Prefix pages are at their
    global positions (Δ = 0); cross pages too, causal by stored position."""
    segs = [s for s in view.segments if s.query == query]
    cross = [s for s in segs if s.kind == 2][0]
    ctoks = segment_tokens(cross, queries)
    p = cross.pos0 + np.arange(cross.tok_len)
    scores_q, ks, vs, masks = [], [], [], []
    for seg in segs:
        k, v = _pages(pool, seg, bs)
        delta = seg.pos0 if seg.kind == 1 else 0
        stored = np.arange(seg.tok_len) + (seg.pos0 if seg.kind == 2 else 0)
        q = rope(_f64(eq[ctoks]), (p - delta)[:, None].astype(np.float64), base)
        scores_q.append(q)
        ks.append(k)
        vs.append(v)
        masks.append(stored[None, :] + delta <= p[:, None])
    # one softmax over the concatenated key sets; each set scored with its own rotated q
    R, hq, d = scores_q[0].shape
    g = hq // ks[0].shape[1]
    heads = list(range(hq)) if heads is None else list(heads)
    out = np.zeros((R, len(heads), d))
    lse = np.zeros((R, len(heads)))
    for j, h in enumerate(heads):
        s = np.concatenate([(qq[:, h, :] @ kk[:, h // g, :].T) / np.sqrt(d)
                            for qq, kk in zip(scores_q, ks)], axis=1)
        s = np.where(np.concatenate(masks, axis=1), s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        pr = np.exp(s - m)
        l = pr.sum(axis=1, keepdims=True)
        out[:, j, :] = (pr @ np.concatenate([vv[:, h // g, :] for vv in vs])) / l
        lse[:, j] = (m + np.log(l))[:, 0]
    return out, lse
