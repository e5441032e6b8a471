"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no RoPE, no hashing, no planning, no
attention). It only draws token ids, span-query trees and per-layer q/k/v tables, with the
shapes and structure of the paper's workloads:

* token ids uniform over ``vocab`` from ``numpy.random.Generator(PCG64(seed))`` — the paper's
  RAG microbenchmark uses "randomly generated content" (§5.6, P:669 / line 530 of the
  LaTeX body);
* a token's pre-RoPE q/k/v for layer ``l`` is row ``token`` of tables E_q[V,Hq,d], E_k[V,Hkv,d],
  E_v[V,Hkv,d] drawn N(0,1) with seed ``1000*k + l`` and rounded to bf16 (or kept fp32), so
  identical content gives identical KV and cache hits are exact (stand-in for the QKV
  projections of a real model);
* the tree shapes are the RAG form G[⋈[S, ⊕[F…], U]] and the judge form ⋈[prefix, ⊕[c…],
  suffix] (SURVEY §8(b) accepted tree).

Both ``oracle/`` and the product binding import this module; it imports neither.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

# Node op codes of the ABI tree (include/spanq.h: spq_op).
OP_TOKENS = 0
OP_PLUS = 1
OP_CROSS = 2


@dataclass(frozen=True)
class Shape:
    """Model/cache shape of one configuration (SURVEY §8 notation)."""

    hq: int
    hkv: int
    d: int
    layers: int = 1
    block_size: int = 64
    rope_base: float = 10000.0
    model_salt: int = 0
    dtype: str = "bf16"  # "bf16" or "fp32"
    vocab: int = 8192


@dataclass
class SpanQuery:
    """⋈[prefix, ⊕[fragments…], cross] — prefix may be empty, cross is never empty."""

    prefix: np.ndarray
    fragments: List[np.ndarray]
    cross: np.ndarray
    # optional alternative tree encoding for the same flat content (tests of flattening):
    # list of groups; each group is a list of fragment indices joined by ⋈ into one fragment,
    # groups nested under extra ⊕ when nest=True.
    nest: bool = False

    @property
    def n_tokens(self) -> int:
        return len(self.prefix) + sum(len(f) for f in self.fragments) + len(self.cross)


@dataclass
class Workload:
    name: str
    shape: Shape
    queries: List[SpanQuery]
    seed: int
    # queries planned earlier on the same store (e.g. C3 warms the cache with C2's query)
    warmup_queries: List[SpanQuery] = field(default_factory=list)
    peaky: float = 1.0


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def tokens(g: np.random.Generator, n: int, vocab: int) -> np.ndarray:
    return g.integers(0, vocab, size=n, dtype=np.int64).astype(np.int32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32 holding bf16."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (b.astype(np.uint32) << 16).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 array holding bf16 values -> uint16 bit patterns."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def layer_tables(shape: Shape, layer: int, cfg_seed: int, peaky: float = 1.0):
    """E_q [V,Hq,d], E_k [V,Hkv,d], E_v [V,Hkv,d] as float32 (bf16-exact if dtype=='bf16')."""
    g = rng(1000 * cfg_seed + layer)
    V = shape.vocab
    eq = g.standard_normal((V, shape.hq, shape.d), dtype=np.float32) * np.float32(peaky)
    ek = g.standard_normal((V, shape.hkv, shape.d), dtype=np.float32)
    ev = g.standard_normal((V, shape.hkv, shape.d), dtype=np.float32)
    if shape.dtype == "bf16":
        eq, ek, ev = round_to_bf16(eq), round_to_bf16(ek), round_to_bf16(ev)
    return eq, ek, ev


# ----------------------------------------------------------------------------- trees
def query_to_tree(q: SpanQuery):
    """Encode a SpanQuery as the ABI pre-order node list + token array.

    Returns (nodes int64 [n,4] = (op, num_children, tok_begin, tok_len), tokens int32).
    With ``q.nest`` the fragments are split over a nested ⊕ and the last fragment is written
    as a ⋈ of two TOKENS leaves (both are flattened by the planner).
    """
    toks: List[np.ndarray] = []
    off = 0

    def leaf(arr):
        nonlocal off
        toks.append(np.asarray(arr, dtype=np.int32))
        node = (OP_TOKENS, 0, off, len(arr))
        off += len(arr)
        return node

    nodes = []
    children = (1 if len(q.prefix) else 0) + (1 if q.fragments else 0) + 1
    nodes.append((OP_CROSS, children, 0, 0))
    if len(q.prefix):
        nodes.append(leaf(q.prefix))
    if q.fragments:
        frs = list(q.fragments)
        if q.nest and len(frs) >= 3:
            head, mid, last = frs[0], frs[1:-1], frs[-1]
            nodes.append((OP_PLUS, 3, 0, 0))
            nodes.append(leaf(head))
            nodes.append((OP_PLUS, len(mid), 0, 0))
            for f in mid:
                nodes.append(leaf(f))
            if len(last) >= 2:
                h = len(last) // 2
                nodes.append((OP_CROSS, 2, 0, 0))
                nodes.append(leaf(last[:h]))
                nodes.append(leaf(last[h:]))
            else:
                nodes.append(leaf(last))
        else:
            nodes.append((OP_PLUS, len(frs), 0, 0))
            for f in frs:
                nodes.append(leaf(f))
    nodes.append(leaf(q.cross))
    tok = np.concatenate(toks) if toks else np.zeros(0, np.int32)
    return np.asarray(nodes, dtype=np.int64).reshape(-1, 4), tok


# ----------------------------------------------------------------------------- configs
SHAPE_8B = dict(hq=32, hkv=8, d=128)
SHAPE_2B = dict(hq=32, hkv=8, d=64)


def make_rag(seed: int, shape: Shape, n_prefix: int, n_frag: int, frag_len, n_cross: int,
             name: str = "rag") -> Workload:
    g = rng(seed)
    prefix = tokens(g, n_prefix, shape.vocab)
    lens = [frag_len] * n_frag if np.isscalar(frag_len) else list(frag_len)
    frags = [tokens(g, L, shape.vocab) for L in lens]
    cross = tokens(g, n_cross, shape.vocab)
    return Workload(name, shape, [SpanQuery(prefix, frags, cross)], seed)


def c1(seed: int = 1, variant: str = "base") -> Workload:
    """C1: tiny plus-span, fp32 (BASELINE.json configs[0])."""
    shape = Shape(hq=2, hkv=2, d=64, block_size=16, dtype="fp32", vocab=1024)
    n_prefix = 0
    if variant == "gqa":
        shape = Shape(hq=4, hkv=2, d=64, block_size=16, dtype="fp32", vocab=1024)
    if variant == "prefix":
        n_prefix = 16
    if variant == "bs2":
        shape = Shape(hq=2, hkv=2, d=64, block_size=2, dtype="fp32", vocab=1024)
    w = make_rag(seed, shape, n_prefix, 4, 64, 32, name=f"C1-{variant}")
    if variant == "permuted":
        g = rng(seed + 7)
        q = w.queries[0]
        perm = g.permutation(len(q.fragments))
        w.queries[0] = SpanQuery(q.prefix, [q.fragments[i] for i in perm], q.cross)
    return w


def c2(seed: int = 2, block_size: int = 64, scale: float = 1.0, dtype: str = "bf16") -> Workload:
    """C2: RAG 8B shape, P 512 + 16 x 1024 fragments + 256 cross, cold (configs[1])."""
    shape = Shape(**SHAPE_8B, block_size=block_size, dtype=dtype)
    s = lambda n: max(1, int(round(n * scale)))
    return make_rag(seed, shape, s(512), 16 if scale >= 1 else max(2, int(16 * scale)),
                    s(1024), s(256), name="C2")


def c3(seed: int = 3, hit_frac: float = 0.75, block_size: int = 64, scale: float = 1.0) -> Workload:
    """C3: after a C2-like query, same prefix, a fraction of its fragments + new ones,
    randomly permuted, new cross (configs[2]). warmup_queries holds the C2-like query."""
    base = c2(seed=seed, block_size=block_size, scale=scale)
    q0 = base.queries[0]
    g = rng(seed + 1)
    n = len(q0.fragments)
    n_keep = int(round(hit_frac * n))
    keep = list(g.choice(n, size=n_keep, replace=False))
    new = [tokens(g, len(q0.fragments[0]), base.shape.vocab) for _ in range(n - n_keep)]
    frs = [q0.fragments[i] for i in keep] + new
    perm = g.permutation(len(frs))
    frs = [frs[i] for i in perm]
    cross = tokens(g, len(q0.cross), base.shape.vocab)
    return Workload("C3", base.shape, [SpanQuery(q0.prefix, frs, cross)], seed,
                    warmup_queries=[q0])


def c4(seed: int = 4, scale: float = 1.0, block_size: int = 64) -> Workload:
    """C4: judge/generator, 2B shape, 8 candidates x 2048 + 512 judge prompt (configs[3])."""
    shape = Shape(**SHAPE_2B, block_size=block_size)
    s = lambda n: max(1, int(round(n * scale)))
    return make_rag(seed, shape, 0, 8 if scale >= 1 else max(2, int(8 * scale)), s(2048),
                    s(512), name="C4")


def c5(seed: int = 5, n_queries: int = 256, n_frag: int = 64, frag_len: int = 2048,
       pool: int = 512, shared_per_query: int = 32, n_prefix: int = 512, n_cross: int = 256,
       block_size: int = 64) -> Workload:
    """C5: batch of span queries with cross-query fragment overlap (configs[4])."""
    shape = Shape(**SHAPE_8B, block_size=block_size)
    g = rng(seed)
    prefix = tokens(g, n_prefix, shape.vocab)
    pool_frags = [tokens(g, frag_len, shape.vocab) for _ in range(pool)]
    qs = []
    for _ in range(n_queries):
        shared = [pool_frags[i] for i in g.choice(pool, size=shared_per_query, replace=False)]
        private = [tokens(g, frag_len, shape.vocab) for _ in range(n_frag - shared_per_query)]
        frs = shared + private
        perm = g.permutation(len(frs))
        qs.append(SpanQuery(prefix, [frs[i] for i in perm], tokens(g, n_cross, shape.vocab)))
    return Workload("C5", shape, qs, seed)


def random_queries(seed: int, n_queries: int, vocab: int = 64, max_frag: int = 6,
                   max_len: int = 40, max_prefix: int = 40, max_cross: int = 20,
                   reuse_p: float = 0.4) -> List[SpanQuery]:
    """Random small trees with repeated / permuted fragments (planner differential tests)."""
    g = rng(seed)
    pool: List[np.ndarray] = []
    prefixes: List[np.ndarray] = [tokens(g, int(g.integers(0, max_prefix + 1)), vocab)]
    qs = []
    for _ in range(n_queries):
        if g.random() < 0.5:
            prefix = prefixes[int(g.integers(0, len(prefixes)))]
        else:
            prefix = tokens(g, int(g.integers(0, max_prefix + 1)), vocab)
            prefixes.append(prefix)
        frs = []
        for _ in range(int(g.integers(0, max_frag + 1))):
            if pool and g.random() < reuse_p:
                frs.append(pool[int(g.integers(0, len(pool)))])
            else:
                f = tokens(g, int(g.integers(1, max_len + 1)), vocab)
                pool.append(f)
                frs.append(f)
        cross = tokens(g, int(g.integers(1, max_cross + 1)), vocab)
        qs.append(SpanQuery(prefix, frs, cross, nest=bool(g.random() < 0.3)))
    return qs


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}
