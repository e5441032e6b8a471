"""k-ary judge reduction schedule and bulk clustering order: the oracle's plain
definitions pinned to the paper's / SPEC's examples, and the library's host implementations
(spq_reduce_tree, spq_bulk_order) bit-exact against them."""
import numpy as np
import pytest

from oracle import reduction
from oracle.store import Store
from paper_2511_02749_b200 import inputs, spanq


def test_paper_and_spec_examples():
    plies, ch = reduction.reduce_tree(8, 2)  # PAPER Fig. 13: "into 3 2-way judge steps"
    assert len(plies) == 3 and len(ch) == 7 and [len(p) for p in plies] == [4, 2, 1]
    assert ch[:4] == [[0, 1], [2, 3], [4, 5], [6, 7]] and ch[4:] == [[8, 9], [10, 11], [12, 13]]
    plies, ch = reduction.reduce_tree(9, 3)  # SPEC: n=9, k=3 -> 2 plies, 4 judge nodes
    assert len(plies) == 2 and len(ch) == 4
    for n in range(1, 5):  # n <= k: the query unchanged — one judge over every candidate
        plies, ch = reduction.reduce_tree(n, 4)
        assert plies == [[0]] and ch == [list(range(n))]


@pytest.mark.parametrize("n,k", [(n, k) for n in range(1, 41) for k in (2, 3, 4, 5)])
def test_reduce_tree_structure_and_library(n, k):
    plies, ch = reduction.reduce_tree(n, k)
    # every item but the root is read exactly once; judges read <= k items, >= 2 unless n == 1
    seen = [x for c in ch for x in c]
    assert sorted(seen) == sorted(set(seen)) and set(seen) == set(range(n + len(ch) - 1))
    assert all(1 <= len(c) <= k for c in ch) and all(len(c) >= 2 for c in ch[:-1] or [[0, 1]])
    # ceil(log_k n) plies (SPEC), at least one
    p, m = 0, 1
    while m < n:
        m *= k
        p += 1
    assert len(plies) == max(1, p)
    assert spanq.reduce_tree(n, k) == (plies, ch)


def test_bulk_order_hand_example():
    # q0 = {a, b}, q1 = {c, d}, q2 = {a, b}, q3 = {c, d}: with a one-query window q0 is followed
    # by q2 (shares a, b), then q1 (no overlap: lowest index) and q3 (shares c, d)
    bs = 4
    root = Store(16, 2, 1, 8, bs).root
    g = np.random.default_rng(3)
    a, b, c, d = (g.integers(0, 100, 8).astype(np.int32) for _ in range(4))
    x = g.integers(0, 100, 3).astype(np.int32)
    qs = [inputs.SpanQuery(np.zeros(0, np.int32), fr, x) for fr in ([a, b], [c, d], [a, b], [c, d])]
    blocks = reduction.query_blocks(qs[0], bs)
    assert reduction.bulk_order(qs, bs, root, blocks) == [0, 2, 1, 3]
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=8, block_size=bs), 16, device=-1)
    assert ctx.bulk_order(qs, blocks).tolist() == [0, 2, 1, 3]
    # no shared units: arrival order
    qs2 = [inputs.SpanQuery(np.zeros(0, np.int32), [g.integers(0, 100, 8).astype(np.int32)], x) for _ in range(5)]
    assert ctx.bulk_order(qs2, 4).tolist() == [0, 1, 2, 3, 4]


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("window", [0, 1, 40, 200])
def test_bulk_order_library_vs_oracle(seed, window):
    sh = inputs.Shape(hq=2, hkv=1, d=8, block_size=8)
    w = inputs.c5(seed=seed, n_queries=24, n_frag=6, frag_len=20, pool=10, shared_per_query=3, n_prefix=12,
                  n_cross=5, block_size=8)
    ctx = spanq.Context(sh, 300, device=-1)
    root = Store(300, sh.hq, sh.hkv, sh.d, sh.block_size, sh.rope_base, sh.model_salt).root
    got = ctx.bulk_order(w.queries, window).tolist()
    assert sorted(got) == list(range(len(w.queries)))
    assert got == reduction.bulk_order(w.queries, sh.block_size, root, window if window > 0 else 300)
