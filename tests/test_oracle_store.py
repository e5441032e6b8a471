"""Pins for oracle/hashing.py, oracle/tree.py and oracle/store.py (the planner mirror).

Pins: the paper's hit-rate worked examples (golden/hit_rates.json), a hand-computed plan
(golden/plan_bs2_tiny.json), the RFC 7693 BLAKE2b-512 vector (pins hashlib), and the
invariants of P:603 / S:329-333 (context independence, permutation invariance, prefix
monotonicity, no partial ordered blocks), lowest-id allocation and LRU eviction order.
"""
import json
import os

import numpy as np
import pytest

from oracle import hashing
from oracle.store import KIND_CROSS, KIND_FRAG, KIND_PREFIX, OracleENOMEM, Store, hit_rate
from oracle.tree import TreeError, normalize
from paper_2511_02749_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_blake2b_rfc7693_vector():
    import hashlib

    # RFC 7693 Appendix A: BLAKE2b-512("abc")
    assert hashlib.blake2b(b"abc").hexdigest().startswith(
        "ba80a53f981c4d0d6a2797b69f12f6e94c212f14685ac4b74b12bb6fdbffa2d1")
    assert hashing.b2(b"abc").hex() == "cf4ab791c62b8d2b2109c90275287816"


def _ids(words, vocab):
    return np.array([vocab.setdefault(w, len(vocab)) for w in words], np.int32)


def test_paper_hit_rate_examples():
    g = load("hit_rates.json")
    V = {}
    sentinel = np.array([9999], np.int32)
    # E1: chat
    st = Store(64, 1, 1, 2, 2)
    st.plan([(_ids(g["E1_chat"]["request1"], V), [], sentinel)])
    before = dict(st.stats)
    st.plan([(_ids(g["E1_chat"]["request2"], V), [], sentinel)])
    assert st.stats["hit_tokens"] - before["hit_tokens"] == g["E1_chat"]["hit_tokens"]
    assert round(100 * 4 / g["E1_chat"]["context_tokens"]) == g["E1_chat"]["rate_percent"]
    # E2: RAG on stock vLLM (no spans): reversed order kills reuse after the system prompt
    st = Store(64, 1, 1, 2, 2)
    st.plan([(_ids(g["E2_rag_stock"]["request1"], V), [], sentinel)])
    before = dict(st.stats)
    st.plan([(_ids(g["E2_rag_stock"]["request2"], V), [], sentinel)])
    hit = st.stats["hit_tokens"] - before["hit_tokens"]
    assert hit == g["E2_rag_stock"]["hit_tokens"]
    assert round(100 * hit / g["E2_rag_stock"]["input_tokens"]) == g["E2_rag_stock"]["rate_percent"]
    # E2 with span queries: both fragments hit in either order
    st = Store(64, 1, 1, 2, 2)
    S, f1, f2 = _ids(["S", "S'"], V), _ids(["f1a", "f1b"], V), _ids(["f2a", "f2b"], V)
    st.plan([(S, [f1, f2], sentinel)])
    before = dict(st.stats)
    st.plan([(S, [f2, f1], sentinel)])
    assert st.stats["hit_tokens"] - before["hit_tokens"] == 6
    # E3: nested generation on stock vLLM
    st = Store(64, 1, 1, 2, 2)
    for r in g["E3_nested_stock"]["earlier"]:
        st.plan([(_ids(r, V), [], sentinel)])
    before = dict(st.stats)
    st.plan([(_ids(g["E3_nested_stock"]["request3"], V), [], sentinel)])
    hit = st.stats["hit_tokens"] - before["hit_tokens"]
    assert hit == g["E3_nested_stock"]["hit_tokens"]
    assert round(100 * hit / 7) == g["E3_nested_stock"]["rate_percent"]


def _check_plan(view, exp, stats_delta):
    assert len(view.segments) == len(exp["segments"])
    for s, e in zip(view.segments, exp["segments"]):
        assert s.kind == e["kind"]
        assert s.blocks == e["blocks"]
        assert s.hit == e["hit"]
        assert s.compute_begin == e["compute_begin"]
        assert s.write == e["write"]
        if "pos0" in e:
            assert s.pos0 == e["pos0"]
    assert view.prefill_pos.tolist() == exp["prefill_pos"]
    assert view.prefill_slot.tolist() == exp["prefill_slot"]
    assert view.join_pos.tolist() == exp["join_pos"]
    assert view.join_slot.tolist() == exp["join_slot"]
    assert sorted(view.pad_slots.tolist()) == exp["pad_slots"]
    assert stats_delta["hit_tokens"] == exp["hit_tokens"]
    assert stats_delta["input_tokens"] == exp["input_tokens"]


def test_hand_computed_plan_bs2():
    g = load("plan_bs2_tiny.json")
    q = g["query"]
    query = (np.array(q["prefix"]), [np.array(f) for f in q["fragments"]], np.array(q["cross"]))
    st = Store(g["num_blocks"], 1, 1, 2, g["block_size"])
    s0 = dict(st.stats)
    v1 = st.plan([query])
    _check_plan(v1, g["plan1"], {k: st.stats[k] - s0[k] for k in s0})
    st.release(v1)
    s1 = dict(st.stats)
    v2 = st.plan([query])
    _check_plan(v2, g["plan2"], {k: st.stats[k] - s1[k] for k in s1})


def test_context_independence_and_permutation():
    root = hashing.root_digest(32, 8, 128, 4, 1e4, 0)
    g = np.random.default_rng(0)
    f = g.integers(0, 100, 10)
    a = hashing.fragment_chain(f, 4, root)
    assert a == hashing.fragment_chain(f.copy(), 4, root)
    # the fragment's digests do not depend on what precedes it (suspension)
    st = Store(128, 32, 8, 128, 4)
    v1 = st.plan([(g.integers(0, 100, 9), [f], np.array([1]))])
    v2 = st.plan([(g.integers(0, 100, 5), [g.integers(0, 100, 7), f], np.array([1]))])
    d1 = [s.digests for s in v1.segments if s.kind == KIND_FRAG][0]
    d2 = [s.digests for s in v2.segments if s.kind == KIND_FRAG][1]
    assert d1 == d2 == a
    assert [s.hit for s in v2.segments if s.kind == KIND_FRAG] == [0, 1]
    # prefix chain: changing an early block changes every later digest
    p = g.integers(0, 100, 12)
    p2 = p.copy()
    p2[1] += 1
    h1, h2 = hashing.prefix_chain(p, 4, root), hashing.prefix_chain(p2, 4, root)
    assert all(x != y for x, y in zip(h1, h2))
    # the join fold is order-sensitive (R6) but built only from fragment identities
    s1, s2 = b"a" * 16, b"b" * 16
    assert hashing.join_fold(root, [s1, s2]) != hashing.join_fold(root, [s2, s1])
    # tail length enters the digest
    assert hashing.fragment_chain([5, 6], 4, root) != hashing.fragment_chain([5, 6, 0], 4, root)


def test_prefix_monotonicity_and_no_partial_ordered_blocks():
    g = np.random.default_rng(1)
    for trial in range(30):
        st = Store(256, 2, 2, 4, 4)
        base = g.integers(0, 20, int(g.integers(1, 30)))
        st.plan([(base, [], np.array([1]))])
        q = base.copy()
        if len(q) > 2:
            q[int(g.integers(0, len(q)))] += 100
        v = st.plan([(q, [], np.array([1]))])
        seg = v.segments[0]
        nfull = len(q) // 4
        # hits form a prefix and stop at the first miss
        assert seg.hit <= nfull
        assert seg.compute_begin == min(seg.hit * 4, len(q))
        # partial tails are never inserted into the index
        for dig, ntok in [(m[0], m[1]) for m in st.meta.values()]:
            pass
        for b, (dig, ntok, _) in st.meta.items():
            assert dig in st.index
    # every partial ordered tail block is plan-private (not in meta)
    st = Store(64, 1, 1, 2, 4)
    v = st.plan([(np.arange(6), [], np.arange(5))])
    pre, cr = v.segments[0], v.segments[-1]
    assert pre.blocks[-1] in v.private and cr.blocks[-1] in v.private
    assert pre.blocks[-1] not in st.meta and cr.blocks[-1] not in st.meta


def test_slot_invariants_random():
    qs = inputs.random_queries(11, 40, vocab=30)
    st = Store(4096, 4, 2, 8, 4)
    for i in range(0, 40, 4):
        batch = [(q.prefix, q.fragments, q.cross) for q in qs[i:i + 4]]
        v = st.plan(batch)
        slots = np.concatenate([v.prefill_slot, v.join_slot])
        written = slots[slots >= 0]
        assert len(np.unique(written)) == len(written)  # no slot written twice
        assert not set(written.tolist()) & set(v.pad_slots.tolist())
        for s in v.segments:
            for b, w in zip(s.blocks, s.write):
                if s.kind == KIND_FRAG and s.hit:
                    assert not w  # resident blocks are never rewritten
        st.release(v)


def test_lowest_id_allocation_and_lru_eviction():
    st = Store(6, 1, 1, 2, 2)
    a = (np.zeros(0, np.int32), [np.array([1, 2])], np.array([3, 4]))
    b = (np.zeros(0, np.int32), [np.array([5, 6])], np.array([7, 8]))
    va = st.plan([a])  # plan 1: frag -> 0, cross -> 1
    assert [s.blocks for s in va.segments] == [[0], [1]]
    st.release(va)
    vb = st.plan([b])  # plan 2: 2, 3
    assert [s.blocks for s in vb.segments] == [[2], [3]]
    st.release(vb)
    c = (np.zeros(0, np.int32), [np.array([9, 9])], np.array([9, 8]))
    vc = st.plan([c])  # plan 3: free 4, 5
    assert [s.blocks for s in vc.segments] == [[4], [5]]
    st.release(vc)
    d = (np.zeros(0, np.int32), [np.array([1, 2])], np.array([10, 11]))
    vd = st.plan([d])  # plan 4: fragment [1,2] hits block 0 (last_use -> 4); cross needs a
    # block: no free ids; evict smallest (last_use, id) among unpinned = block 1 (plan 1)
    assert vd.segments[0].hit == 1 and vd.segments[0].blocks == [0]
    assert vd.segments[1].blocks == [1]
    assert st.stats["evictions"] == 1
    st.release(vd)


def test_enomem_rolls_back():
    st = Store(3, 1, 1, 2, 2)
    q = (np.array([1, 2, 3, 4]), [np.array([5, 6])], np.array([7, 8]))  # needs 4 blocks
    before = (dict(st.index), dict(st.meta), set(st.free), list(st.pins), st.plan_no, dict(st.stats))
    with pytest.raises(OracleENOMEM):
        st.plan([q])
    assert (st.index, st.meta, st.free, st.pins, st.plan_no, st.stats) == before
    # pinned blocks are not evictable: a live plan holds all 3 blocks
    st2 = Store(3, 1, 1, 2, 2)
    v = st2.plan([(np.zeros(0, np.int32), [np.array([1, 2])], np.array([3, 4]))])
    with pytest.raises(OracleENOMEM):
        st2.plan([(np.zeros(0, np.int32), [np.array([5, 6])], np.array([7, 8]))])
    st2.release(v)
    st2.plan([(np.zeros(0, np.int32), [np.array([5, 6])], np.array([7, 8]))])


def test_in_plan_dedupe():  # R11
    st = Store(64, 1, 1, 2, 2)
    f = np.array([4, 5, 6])
    v = st.plan([(np.zeros(0, np.int32), [f, np.array([1]), f], np.array([9]))])
    frs = [s for s in v.segments if s.kind == KIND_FRAG]
    assert [s.hit for s in frs] == [0, 0, 1]
    assert frs[0].blocks == frs[2].blocks
    assert frs[2].pos0 == 4  # attended at its own Δ
    assert len([j for j in v.jobs if v.segments[j].kind == KIND_FRAG]) == 2


def test_tree_normalization_and_errors():
    q = inputs.SpanQuery(np.array([1, 2]), [np.array([3]), np.array([4, 5]), np.array([6, 7, 8])],
                         np.array([9]), nest=True)
    nodes, tok = inputs.query_to_tree(q)
    p, frs, c = normalize(nodes, tok)
    assert p.tolist() == [1, 2] and c.tolist() == [9]
    assert [f.tolist() for f in frs] == [[3], [4, 5], [6, 7, 8]]
    bad = [
        [(2, 1, 0, 0), (1, 0, 0, 0)],  # PLUS with no child / last child not TOKENS
        [(2, 1, 0, 0), (0, 0, 0, 0)],  # empty cross
        [(5, 0, 0, 1)],  # bad op
        [(2, 2, 0, 0), (0, 0, 0, 1)],  # arity mismatch
    ]
    for b in bad:
        with pytest.raises(TreeError):
            normalize(np.array(b), np.array([1, 2, 3]))
    with pytest.raises(TreeError):
        normalize(np.array([(2, 1, 0, 0), (0, 0, 0, 1)]), np.array([-1]))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partition_covers_the_single_rank_plan(world):
    # Partitioning (home q mod W, fragment owner u64le(s_last) mod W) must split, not change, the
    # work of the W = 1 plan: with cold stores, (1) every distinct fragment is prefilled on exactly
    # one rank — its owner — with the same rows as in the W = 1 plan, (2) every query's join rows
    # are on exactly its home rank with the same positions, (3) the prefix rows follow their
    # query, and (4) what a rank receives from an owner is exactly what that owner sends it.
    qs = [(q.prefix, q.fragments, q.cross) for q in inputs.random_queries(40 + world, 24, vocab=10, max_len=18,
                                                                          reuse_p=0.5)]
    mk = lambda: Store(1 << 14, 4, 2, 16, 4, 10000.0, 0)
    one = mk().plan(qs)
    parts = [mk().plan(qs, rank=r, world=world) for r in range(world)]

    def frag_rows(v):
        out = {}
        for j in v.jobs:
            s = v.segments[j]
            if s.kind == KIND_FRAG:
                out[s.digests[-1]] = out.get(s.digests[-1], 0) + (s.tok_len - s.compute_begin)
        return out

    base = frag_rows(one)
    seen = {}
    for r, v in enumerate(parts):
        for d, n in frag_rows(v).items():
            assert hashing.owner_rank(d, world) == r
            assert d not in seen
            seen[d] = n
    assert seen == base
    for qi in range(len(qs)):
        home = qi % world
        for r, v in enumerate(parts):
            cross = [s for s in v.segments if s.kind == KIND_CROSS and s.query == qi]
            pref = [s for s in v.segments if s.kind == KIND_PREFIX and s.query == qi]
            assert len(cross) == (1 if r == home else 0)
            assert (len(pref) > 0) == (r == home and len(qs[qi][0]) > 0)
    join_pos = np.concatenate([v.join_pos for v in parts])
    assert sorted(join_pos.tolist()) == sorted(one.join_pos.tolist())
    assert sum(v.n_join_queries for v in parts) == len(qs)
    # exchange lists: counts agree pairwise, and receivers hold blocks for exactly the remote
    # fragments their joins read
    for r in range(world):
        for p in range(world):
            assert len(parts[r].send.get(p, [])) == len(parts[p].recv.get(r, []))
