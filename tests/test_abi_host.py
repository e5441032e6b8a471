"""C-ABI library: loads, exports every symbol of include/spanq.h, and its host-side planner /
content-hash store is bit-exact against the oracle's independent mirror (hashes, block tables,
slot maps, jobs, pad slots, stats, eviction, ENOMEM rollback). CPU only (host-only ctx)."""
import os
import re

import numpy as np
import pytest

from oracle import hashing
from oracle.store import OracleENOMEM, Store
from oracle.tree import normalize
from paper_2511_02749_b200 import inputs, spanq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "spanq.h")).read()
    declared = set(re.findall(r"\b(spq_[a-z_]+)\s*\(", hdr))
    declared -= {"spq_status"}
    L = spanq.lib()
    for name in sorted(declared):
        assert hasattr(L, name), f"{name} missing from libspanq.so"
    assert declared == set(spanq.SIGNATURES), declared ^ set(spanq.SIGNATURES)
    assert b"sm_100a" in L.spq_version()


def test_no_gpu_calls_fail_loudly_on_host_only_ctx():
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16, dtype="fp32"), 64, device=-1)
    p = ctx.plan([inputs.c1().queries[0]])
    with pytest.raises(spanq.SpanqError) as e:
        p.prefill(0, None, None, None, None)
    assert e.value.status == spanq.ESTATE
    for phase, status in [(0, spanq.ESTATE), (1, spanq.ESTATE), (2, spanq.EINVAL), (-1, spanq.EINVAL)]:
        with pytest.raises(spanq.SpanqError) as e:
            p.join_phase(0, phase, None, None, None, None)
        assert e.value.status == status
    p.release()


def test_released_plan_handle_reports_estate():
    # spq_plan_release keeps the emptied handle reserved: later calls return SPQ_ESTATE instead
    # of touching freed memory (spanq.h), and the store has no pins left
    import ctypes as C

    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16, dtype="fp32"), 64, device=-1)
    p = ctx.plan([inputs.c1().queries[0]])
    assert ctx.stats()["pinned_blocks"] > 0
    h = p.handle
    p.release()
    assert ctx.stats()["pinned_blocks"] == 0
    L = spanq.lib()
    assert L.spq_plan_view_get(h, C.byref(spanq.spq_plan_view())) == spanq.ESTATE
    assert L.spq_plan_release(ctx.handle, h, None) == spanq.ESTATE
    assert L.spq_join_phase(ctx.handle, h, 0, 1, None, None, None, None, None, None) == spanq.ESTATE
    assert b"after release" in L.spq_last_error()
    # many plans later (inside the 1024-release window) the first handle is still reported
    for _ in range(50):
        ctx.plan([inputs.c1().queries[0]]).release()
    assert L.spq_plan_release(ctx.handle, h, None) == spanq.ESTATE


def test_options_validate():
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16), 64, device=-1)
    for key, value in [(spanq.OPT_EXP2, 0), (spanq.OPT_EXP2, 1), (spanq.OPT_EXP2, 2), (spanq.OPT_EXP2, 3),
                       (spanq.OPT_EXP2, 4), (spanq.OPT_RESCALE_THRESHOLD, 0), (spanq.OPT_RESCALE_THRESHOLD, 8),
                       (spanq.OPT_PDL, 0), (spanq.OPT_PDL, 1), (spanq.OPT_PAIR, 0), (spanq.OPT_PAIR, 1)]:
        ctx.set_option(key, value)
    for key, value in [(spanq.OPT_EXP2, 5), (spanq.OPT_EXP2, -1), (spanq.OPT_RESCALE_THRESHOLD, -1), (99, 0)]:
        with pytest.raises(spanq.SpanqError) as e:
            ctx.set_option(key, value)
        assert e.value.status == spanq.EINVAL
    # the product library has no tracing (only the profiling build, tools/)
    with pytest.raises(spanq.SpanqError) as e:
        ctx.set_trace(None, 1)
    assert e.value.status == spanq.EINVAL


def oracle_arrays(view):
    segs = view.segments
    return dict(
        seg_query=np.array([s.query for s in segs], np.int32),
        seg_kind=np.array([s.kind for s in segs], np.int32),
        seg_frag_idx=np.array([s.frag_idx for s in segs], np.int32),
        seg_tok_len=np.array([s.tok_len for s in segs], np.int32),
        seg_pos0=np.array([s.pos0 for s in segs], np.int32),
        seg_hit=np.array([s.hit for s in segs], np.int32),
        seg_compute_begin=np.array([s.compute_begin for s in segs], np.int32),
        blocks=np.array([b for s in segs for b in s.blocks], np.int32),
        block_write=np.array([w for s in segs for w in s.write], np.uint8),
        digests=np.frombuffer(b"".join(d for s in segs for d in s.digests), np.uint8).reshape(-1, 16),
        join_digests=np.frombuffer(b"".join(view.join_digests), np.uint8).reshape(-1, 16),
        jobs=np.array(view.jobs, np.int32),
        prefill_pos=view.prefill_pos, prefill_slot=view.prefill_slot,
        join_pos=view.join_pos, join_slot=view.join_slot, pad_slots=view.pad_slots,
    )


STAT_KEYS = ["lookups", "hit_blocks", "miss_blocks", "hit_tokens", "input_tokens", "evictions",
             "inserted_blocks"]


def assert_same(cv, ov):
    oa = oracle_arrays(ov)
    for k, v in oa.items():
        np.testing.assert_array_equal(cv[k], v, err_msg=k)


def flat(q):
    return (q.prefix, q.fragments, q.cross)


@pytest.mark.parametrize("seed,bs,nblk", [(1, 4, 4096), (2, 2, 90), (3, 8, 40), (4, 16, 25), (5, 3, 60)])
def test_planner_bit_exact_vs_oracle_random(seed, bs, nblk):
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=bs, dtype="fp32", rope_base=5000.0, model_salt=seed)
    ctx = spanq.Context(shape, nblk, device=-1)
    ost = Store(nblk, 4, 2, 64, bs, 5000.0, seed)
    qs = inputs.random_queries(seed, 60, vocab=12, max_len=30)
    g = np.random.default_rng(seed)
    live = []
    i = 0
    n_plans = n_enomem = 0
    while i < len(qs):
        k = int(g.integers(1, 5))
        batch = qs[i:i + k]
        i += k
        try:
            ov = ost.plan([flat(q) for q in batch])
        except OracleENOMEM:
            ov = None
        if ov is None:
            with pytest.raises(spanq.SpanqError) as e:
                ctx.plan(batch)
            assert e.value.status == spanq.ENOMEM
            n_enomem += 1
        else:
            cp = ctx.plan(batch)
            assert_same(cp.view(), ov)
            live.append((cp, ov))
            n_plans += 1
        cs = ctx.stats()
        for key in STAT_KEYS:
            assert cs[key] == ost.stats[key], key
        assert cs["resident_blocks"] == len(ost.index)
        assert cs["free_blocks"] == len(ost.free)
        # release some live plans (out of order) to exercise pins / LRU
        while live and g.random() < 0.6:
            j = int(g.integers(0, len(live)))
            cp, ov = live.pop(j)
            cp.release()
            ost.release(ov)
        if g.random() < 0.05:
            ctx.evict_all()
            ost.evict_all()
    assert n_plans > 5


def test_block_hashes_lookup_insert_vs_oracle():
    shape = inputs.Shape(hq=32, hkv=8, d=128, block_size=4)
    ctx = spanq.Context(shape, 64, device=-1)
    ost = Store(64, 32, 8, 128, 4)
    q = inputs.SpanQuery(np.arange(10, dtype=np.int32), [np.arange(5, dtype=np.int32) + 100,
                                                         np.arange(9, dtype=np.int32) + 200],
                         np.arange(6, dtype=np.int32) + 300, nest=False)
    d = ctx.block_hashes(q)
    h = hashing.prefix_chain(q.prefix, 4, ost.root)
    s = [hashing.fragment_chain(f, 4, ost.root) for f in q.fragments]
    J = hashing.join_fold(h[-1], [x[-1] for x in s])
    x = hashing.cross_chain(q.cross, 4, J)
    exp = h + s[0] + s[1] + [J] + x
    assert [bytes(r) for r in d] == exp
    # insert / lookup
    ids = ctx.insert(d[:5], [4, 4, 2, 4, 1])
    oids = ost.insert(exp[:5], [4, 4, 2, 4, 1])
    assert ids.tolist() == oids
    assert ctx.lookup(d).tolist() == ost.lookup(exp)
    # inserting more unpinned blocks than capacity evicts LRU blocks (same victims)
    many = np.random.default_rng(0).integers(0, 256, (80, 16), dtype=np.uint8)
    assert ctx.insert(many, [2] * 80).tolist() == ost.insert([bytes(r) for r in many], [2] * 80)
    assert ctx.lookup(d).tolist() == ost.lookup(exp)
    # with every block pinned by a live plan, insert fails with ENOMEM and rolls back
    ctx2 = spanq.Context(shape, 3, device=-1)
    ost2 = Store(3, 32, 8, 128, 4)
    small = inputs.SpanQuery(np.zeros(0, np.int32), [np.arange(8, dtype=np.int32)], np.arange(3, dtype=np.int32))
    cp = ctx2.plan([small])
    ov = ost2.plan([flat(small)])
    with pytest.raises(spanq.SpanqError) as e:
        ctx2.insert(many[:2], [1, 1])
    assert e.value.status == spanq.ENOMEM
    with pytest.raises(OracleENOMEM):
        ost2.insert([bytes(r) for r in many[:2]], [1, 1])
    assert ctx2.stats()["inserted_blocks"] == ost2.stats["inserted_blocks"]
    assert ctx.stats()["evictions"] == ost.stats["evictions"]


def test_invalid_trees_einval():
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16), 64, device=-1)
    bad = [
        (np.array([(2, 1, 0, 0), (1, 0, 0, 0)]), np.array([1], np.int32)),
        (np.array([(2, 1, 0, 0), (0, 0, 0, 0)]), np.array([1], np.int32)),
        (np.array([(5, 0, 0, 1)]), np.array([1], np.int32)),
        (np.array([(2, 2, 0, 0), (0, 0, 0, 1)]), np.array([1], np.int32)),
        (np.array([(2, 1, 0, 0), (0, 0, 0, 1)]), np.array([-3], np.int32)),
        (np.array([(2, 1, 0, 0), (0, 0, 0, 5)]), np.array([1, 2], np.int32)),
    ]
    for nodes, toks in bad:
        with pytest.raises(spanq.SpanqError) as e:
            ctx.plan([(nodes, toks)])
        assert e.value.status == spanq.EINVAL
    assert ctx.stats()["plans"] == 0


def test_nested_tree_flattening_matches_oracle():
    qs = inputs.random_queries(77, 30, vocab=20)
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=4), 4096, device=-1)
    ost = Store(4096, 2, 1, 64, 4)
    for q in qs:
        nodes, toks = inputs.query_to_tree(q)
        p, f, c = normalize(nodes, toks)
        ov = ost.plan([(p, f, c)])
        cp = ctx.plan([(nodes, toks)])
        assert_same(cp.view(), ov)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_paper_configs_plan_bit_exact(cfg):
    w = inputs.CONFIGS[cfg]()
    s = w.shape
    nblk = 4096
    ctx = spanq.Context(s, nblk, device=-1)
    ost = Store(nblk, s.hq, s.hkv, s.d, s.block_size, s.rope_base, s.model_salt)
    for q in w.warmup_queries:
        ctx.plan([q]).release()
        ost.release(ost.plan([flat(q)]))
    cp = ctx.plan(w.queries)
    ov = ost.plan([flat(q) for q in w.queries])
    assert_same(cp.view(), ov)
    if cfg == "C3":
        frag_hits = [h for h, k in zip(cp.view()["seg_hit"], cp.view()["seg_kind"]) if k == 1]
        assert sum(frag_hits) == 12  # 75% fragment hits (configs[2])


@pytest.mark.parametrize("scalar", [False, True])
def test_block_hashes_both_blake2b_paths(scalar):
    # the library uses an AVX2 BLAKE2b compression when the CPU has it; the scalar RFC 7693 path
    # (SPQ_OPT_HASH_SCALAR, process-wide — set before the ctx computes its root digest) must give
    # the same digests
    sh = inputs.Shape(hq=32, hkv=8, d=128, block_size=64)
    spanq.Context(sh, 64, device=-1).set_option(spanq.OPT_HASH_SCALAR, 1 if scalar else 0)
    try:
        ctx = spanq.Context(sh, 64, device=-1)
        q = inputs.SpanQuery(np.arange(300, dtype=np.int32), [np.arange(200, dtype=np.int32) * 7],
                             np.arange(70, dtype=np.int32) + 5, nest=False)
        d = [bytes(r) for r in ctx.block_hashes(q)]
        root = Store(64, 32, 8, 128, 64).root
        h = hashing.prefix_chain(q.prefix, 64, root)
        s = hashing.fragment_chain(q.fragments[0], 64, root)
        J = hashing.join_fold(h[-1], [s[-1]])
        assert d == h + s + [J] + hashing.cross_chain(q.cross, 64, J)
    finally:
        spanq.Context(sh, 64, device=-1).set_option(spanq.OPT_HASH_SCALAR, 0)


@pytest.mark.parametrize("crop", [False, True])
def test_commit_span_plus_distribution(crop):
    # plus distribution: an inner generate ⋈[input] whose input and generated tokens
    # are committed as a span is found by a later query that uses (input ‖ output) as a ⊕
    # fragment — the F-chain digests of those tokens (oracle hashing) point at the inner plan's
    # own blocks, which survive its release as cached blocks. crop drops the trailing partial
    # block: the committed fragment is the full blocks only.
    bs = 16
    sh = inputs.Shape(hq=2, hkv=1, d=64, block_size=bs)
    ctx = spanq.Context(sh, 256, device=-1)
    g = np.random.default_rng(9)
    inp, gen = g.integers(0, 500, 40).astype(np.int32), g.integers(0, 500, 30).astype(np.int32)
    inner = inputs.SpanQuery(np.zeros(0, np.int32), [], inp)
    p = ctx.plan([inner])
    v = p.view()
    cross_blocks = list(v["blocks"])
    p.decode_reserve(32)
    n = p.commit_span(0, gen, crop=crop)
    span = np.concatenate([inp, gen])
    assert n == (len(span) // bs * bs if crop else len(span))
    root = Store(16, 2, 1, 64, bs).root
    dig = hashing.fragment_chain(span[:n], bs, root)
    ids = ctx.lookup(np.frombuffer(b"".join(dig), np.uint8))
    assert (ids >= 0).all() and len(set(ids.tolist())) == len(ids)
    assert ids[:len(cross_blocks)].tolist() == cross_blocks  # the input's own blocks, in order
    p.release()
    assert (ctx.lookup(np.frombuffer(b"".join(dig), np.uint8)) == ids).all()  # cached, not freed
    outer = inputs.SpanQuery(g.integers(0, 500, 8).astype(np.int32), [span[:n]], g.integers(0, 500, 5).astype(np.int32))
    ov = ctx.plan([outer]).view()
    frag = [i for i, k in enumerate(ov["seg_kind"]) if k == 1][0]
    assert ov["seg_hit"][frag] == 1 and ov["n_jobs"] == 1  # only the outer prefix is prefilled
    if crop:  # the uncropped span misses (its trailing partial block was never committed)
        o2 = ctx.plan([inputs.SpanQuery(outer.prefix, [span], outer.cross)]).view()
        assert o2["seg_hit"][[i for i, k in enumerate(o2["seg_kind"]) if k == 1][0]] == 0


def test_decode_reserve_and_commit_errors():
    ctx = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16), 64, device=-1)
    q = inputs.c1().queries[0]  # has fragments: its cross is not at span-local positions
    p = ctx.plan([inputs.SpanQuery(q.prefix, q.fragments, q.cross)])
    with pytest.raises(spanq.SpanqError) as e:
        p.decode_reserve(0)
    assert e.value.status == spanq.EINVAL
    p.decode_reserve(4)
    with pytest.raises(spanq.SpanqError) as e:
        p.decode_reserve(4)
    assert e.value.status == spanq.ESTATE
    with pytest.raises(spanq.SpanqError) as e:
        p.commit_span(0, [1, 2])
    assert e.value.status == spanq.EINVAL
    with pytest.raises(spanq.SpanqError) as e:
        p.decode_step(0, 0, None, None, None, None)
    assert e.value.status == spanq.ESTATE  # host-only ctx
    with pytest.raises(spanq.SpanqError) as e:  # more than reserved
        ctx.plan([inputs.SpanQuery(np.zeros(0, np.int32), [], q.cross)]).commit_span(0, [1] * 9)
    assert e.value.status == spanq.ESTATE


def test_flat_query_encoding_equals_the_generic_tree():
    """spanq._FlatQueryBuf (the binding's fast path for ⋈[prefix?, ⊕[…]?, cross]) encodes exactly
    the nodes and tokens inputs.query_to_tree + _QueryBuf produce."""
    n_checked = 0
    for seed in range(40):
        for q in inputs.random_queries(seed, 6, vocab=50, max_len=20):
            if q.nest and len(q.fragments) >= 3:
                continue
            a = spanq._FlatQueryBuf(q)
            b = spanq._QueryBuf(*inputs.query_to_tree(q))
            assert a.q.num_nodes == b.q.num_nodes
            np.testing.assert_array_equal(a.nodes, b.nodes[: len(a.nodes)])
            np.testing.assert_array_equal(a.tokens, b.tokens)
            n_checked += 1
    assert n_checked > 100
