"""Pins for oracle/attention.py.

Each pin is independent of the oracle's own formula: closed forms (Q=0 → mean of visible V,
uniform V → V, mask counts of S:467), library special cases (torch SDPA in fp64 on CPU:
ordinary causal prefill for a one-fragment ⊕, explicit-mask attention for the join) and the
invariants north_star lists (one-fragment ⊕ ≡ causal prefill; permutation leaves per-fragment
KV and rows unchanged).
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle.attention import (dense_masked, expected_pages, join_from_pool, join_rows,
                              plan_join_expected, plan_prefill_expected, pool_write,
                              prefill_from_pool, segment_causal, visible_mask)
from oracle import hashing
from oracle.store import Store
from oracle.rope import rope
from paper_2511_02749_b200 import inputs


def tables(hq=4, hkv=2, d=16, V=64, seed=0, scale=1.0):
    g = np.random.default_rng(seed)
    return (g.standard_normal((V, hq, d)) * scale, g.standard_normal((V, hkv, d)),
            g.standard_normal((V, hkv, d)))


def toks(g, n, V=64):
    return g.integers(0, V, n)


def test_mask_counts_closed_form():
    # 2 docs x 4 tokens + 2-token suffix: 29 strictly-lower attended pairs (45 dense);
    # including the diagonal: 29 + 10 = 39 (55 dense).
    m = visible_mask(0, [4, 4], 2)
    assert m.sum() == 39
    assert np.tril(m, -1).sum() == 29
    assert visible_mask(0, [10], 0).sum() == 55
    # growth law P:672 / P:64: span-sparse pairs vs dense at 32 docs of 64 + 16 suffix
    sp = visible_mask(0, [64] * 32, 16).sum()
    dense = visible_mask(0, [64 * 32 + 16], 0).sum()
    assert dense / sp > 3.0  # "reduces prefill load by 3x" on miss


def test_q_zero_gives_mean_of_visible_v():
    g = np.random.default_rng(5)
    eq, ek, ev = tables()
    eq[:] = 0.0
    pre, frs, cr = toks(g, 3), [toks(g, 5), toks(g, 4)], toks(g, 3)
    o, lse, mask = dense_masked(pre, frs, cr, eq, ek, ev, 1e4)
    allt = np.concatenate([pre] + frs + [cr])
    v = ev[allt]
    for h in range(4):
        exp = (mask.astype(float) @ v[:, h // 2, :]) / mask.sum(1, keepdims=True)
        np.testing.assert_allclose(o[:, h, :], exp, atol=1e-13)
        np.testing.assert_allclose(lse[:, h], np.log(mask.sum(1)), atol=1e-13)


def test_uniform_v_gives_v():
    g = np.random.default_rng(6)
    eq, ek, ev = tables()
    ev[:] = np.arange(16, dtype=float)[None, None, :]
    o, _, _ = dense_masked(toks(g, 2), [toks(g, 3)], toks(g, 4), eq, ek, ev, 1e4)
    np.testing.assert_allclose(o, np.broadcast_to(np.arange(16.0), o.shape), atol=1e-12)


def _sdpa(q, k, v, mask):
    """torch SDPA fp64 with explicit boolean mask; q [R,Hq,d], k/v [N,Hkv,d]."""
    hq, hkv = q.shape[1], k.shape[1]
    qt = torch.from_numpy(q).permute(1, 0, 2)[None]
    kt = torch.from_numpy(np.repeat(k, hq // hkv, axis=1)).permute(1, 0, 2)[None]
    vt = torch.from_numpy(np.repeat(v, hq // hkv, axis=1)).permute(1, 0, 2)[None]
    out = F.scaled_dot_product_attention(qt, kt, vt, attn_mask=torch.from_numpy(mask))
    return out[0].permute(1, 0, 2).numpy()


def test_one_fragment_plus_equals_causal_prefill_library():
    # north_star invariant: a one-fragment ⊕ with empty prefix == ordinary causal prefill of F‖Q.
    g = np.random.default_rng(7)
    eq, ek, ev = tables()
    f, cr = toks(g, 9), toks(g, 5)
    o, _, _ = dense_masked([], [f], cr, eq, ek, ev, 1e4)
    t = np.concatenate([f, cr])
    pos = np.arange(len(t), dtype=float)[:, None]
    q, k, v = rope(eq[t], pos, 1e4), rope(ek[t], pos, 1e4), ev[t]
    hq, hkv = 4, 2
    qt = torch.from_numpy(q).permute(1, 0, 2)[None]
    kt = torch.from_numpy(np.repeat(k, 2, axis=1)).permute(1, 0, 2)[None]
    vt = torch.from_numpy(np.repeat(v, 2, axis=1)).permute(1, 0, 2)[None]
    ref = F.scaled_dot_product_attention(qt, kt, vt, is_causal=True)[0].permute(1, 0, 2).numpy()
    np.testing.assert_allclose(o, ref, atol=1e-12)


def test_dense_matches_library_with_explicit_mask_gqa():
    g = np.random.default_rng(8)
    eq, ek, ev = tables(hq=8, hkv=2, d=32, scale=3.0)
    pre, frs, cr = toks(g, 6), [toks(g, 7), toks(g, 3), toks(g, 5)], toks(g, 6)
    o, lse, mask = dense_masked(pre, frs, cr, eq, ek, ev, 1e4)
    t = np.concatenate([pre] + frs + [cr])
    pos = np.arange(len(t), dtype=float)[:, None]
    q, k, v = rope(eq[t], pos, 1e4), rope(ek[t], pos, 1e4), ev[t]
    np.testing.assert_allclose(o, _sdpa(q, k, v, mask), atol=1e-12)
    # LSE against torch.logsumexp of the explicitly masked scores
    s = torch.einsum("rhd,nhd->hrn", torch.from_numpy(q),
                     torch.from_numpy(np.repeat(k, 4, axis=1))) / np.sqrt(32)
    s = s.masked_fill(~torch.from_numpy(mask)[None], float("-inf"))
    np.testing.assert_allclose(lse, torch.logsumexp(s, -1).T.numpy(), atol=1e-12)


def test_segmentwise_equals_plain_definition():
    # fragment rows at span-local positions == dense rows at global positions (relative RoPE);
    # join rows at global positions == dense cross rows.
    g = np.random.default_rng(9)
    eq, ek, ev = tables(hq=4, hkv=1, d=32, scale=2.0)
    pre, frs, cr = toks(g, 11), [toks(g, 13), toks(g, 1), toks(g, 8)], toks(g, 7)
    o, lse, _ = dense_masked(pre, frs, cr, eq, ek, ev, 1e4)
    po, pl = segment_causal(pre, eq, ek, ev, 1e4)
    np.testing.assert_allclose(po, o[:11], atol=1e-12)
    off = 11
    for f in frs:
        fo, fl = segment_causal(f, eq, ek, ev, 1e4)
        np.testing.assert_allclose(fo, o[off:off + len(f)], atol=1e-12)
        np.testing.assert_allclose(fl, lse[off:off + len(f)], atol=1e-12)
        off += len(f)
    jo, jl = join_rows(pre, frs, cr, eq, ek, ev, 1e4)
    np.testing.assert_allclose(jo, o[off:], atol=1e-12)
    np.testing.assert_allclose(jl, lse[off:], atol=1e-12)
    # row / head subsets
    so, sl = join_rows(pre, frs, cr, eq, ek, ev, 1e4, rows=[0, 6], heads=[3, 1])
    np.testing.assert_allclose(so, jo[[0, 6]][:, [3, 1]], atol=1e-13)


def test_permutation_leaves_fragment_kv_and_rows_unchanged():
    g = np.random.default_rng(10)
    eq, ek, ev = tables()
    pre, frs, cr = toks(g, 4), [toks(g, 6), toks(g, 5), toks(g, 7)], toks(g, 3)
    o1, _, _ = dense_masked(pre, frs, cr, eq, ek, ev, 1e4)
    perm = [2, 0, 1]
    o2, _, _ = dense_masked(pre, [frs[i] for i in perm], cr, eq, ek, ev, 1e4)
    starts1 = np.cumsum([4] + [len(f) for f in frs])[:-1]
    starts2 = np.cumsum([4] + [len(frs[i]) for i in perm])[:-1]
    for new_i, old_i in enumerate(perm):
        L = len(frs[old_i])
        np.testing.assert_allclose(o2[starts2[new_i]:starts2[new_i] + L],
                                   o1[starts1[old_i]:starts1[old_i] + L], atol=1e-12)
    # the join itself is order-sensitive (positions change) — reading R6
    assert not np.allclose(o1[-3:], o2[-3:])


def _plan_pages(view, queries, ek, ev, bs):
    """{fragment content key: [K/V pages of its blocks in chain order]} after the plan's K1."""
    pool = pool_write({}, view, queries, ek, ev, 1e4, bs)
    out = {}
    for seg in view.segments:
        if seg.kind == 1:
            key = queries[seg.query][1][seg.frag_idx].tobytes()
            out[key] = [pool[b * bs + t] for b in seg.blocks for t in range(bs) if b * bs + t in pool]
    return out, pool


def test_permutation_leaves_stored_fragment_kv_unchanged():
    """north_star invariant on the STORED KV: two fresh stores plan the same query with its
    fragments in two ⊕ orders; every fragment's blocks carry the same digests and K1 stores
    the same pages (span-local positions, R2) although its global position Δ_f moved."""
    g = np.random.default_rng(20)
    eq, ek, ev = tables()
    bs = 4
    pre, frs, cr = toks(g, 9), [toks(g, 6), toks(g, 11), toks(g, 7), toks(g, 1)], toks(g, 5)
    perm = [3, 1, 0, 2]
    qa = [(pre, frs, cr)]
    qb = [(pre, [frs[i] for i in perm], cr)]
    va = Store(64, 4, 2, 16, bs).plan(qa)
    vb = Store(64, 4, 2, 16, bs).plan(qb)
    pa, _ = _plan_pages(va, qa, ek, ev, bs)
    pb, _ = _plan_pages(vb, qb, ek, ev, bs)
    assert set(pa) == set(pb) and len(pa) == 4
    for key in pa:
        assert len(pa[key]) == len(np.frombuffer(key, np.int64))
        for (k1, v1), (k2, v2) in zip(pa[key], pb[key]):
            np.testing.assert_array_equal(k1, k2)
            np.testing.assert_array_equal(v1, v2)
    da = {queries_key: seg.digests for seg in va.segments if seg.kind == 1
          for queries_key in [qa[0][1][seg.frag_idx].tobytes()]}
    db = {queries_key: seg.digests for seg in vb.segments if seg.kind == 1
          for queries_key in [qb[0][1][seg.frag_idx].tobytes()]}
    assert da == db
    # a plan that placed a fragment's rows at their global positions would store other pages:
    # the moved fragments' Δ_f differ between the two orders, so this check has teeth
    moved = [s for s in va.segments if s.kind == 1 and s.pos0 != [t for t in vb.segments if t.kind == 1 and
             np.array_equal(qb[0][1][t.frag_idx], qa[0][1][s.frag_idx])][0].pos0]
    assert moved


def _multi_query_case():
    """A batch with a shared prefix (partly hit after a warm-up), a fragment repeated inside the
    plan and across queries, and a partially resident fragment (the LRU evicted two of its
    four blocks). Returns the store, the batch, bs and the history [(plan view, batch)]."""
    g = np.random.default_rng(21)
    bs = 4
    pre = toks(g, 10)
    fa, fb, fc, fd, fx = toks(g, 9), toks(g, 6), toks(g, 13), toks(g, 3), toks(g, 5)
    st = Store(64, 4, 2, 16, bs)
    history = []

    def run(batch):
        v = st.plan(batch)
        history.append((v, batch))
        st.release(v)
        return v

    run([(np.zeros(0, np.int64), [fc], toks(g, 1))])  # plan 1: fc -> blocks 0..3
    run([(pre[:8], [fx], toks(g, 1))])  # plan 2: two prefix blocks + fx, newer than fc
    free = len(st.free)
    # plan 3: a fragment of free + 1 blocks and a 1-token cross evict exactly the two LRU blocks,
    # fc's first two
    run([(np.zeros(0, np.int64), [toks(g, bs * (free + 1))], toks(g, 1))])
    res = st.lookup(hashing.fragment_chain(fc, bs, st.root))
    assert res[0] < 0 and res[1] < 0 and res[2] >= 0 and res[3] >= 0
    queries = [(pre, [fc, fa, fb, fa], toks(g, 7)),
               (pre, [fd, fb], toks(g, 5)),
               (np.zeros(0, np.int64), [fc, fa], toks(g, 4))]
    return st, queries, bs, history


def test_plan_level_expected_equals_dense_definition():
    """plan_prefill_expected / plan_join_expected (what the GPU tests compare against) equal the
    plain dense definition's rows, on a multi-query plan with a hit prefix, repeated fragments
    and partial residency."""
    eq, ek, ev = tables(seed=3)
    st, queries, bs, _ = _multi_query_case()
    view = st.plan(queries)
    kinds = [(s.kind, s.hit, s.compute_begin, s.tok_len) for s in view.segments]
    assert any(k == 0 and 0 < cb < n for k, _, cb, n in kinds)  # prefix partly hit
    frag_jobs = [view.segments[i] for i in view.jobs if view.segments[i].kind == 1]
    assert any(not all(s.write) and any(s.write) for s in frag_jobs)  # partial residency
    eo, el = plan_prefill_expected(view, queries, eq, ek, ev, 1e4)
    r = 0
    for si in view.jobs:
        seg = view.segments[si]
        prefix, frags, cross = queries[seg.query]
        o, l, _ = dense_masked(prefix, frags, cross, eq, ek, ev, 1e4)
        n = seg.tok_len - seg.compute_begin
        g0 = seg.pos0 + seg.compute_begin
        np.testing.assert_allclose(eo[r:r + n], o[g0:g0 + n], atol=1e-12)
        np.testing.assert_allclose(el[r:r + n], l[g0:g0 + n], atol=1e-12)
        r += n
    assert r == len(eo) == len(view.prefill_pos)
    jo, jl = plan_join_expected(view, queries, eq, ek, ev, 1e4)
    r = 0
    for prefix, frags, cross in queries:
        o, l, _ = dense_masked(prefix, frags, cross, eq, ek, ev, 1e4)
        np.testing.assert_allclose(jo[r:r + len(cross)], o[-len(cross):], atol=1e-12)
        np.testing.assert_allclose(jl[r:r + len(cross)], l[-len(cross):], atol=1e-12)
        r += len(cross)


def test_method_from_pool_equals_definition_and_hit_join_equals_recompute():
    """The method's own steps on a simulated pool — K1 writes at stored positions, K2 over a
    job's pages, K3 with Q counter-rotated by Δ_f — give the plain definition's rows;
    a second, all-hit plan of the same batch writes no fragment page and its join equals the
    recompute join (north_star invariant), also with the fragments permuted."""
    eq, ek, ev = tables(seed=4)
    st, queries, bs, history = _multi_query_case()
    pool = {}
    for hv, hb in history:  # the pages the warm-up plans left behind (evicted ones overwritten)
        pool_write(pool, hv, hb, ek, ev, 1e4, bs)
    view = st.plan(queries)
    pool_write(pool, view, queries, ek, ev, 1e4, bs)
    po, pl = prefill_from_pool(view, queries, pool, eq, 1e4, bs)
    eo, el = plan_prefill_expected(view, queries, eq, ek, ev, 1e4)
    np.testing.assert_allclose(po, eo, atol=1e-12)
    np.testing.assert_allclose(pl, el, atol=1e-12)
    cold = []
    for qi, (prefix, frags, cross) in enumerate(queries):
        jo, jl = join_from_pool(view, queries, pool, eq, 1e4, bs, qi)
        o, l, _ = dense_masked(prefix, frags, cross, eq, ek, ev, 1e4)
        np.testing.assert_allclose(jo, o[-len(cross):], atol=1e-12)
        np.testing.assert_allclose(jl, l[-len(cross):], atol=1e-12)
        cold.append(jo)
    st.release(view)
    frag_slots = {b * bs + t for s in view.segments if s.kind == 1 for b in s.blocks for t in range(bs)}
    before = {sl: pool[sl] for sl in frag_slots if sl in pool}
    # warm: every fragment hits; then the same batch with each query's fragments reversed
    for batch in (queries, [(p, f[::-1], c) for p, f, c in queries]):
        hot = st.plan(batch)
        assert all(s.hit == 1 for s in hot.segments if s.kind == 1)
        assert not any(s.kind == 1 for s in (hot.segments[i] for i in hot.jobs))
        pool_write(pool, hot, batch, ek, ev, 1e4, bs)
        for sl, (k, v) in before.items():  # cached fragment KV untouched, bit for bit
            assert pool[sl][0] is k and pool[sl][1] is v
        for qi, (prefix, frags, cross) in enumerate(batch):
            jo, _ = join_from_pool(hot, batch, pool, eq, 1e4, bs, qi)
            if batch is queries:
                np.testing.assert_allclose(jo, cold[qi], atol=1e-13)
            o, _, _ = dense_masked(prefix, frags, cross, eq, ek, ev, 1e4)
            np.testing.assert_allclose(jo, o[-len(cross):], atol=1e-12)
        st.release(hot)


def test_counter_rotation_is_needed():
    """Teeth for join_from_pool: reading fragment pages without counter-rotating Q (as if the
    cached K were at global positions) does not give the definition."""
    eq, ek, ev = tables(seed=5)
    g = np.random.default_rng(22)
    bs = 4
    queries = [(toks(g, 5), [toks(g, 7), toks(g, 6)], toks(g, 3))]
    view = Store(32, 4, 2, 16, bs).plan(queries)
    pool = pool_write({}, view, queries, ek, ev, 1e4, bs)
    for s in view.segments:
        if s.kind == 1:
            s.pos0 = 0  # Δ_f dropped: Q would be rotated at p, keys at span-local t
    jo, _ = join_from_pool(view, queries, pool, eq, 1e4, bs, 0)
    o, _, _ = dense_masked(*queries[0], eq, ek, ev, 1e4)
    assert not np.allclose(jo, o[-3:], atol=1e-6)


def test_workload_shapes():
    w = inputs.c2()
    q = w.queries[0]
    assert len(q.prefix) == 512 and len(q.fragments) == 16 and len(q.cross) == 256
    assert all(len(f) == 1024 for f in q.fragments)
    assert inputs.c4().queries[0].n_tokens == 8 * 2048 + 512
    w3 = inputs.c3()
    kept = sum(any(np.array_equal(f, g) for g in w3.warmup_queries[0].fragments)
               for f in w3.queries[0].fragments)
    assert kept == 12


def test_decode_row_is_the_last_row_of_the_extended_query():
    from oracle import attention as oatt
    # decode_row (generated token t) == the plain definition's last row of the query whose
    # ordered cross segment is cross ‖ gen[0..t] (dense masked attention, written out)
    from paper_2511_02749_b200 import inputs

    sh = inputs.Shape(hq=4, hkv=2, d=16, block_size=4, vocab=64, dtype="fp32")
    eq, ek, ev = inputs.layer_tables(sh, 0, 77)
    g = np.random.default_rng(5)
    prefix, frags, cross = g.integers(0, 64, 5), [g.integers(0, 64, 7), g.integers(0, 64, 3)], g.integers(0, 64, 4)
    gen = g.integers(0, 64, 6)
    for t in range(len(gen)):
        o, lse = oatt.decode_row(prefix, frags, cross, gen, t, eq, ek, ev, sh.rope_base)
        do, dl, _ = oatt.dense_masked(prefix, frags, np.concatenate([cross, gen[: t + 1]]), eq, ek, ev, sh.rope_base)
        np.testing.assert_allclose(o[0], do[-1], atol=1e-12)
        np.testing.assert_allclose(lse[0], dl[-1], atol=1e-12)


def test_split_join_partials_merge_to_the_join():
    # owner-side split join (f1): the home's partial over prefix + its local fragments + cross and
    # each owner's partial over its fragments, merged by LSE, is the join (the plain definition's
    # cross rows) — and leaving any one part out is not
    from oracle import attention as oatt
    from paper_2511_02749_b200 import inputs

    sh = inputs.Shape(hq=4, hkv=2, d=16, block_size=4, vocab=64, dtype="fp32")
    eq, ek, ev = inputs.layer_tables(sh, 0, 91)
    g = np.random.default_rng(12)
    for trial in range(6):
        prefix = g.integers(0, 64, int(g.integers(0, 7)))
        frags = [g.integers(0, 64, int(g.integers(1, 9))) for _ in range(int(g.integers(1, 6)))]
        cross = g.integers(0, 64, int(g.integers(1, 6)))
        owner = g.integers(0, 3, len(frags))  # 0 = the home rank
        parts = [oatt.join_rows_subset(prefix, frags, cross, eq, ek, ev, sh.rope_base, True, owner == 0)]
        for w in (1, 2):
            if (owner == w).any():
                parts.append(oatt.join_rows_subset(prefix, frags, cross, eq, ek, ev, sh.rope_base, False, owner == w))
        o, lse = oatt.merge_lse(parts)
        jo, jl = oatt.join_rows(prefix, frags, cross, eq, ek, ev, sh.rope_base)
        np.testing.assert_allclose(o, jo, atol=1e-12)
        np.testing.assert_allclose(lse, jl, atol=1e-12)
        if len(parts) > 1:
            o2, _ = oatt.merge_lse(parts[:-1])
            assert np.abs(o2 - jo).max() > 1e-6
