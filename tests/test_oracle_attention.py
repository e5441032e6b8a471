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

from oracle.attention import (dense_masked, expected_pages, join_rows, segment_causal,
                              visible_mask)
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
        k1, v1 = expected_pages(frs[old_i], None, ek, ev, 1e4, np.arange(L))
        np.testing.assert_array_equal(k1, expected_pages(frs[old_i], None, ek, ev, 1e4,
                                                         np.arange(L))[0])
    # the join itself is order-sensitive (positions change) — reading R6
    assert not np.allclose(o1[-3:], o2[-3:])


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
