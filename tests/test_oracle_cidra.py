"""Pins for oracle/cidra.py (the plain out-of-place definition of CIDRA repositioning, P:610,
P:618-627). Each pin is fixed by the mathematics or the SPEC examples, not by
re-running the oracle's own formula."""
import numpy as np
import pytest

from oracle.cidra import out_degree_duplicates, reposition, validate
from oracle.rope import rope

BASE = 10000.0


def _encoded_pool(seed, L=2, nblk=6, hkv=2, bs=4, d=8):
    """Raw (position-free) vectors r and a pool whose block b holds r[b] encoded at positions
    pos0[b] + t — what a prefill at those positions would have stored."""
    g = np.random.default_rng(seed)
    raw = g.standard_normal((L, nblk, hkv, bs, d))
    pos0 = g.integers(0, 5000, size=nblk)
    t = np.arange(bs)
    k = np.stack([rope(raw[:, b], pos0[b] + t, BASE) for b in range(nblk)], axis=1)
    v = g.standard_normal((L, nblk, hkv, bs, d))
    return raw, pos0, k, v


def test_direct_application():
    # S:386 "rerope(rope(x,5),5,9) = rope(x,9)" lifted to blocks: moving a block that holds
    # rope(r, p0 + t) to new positions p1 + t must give rope(r, p1 + t) — the encoding a fresh
    # prefill at p1 would store (pinned by rope() alone).
    raw, pos0, k, v = _encoded_pool(0)
    moves = [(1, 4, int(pos0[1]), 777), (4, 1, int(pos0[4]), 12)]  # a swap with new positions
    k1, v1 = reposition(k, v, moves, BASE)
    t = np.arange(k.shape[3])
    np.testing.assert_allclose(k1[:, 4], rope(raw[:, 1], 777 + t, BASE), atol=1e-12)
    np.testing.assert_allclose(k1[:, 1], rope(raw[:, 4], 12 + t, BASE), atol=1e-12)
    np.testing.assert_array_equal(v1[:, 4], v[:, 1])  # S:413 swap: V exchanged exactly
    np.testing.assert_array_equal(v1[:, 1], v[:, 4])


def test_untouched_blocks_and_identity_move():
    # S:411 "any single move -> same as rerope on that block"; blocks no move writes keep their
    # bytes; a move with new == old position is the identity (here up to the fp64
    # rounding of reversing and re-applying the rotation)
    raw, pos0, k, v = _encoded_pool(1)
    k1, v1 = reposition(k, v, [(2, 2, 40, 40), (3, 0, 7, 7)], BASE)
    for b in (1, 3, 4, 5):
        np.testing.assert_array_equal(k1[:, b], k[:, b])
        np.testing.assert_array_equal(v1[:, b], v[:, b])
    np.testing.assert_allclose(k1[:, 2], k[:, 2], rtol=0, atol=1e-13)
    np.testing.assert_allclose(k1[:, 0], k[:, 3], rtol=0, atol=1e-13)
    np.testing.assert_array_equal(v1[:, 2], v[:, 2])
    np.testing.assert_array_equal(v1[:, 0], v[:, 3])


def test_cycle_uses_pristine_sources():
    # a 3-cycle 0 -> 1 -> 2 -> 0: every destination gets its source's ORIGINAL content, whatever
    # order an in-place schedule would use ("from pristine sources")
    raw, pos0, k, v = _encoded_pool(2)
    moves = [(0, 1, int(pos0[0]), 100), (1, 2, int(pos0[1]), 200), (2, 0, int(pos0[2]), 300)]
    k1, v1 = reposition(k, v, moves, BASE)
    t = np.arange(k.shape[3])
    for src, dst, _, new in moves:
        np.testing.assert_allclose(k1[:, dst], rope(raw[:, src], new + t, BASE), atol=1e-12)
        np.testing.assert_array_equal(v1[:, dst], v[:, src])


def test_conflicting_demands_duplicate():
    # S:397 "two queries demand block A at positions 10 and 20 -> one duplication": both
    # destinations hold A at their own positions, A itself is unchanged (not a destination)
    raw, pos0, k, v = _encoded_pool(3)
    a = 5
    moves = [(a, 0, int(pos0[a]), 10), (a, 3, int(pos0[a]), 20)]
    k1, _ = reposition(k, v, moves, BASE)
    t = np.arange(k.shape[3])
    np.testing.assert_allclose(k1[:, 0], rope(raw[:, a], 10 + t, BASE), atol=1e-12)
    np.testing.assert_allclose(k1[:, 3], rope(raw[:, a], 20 + t, BASE), atol=1e-12)
    np.testing.assert_array_equal(k1[:, a], k[:, a])
    assert out_degree_duplicates(moves) == 1
    assert out_degree_duplicates([(0, 1, 0, 0), (0, 2, 0, 0), (0, 3, 0, 0), (1, 0, 0, 0)]) == 2


def test_pair_norms_preserved():
    # ReRoPE rotates each (i, i + d/2) pair: per-pair norms are invariant
    _, pos0, k, v = _encoded_pool(4, d=16)
    k1, _ = reposition(k, v, [(0, 1, 0, 123456)], BASE)
    h = k.shape[-1] // 2
    n0 = k[:, 0, ..., :h] ** 2 + k[:, 0, ..., h:] ** 2
    n1 = k1[:, 1, ..., :h] ** 2 + k1[:, 1, ..., h:] ** 2
    np.testing.assert_allclose(n1, n0, rtol=1e-12)


def test_validate():
    validate([(0, 1, 0, 0), (1, 0, 0, 0)], 2)
    with pytest.raises(ValueError):
        validate([(0, 1, 0, 0), (2, 1, 0, 0)], 3)  # block 1 written twice
    with pytest.raises(ValueError):
        validate([(0, 3, 0, 0)], 3)
    with pytest.raises(ValueError):
        validate([(-1, 0, 0, 0)], 3)
