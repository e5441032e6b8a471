"""Pins for oracle/rope.py (no implementation to compare with: closed forms + SPEC examples)."""
import numpy as np
import pytest

from oracle.rope import inv_freq, rerope, rope


def test_identity_at_zero():  # S:376 "pos=0 -> identity"
    x = np.random.default_rng(0).standard_normal((5, 64))
    np.testing.assert_array_equal(rope(x, np.zeros(5), 10000.0), x)


def test_d2_unit_vector():  # S:377 "unit pair, d=2, base=10000, pos=p -> (cos p, sin p)"
    for p in [0.0, 1.0, 3.0, 1000.0]:
        out = rope(np.array([1.0, 0.0]), p, 10000.0)
        np.testing.assert_allclose(out, [np.cos(p), np.sin(p)], rtol=0, atol=1e-15)


def test_rotate_half_pairing_d4_closed_form():
    # d=4, base=10000: θ = [1, 10000^(-1/2) = 0.01]; rotate-half pairs (0,2), (1,3) (reading R15).
    np.testing.assert_allclose(inv_freq(4, 10000.0), [1.0, 0.01], rtol=1e-15)
    p = 2.0
    x = np.array([1.0, 0.0, 0.0, 0.0])
    np.testing.assert_allclose(rope(x, p, 10000.0), [np.cos(2), 0, np.sin(2), 0], atol=1e-15)
    x = np.array([0.0, 1.0, 0.0, 0.0])
    np.testing.assert_allclose(rope(x, p, 10000.0), [0, np.cos(0.02), 0, np.sin(0.02)], atol=1e-15)
    x = np.array([0.0, 0.0, 1.0, 0.0])  # second half rotates the other way
    np.testing.assert_allclose(rope(x, p, 10000.0), [-np.sin(2), 0, np.cos(2), 0], atol=1e-15)


def test_norm_preserved():
    x = np.random.default_rng(1).standard_normal((7, 3, 128))
    pos = np.arange(7)[:, None] * 977.0
    np.testing.assert_allclose(np.linalg.norm(rope(x, pos, 10000.0), axis=-1),
                               np.linalg.norm(x, axis=-1), rtol=1e-13)


def test_rerope_direct_and_composition():
    x = np.random.default_rng(2).standard_normal(64)
    np.testing.assert_allclose(rerope(rope(x, 5, 1e4), 5, 9, 1e4), rope(x, 9, 1e4), atol=1e-12)
    a = rerope(rerope(x, 3, 11, 1e4), 11, 40, 1e4)
    np.testing.assert_allclose(a, rerope(x, 3, 40, 1e4), atol=1e-12)


def test_relative_property():
    # <rope(q,a), rope(k,b)> depends only on a-b: the fact that lets fragment KV stay at
    # span-local positions and the join counter-rotate Q by Δ.
    g = np.random.default_rng(3)
    q, k = g.standard_normal(128), g.standard_normal(128)
    for a, b, dlt in [(10, 3, 100), (5000, 4000, 17), (130000, 129000, 65536)]:
        lhs = rope(q, a, 1e4) @ rope(k, b, 1e4)
        rhs = rope(q, a + dlt, 1e4) @ rope(k, b + dlt, 1e4)
        rel = rope(q, a - b, 1e4) @ k
        assert abs(lhs - rhs) < 1e-9 and abs(lhs - rel) < 1e-9
