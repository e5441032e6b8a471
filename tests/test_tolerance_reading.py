"""Reading R29: why the bf16 path's bar is max-abs <= 1e-2 + 2^-9 |O_ref|.

The premise, asserted here on CPU (no kernel involved): an fp64 computation that only rounds the
operands the bf16 path stores in bf16 — Q after RoPE, the cached K (RoPE'd, SPEC S:370-373 / R18)
and P before PV — is itself more than 1e-2 from the exact fp64 result on the smoke case of
`__graft_entry__.smoke()`, while its share of elements above 1e-2 is tiny. So no bf16-storage
kernel can guarantee the flat 1e-2 everywhere, and the GPU tests bound the share above it
(tests/test_gpu_parity.py FLAT_SHARE_MAX) instead of dropping the flat bar.
"""
import numpy as np
import torch

from oracle import rope as orope
from paper_2511_02749_b200 import inputs


def _bf(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).double().numpy()


def test_bf16_rounding_alone_exceeds_flat_bar_on_smoke_case():
    s = inputs.Shape(**inputs.SHAPE_8B, block_size=64, vocab=2048)
    w = inputs.make_rag(11, s, 130, 3, [200, 128, 77], 140)
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    q = w.queries[0]
    worst, above, total = 0.0, 0, 0
    for toks in [q.prefix] + list(q.fragments):
        L = len(toks)
        pos = np.arange(L)[:, None]
        Q = orope.rope(eq[toks].astype(np.float64), pos, s.rope_base)
        K = np.repeat(orope.rope(ek[toks].astype(np.float64), pos, s.rope_base), s.hq // s.hkv, axis=1)
        V = np.repeat(ev[toks].astype(np.float64), s.hq // s.hkv, axis=1)
        mask = np.tril(np.ones((L, L), bool))

        def attn(Qx, Kx, round_p):
            S = np.where(mask[None], np.einsum("qhd,khd->hqk", Qx, Kx) / np.sqrt(s.d), -np.inf)
            P = np.exp(S - S.max(-1, keepdims=True))
            lsum = P.sum(-1, keepdims=True)
            P = _bf(P) if round_p else P
            return np.einsum("hqk,khd->qhd", P, V) / lsum.transpose(1, 0, 2)

        exact = attn(Q, K, False)
        emul = attn(_bf(Q), _bf(K), True)
        d = np.abs(emul - exact)
        worst = max(worst, float(d.max()))
        above += int((d > 1e-2).sum())
        total += d.size
        # every element is inside the widened per-element bar
        assert (d <= 1e-2 + 2.0 ** -9 * np.abs(exact)).all()
    assert worst >= 1e-2, worst  # R29's premise: the rounding alone breaks the flat bar
    assert 0 < above <= 1e-4 * total, (above, total)
