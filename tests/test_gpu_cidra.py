"""CIDRA in-place repositioning on the GPU (spq_reposition, K8) against the oracle's
out-of-place definition (oracle/cidra.py): V bit-exact, K within one bf16 rounding of the fp64
result (and equal to its round-to-nearest-even except at near-ties), fp32 pools within 1e-5;
blocks no move writes are untouched. Random move graphs with chains, cycles, self-moves and
duplicated sources, at the 8B (d 128, bs 64) and 2B (d 64) shapes."""
import numpy as np
import pytest
import torch

from oracle import cidra as ocidra
from paper_2511_02749_b200 import inputs, spanq

pytestmark = pytest.mark.gpu


def random_moves(g, nb, n):
    dsts = g.choice(nb, size=n, replace=False)
    srcs = g.integers(0, nb, size=n)
    srcs[: n // 4] = dsts[(np.arange(n // 4) + 1) % max(1, n // 4)]  # force some cycles among dsts
    delta = g.integers(-20000, 20000, size=n)
    delta[::7] = 0
    return [int(x) for x in srcs], [int(x) for x in dsts], [int(x) for x in delta]


CASES = [
    dict(hq=32, hkv=8, d=128, block_size=64, dtype="bf16", layers=2, nblk=96, n=80),
    dict(hq=32, hkv=8, d=64, block_size=16, dtype="bf16", layers=2, nblk=64, n=64),
    dict(hq=2, hkv=2, d=64, block_size=16, dtype="fp32", layers=1, nblk=48, n=40),
    dict(hq=8, hkv=2, d=128, block_size=128, dtype="fp32", layers=2, nblk=24, n=24),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dtype']}-d{c['d']}-bs{c['block_size']}")
@pytest.mark.parametrize("seed", [0, 1])
def test_reposition_matches_definition(case, seed):
    c = dict(case)
    nblk, n = c.pop("nblk"), c.pop("n")
    shape = inputs.Shape(**c)
    ctx = spanq.Context(shape, nblk, device=0, max_position=1 << 15)
    g = torch.Generator(device="cuda").manual_seed(seed)
    ctx.k_pool.copy_(torch.randn(ctx.k_pool.shape, generator=g, device="cuda").to(ctx.k_pool.dtype))
    ctx.v_pool.copy_(torch.randn(ctx.v_pool.shape, generator=g, device="cuda").to(ctx.v_pool.dtype))
    k0 = ctx.k_pool.float().cpu().numpy().astype(np.float64)
    v0 = ctx.v_pool.float().cpu().numpy().astype(np.float64)
    src, dst, delta = random_moves(np.random.default_rng(seed), nblk, n)
    st = ctx.reposition(src, dst, delta)
    torch.cuda.synchronize()
    assert st["moves"] == n and st["cycles"] >= 1
    kr, vr = ocidra.reposition(k0, v0, [(s, d, 0, x) for s, d, x in zip(src, dst, delta)], shape.rope_base)
    k1 = ctx.k_pool.float().cpu().numpy().astype(np.float64)
    v1 = ctx.v_pool.float().cpu().numpy().astype(np.float64)
    np.testing.assert_array_equal(v1, vr)  # V: a byte copy
    untouched = np.setdiff1d(np.arange(nblk), dst)
    np.testing.assert_array_equal(k1[:, untouched], k0[:, untouched])
    err = np.abs(k1 - kr)
    if shape.dtype == "bf16":
        # one bf16 rounding of the fp32 rotation: <= half an ulp of the exact value, plus the fp32
        # evaluation's absolute error (|x|, |y| <~ 5, table entries rounded to 2^-24: <~ 1e-6),
        # which only matters where cancellation makes the exact value tiny
        assert (err <= 2.0 ** -8 * np.abs(kr) * 1.001 + 2e-6).all(), float(err.max())
        rne = torch.from_numpy(kr).to(torch.bfloat16).float().numpy()
        assert np.mean(k1 != rne) < 1e-3  # differs from the exactly rounded value only at near-ties
    else:
        assert err.max() <= 1e-5, float(err.max())
    ctx.close()


def test_layer_range_and_launches():
    shape = inputs.Shape(hq=32, hkv=8, d=128, block_size=64, dtype="bf16", layers=3)
    ctx = spanq.Context(shape, 16, device=0)
    ctx.k_pool.copy_(torch.randn(ctx.k_pool.shape, device="cuda").to(torch.bfloat16))
    ctx.v_pool.copy_(torch.randn(ctx.v_pool.shape, device="cuda").to(torch.bfloat16))
    k0, v0 = ctx.k_pool.clone(), ctx.v_pool.clone()
    n0 = ctx.launch_count()
    ctx.reposition([0, 1], [1, 0], [5, -5], layers=(1, 2))
    torch.cuda.synchronize()
    assert ctx.launch_count() == n0 + 1  # one kernel for the whole move set
    for l in (0, 2):
        assert torch.equal(ctx.k_pool[l], k0[l]) and torch.equal(ctx.v_pool[l], v0[l])
    assert torch.equal(ctx.v_pool[1, 0], v0[1, 1]) and torch.equal(ctx.v_pool[1, 1], v0[1, 0])
    # moving back by the opposite shift restores K up to two bf16 roundings
    ctx.reposition([0, 1], [1, 0], [5, -5], layers=(1, 2))
    torch.cuda.synchronize()
    assert torch.equal(ctx.v_pool, v0)
    assert (ctx.k_pool.float() - k0.float()).abs().max().item() <= 2 ** -7 * k0.float().abs().max().item()
    ctx.close()


def test_reposition_store_effects():
    # moved-into blocks leave the content-hash index (they no longer hold what their digest
    # names), and blocks pinned by a live plan refuse to move (SPQ_ESTATE, nothing moved)
    shape = inputs.Shape(hq=8, hkv=2, d=128, block_size=64, vocab=512)
    ctx = spanq.Context(shape, 64, device=0, max_position=1 << 14)
    q = inputs.make_rag(5, shape, 0, 2, [128, 128], 64).queries[0]
    plan = ctx.plan([q])
    view = plan.view()
    frag_blocks = [int(b) for b in view["blocks"][view["seg_block_off"][0]:][:2]]
    digests = view["digests"][:2]
    with pytest.raises(spanq.SpanqError) as e:
        ctx.reposition([frag_blocks[0]], [60], [5])
    assert e.value.status == spanq.ESTATE
    plan.release()
    torch.cuda.synchronize()
    assert (ctx.lookup(digests) == np.array(frag_blocks)).all()
    ctx.reposition([frag_blocks[0]], [frag_blocks[1]], [5])  # block 1 now holds R(block 0)
    torch.cuda.synchronize()
    ids = ctx.lookup(digests)
    assert ids[0] == frag_blocks[0] and ids[1] == -1
    ctx.close()
