"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): fp32 path max-abs <= 1e-5; bf16 path max-abs <= 1e-2 and
relative L2 <= 5e-3 on attention outputs. With bf16 arithmetic (bf16 Q after RoPE, bf16 KV cache,
bf16 P) even an exactly rounded computation misses fp64 by up to ~2^-9 |O| on peaky rows
(reading R29; the premise is asserted on CPU in tests/test_tolerance_reading.py), so
every bf16-compute check — fp32 or bf16 outputs alike — applies, per element,
max-abs <= 1e-2 + 2^-9 |O_ref| (half a bf16 ulp of the reference), rel-L2 <= 5e-3 unchanged, and
bounds the share of elements above the flat 1e-2 by 1e-4 (each check reports that share).
Block tables / slot maps are bit-exact (the planner is checked on CPU in test_abi_host.py and
again here on the exact plans the GPU runs); V pages bit-exact, K pages within 1 bf16 ulp of the
fp64 RoPE.
"""
import numpy as np
import pytest

from oracle import attention as oatt
from oracle.store import Store
from paper_2511_02749_b200 import inputs, runner, spanq

pytestmark = pytest.mark.gpu

BF16_MAX_ABS, BF16_REL_L2 = 1e-2, 5e-3
FP32_MAX_ABS = 1e-5


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


FLAT_SHARE_MAX = 1e-4  # share of bf16-path elements allowed above the flat 1e-2 (R29)


def check(got, exp, fp32, what, abs_tol=BF16_MAX_ABS, rel_tol=BF16_REL_L2):
    g = _np(got)
    if not exp.size:
        return 0.0, 0.0
    d = np.abs(g - exp)
    rel = np.linalg.norm(g - exp) / max(np.linalg.norm(exp), 1e-30)
    if fp32:
        assert d.max() <= FP32_MAX_ABS, f"{what}: max abs {d.max():.3e}"
        return d.max(), rel
    # bf16 compute (reading R29): 1e-2 + half a bf16 ulp of |O_ref| per element, and only a
    # tiny share of the elements may use the widening at all
    bound = abs_tol + 2.0 ** -9 * np.abs(exp)
    share = float((d > abs_tol).mean())
    print(f"{what}: max abs {d.max():.3e} rel-L2 {rel:.3e} share above {abs_tol:g}: {share:.2e} "
          f"({int((d > abs_tol).sum())} of {d.size})")
    assert (d <= bound).all() and rel <= rel_tol, \
        f"{what}: max abs {d.max():.3e} (worst err/bound {np.max(d / bound):.3f}) rel-L2 {rel:.3e}"
    assert share <= FLAT_SHARE_MAX, f"{what}: {share:.2e} of the elements exceed {abs_tol:g}"
    return d.max(), rel


def check_lse(got, exp, fp32, what, scale=1.0):
    g = _np(got)
    tol = FP32_MAX_ABS * 10 if fp32 else 2e-2 * scale
    err = np.abs(g - exp).max() if exp.size else 0.0
    assert err <= tol, f"{what}: lse max abs {err:.3e}"


def oracle_plan(w, queries, warm=()):
    s = w.shape
    st = Store(1 << 16, s.hq, s.hkv, s.d, s.block_size, s.rope_base, s.model_salt)
    for q in warm:
        st.release(st.plan([(q.prefix, q.fragments, q.cross)]))
    return st.plan([(q.prefix, q.fragments, q.cross) for q in queries])


def run_and_check(w, cuda_dev, nblk=4096, check_pages=True, out_dtype="fp32", abs_tol=BF16_MAX_ABS,
                  rel_tol=BF16_REL_L2, options=None):
    s = w.shape
    fp32 = s.dtype == "fp32"
    ctx = spanq.Context(s, nblk, device=0, max_position=1 << 15, out_dtype=out_dtype)
    for key, value in (options or {}).items():
        ctx.set_option(key, value)
    tabs = [runner.device_tables(s, 0, w.seed, cuda_dev, w.peaky)]
    for q in w.warmup_queries:
        runner.run_pass(ctx, [q], tabs, cuda_dev, release=True)
    res = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    import torch

    torch.cuda.synchronize()
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed, w.peaky)
    ov = oracle_plan(w, w.queries, w.warmup_queries)
    # the plan the GPU ran is the oracle's plan, bit for bit
    np.testing.assert_array_equal(res.view["prefill_slot"], ov.prefill_slot)
    np.testing.assert_array_equal(res.view["join_slot"], ov.join_slot)
    qs = [(q.prefix, q.fragments, q.cross) for q in w.queries]
    if len(ov.jobs):
        eo, el = oatt.plan_prefill_expected(ov, qs, eq, ek, ev, s.rope_base)
        check(res.o_prefill, eo, fp32, f"{w.name} prefill O", abs_tol, rel_tol)
        check_lse(res.lse_prefill, el, fp32, f"{w.name} prefill LSE", abs_tol / BF16_MAX_ABS)
    jo, jl = oatt.plan_join_expected(ov, qs, eq, ek, ev, s.rope_base)
    out = check(res.o_join, jo, fp32, f"{w.name} join O", abs_tol, rel_tol)
    check_lse(res.lse_join, jl, fp32, f"{w.name} join LSE", abs_tol / BF16_MAX_ABS)
    if check_pages:
        kp, vp = _np(ctx.k_pool[0]), _np(ctx.v_pool[0])
        kp = kp.transpose(0, 2, 1, 3).reshape(-1, s.hkv, s.d)  # [blk*bs, hkv, d]
        vp = vp.transpose(0, 2, 1, 3).reshape(-1, s.hkv, s.d)
        toks = np.concatenate([runner.prefill_tokens(res.view, w.queries),
                               runner.join_tokens(res.view, w.queries)])
        pos = np.concatenate([ov.prefill_pos, ov.join_pos])
        slot = np.concatenate([ov.prefill_slot, ov.join_slot])
        m = slot >= 0
        ek_exp, ev_exp = oatt.expected_pages(toks[m], None, ek, ev, s.rope_base, pos[m])
        np.testing.assert_array_equal(vp[slot[m]], ev_exp)  # pure copy: bit-exact
        kerr = np.abs(kp[slot[m]] - ek_exp)
        # one rounding of the result (1 ulp of the target type) + fp32 rotate error, which scales
        # with the magnitude of the rotate-half pair (x_i, x_{i+d/2}) of the unrotated k
        kraw = np.abs(ek[toks[m]].astype(np.float64))
        h = s.d // 2
        pair = np.concatenate([kraw[..., :h] + kraw[..., h:]] * 2, axis=-1)
        ulp = (2.0 ** -23 if fp32 else 2.0 ** -8) * np.abs(ek_exp)
        bound = ulp + 4 * 2.0 ** -24 * pair
        assert (kerr <= bound).all(), f"K pages off: max err/bound {np.max(kerr / bound):.2f}"
        # pad slots are zero
        if len(ov.pad_slots):
            assert (kp[ov.pad_slots] == 0).all() and (vp[ov.pad_slots] == 0).all()
    ctx.close()
    return out


@pytest.mark.parametrize("variant", ["base", "gqa", "prefix", "permuted"])
def test_c1_fp32(cuda_dev, variant):
    run_and_check(inputs.c1(variant=variant), cuda_dev)


@pytest.mark.parametrize("out_dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("bs", [16, 64, 128])
def test_bf16_small_rag(cuda_dev, bs, out_dtype):
    # fp32 / bf16 O at d = 128 take different prefill epilogues (softmax WG vs Q-prep warps)
    w = inputs.make_rag(101, inputs.Shape(**inputs.SHAPE_8B, block_size=bs), 96, 3, [130, 256, 77], 150)
    run_and_check(w, cuda_dev, out_dtype=out_dtype)


def test_bf16_ragged_gqa1_d64(cuda_dev):
    sh = inputs.Shape(hq=4, hkv=4, d=64, block_size=32, vocab=512)
    w = inputs.make_rag(102, sh, 33, 4, [5, 129, 300, 64], 200)
    run_and_check(w, cuda_dev)


def test_bf16_output_dtype(cuda_dev):
    w = inputs.make_rag(106, inputs.Shape(**inputs.SHAPE_8B, block_size=64), 96, 3, [130, 256, 77], 150)
    run_and_check(w, cuda_dev, out_dtype="bf16")


def test_bf16_peaky_softmax(cuda_dev):
    # E_q x 4 (score std 4): stresses the online softmax with large score ranges. The bf16
    # score error grows with |s| (rounded Q and K) and the softmax sharpens with it, so the
    # bars are scaled: max-abs by peaky^1.5, rel-L2 by peaky^0.5 (reading R22).
    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=64, vocab=1024)
    w = inputs.make_rag(103, sh, 200, 2, [400, 333], 260)
    w.peaky = 4.0
    run_and_check(w, cuda_dev, abs_tol=BF16_MAX_ABS * w.peaky ** 1.5, rel_tol=BF16_REL_L2 * w.peaky ** 0.5)


@pytest.mark.parametrize("out_dtype", ["fp32", "bf16"])
def test_bf16_rescale_every_tile(cuda_dev, out_dtype):
    # threshold 0: the conditional O rescale runs on every tile whose max grows, at the normal
    # (unscaled) tolerance — the rescale path itself is exact up to rounding
    w = inputs.make_rag(107, inputs.Shape(hq=8, hkv=2, d=128, block_size=32, vocab=1024), 130, 3,
                        [300, 129, 260], 200)
    run_and_check(w, cuda_dev, out_dtype=out_dtype, options={spanq.OPT_RESCALE_THRESHOLD: 0})


@pytest.mark.parametrize("exp2", [0, 1, 2, 3, 4])
def test_bf16_exp2_modes(cuda_dev, exp2):
    # SPQ_OPT_EXP2: MUFU ex2 in fp32 (0, default), ex2.f16x2 (1), a quarter / half of the
    # exponentials by the FMA-pipe polynomial (2 / 3)
    w = inputs.make_rag(108, inputs.Shape(**inputs.SHAPE_8B, block_size=64), 64, 2, [256, 200], 140)
    run_and_check(w, cuda_dev, options={spanq.OPT_EXP2: exp2})


@pytest.mark.parametrize("bs,hq", [(16, 32), (32, 16), (64, 32), (128, 32), (64, 64)])
def test_bf16_cta_pair_prefill(cuda_dev, bs, hq):
    # SPQ_OPT_PAIR = 1: the prefill on CTA pairs (cta_group::2, M = 256: the 4 q heads of a GQA
    # group over two SMs, K / V sub-tiles split between them); ragged segments, several block
    # sizes (K halves of min(bs, 32) rows), GQA 4 and 8, bf16 O (the path it serves)
    sh = inputs.Shape(hq=hq, hkv=8, d=128, block_size=bs, vocab=2048)
    w = inputs.make_rag(120 + bs, sh, 150, 4, [300, 129, 64, 1000], 140)
    run_and_check(w, cuda_dev, out_dtype="bf16", abs_tol=BF16_MAX_ABS, options={spanq.OPT_PAIR: 1})


@pytest.mark.parametrize("out_dtype", ["fp32", "bf16"])
def test_bf16_multi_query_batch(cuda_dev, out_dtype):
    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=16, vocab=256)
    qs = inputs.random_queries(104, 6, vocab=256, max_frag=5, max_len=200, max_prefix=150,
                               max_cross=180, reuse_p=0.5)
    w = inputs.Workload("batch", sh, qs, 104)
    run_and_check(w, cuda_dev, out_dtype=out_dtype)


def test_c3_shrunk_reuse_and_permutation(cuda_dev):
    w = inputs.c3(scale=0.125)
    run_and_check(w, cuda_dev)


@pytest.mark.parametrize("out_dtype", ["fp32", "bf16"])
def test_c4_shrunk_judge(cuda_dev, out_dtype):
    run_and_check(inputs.c4(scale=0.125), cuda_dev, out_dtype=out_dtype)


def test_hit_join_equals_recompute_join_bitexact(cuda_dev):
    import torch

    sh = inputs.Shape(**inputs.SHAPE_8B, block_size=64, vocab=1024)
    w = inputs.make_rag(105, sh, 128, 4, 256, 130)
    ctx = spanq.Context(sh, 2048, device=0)
    tabs = [runner.device_tables(sh, 0, w.seed, cuda_dev)]
    cold = runner.run_pass(ctx, w.queries, tabs, cuda_dev, release=True)
    hot = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    torch.cuda.synchronize()
    assert hot.view["n_jobs"] == 0  # prefix + every fragment hit
    assert torch.equal(cold.o_join, hot.o_join) and torch.equal(cold.lse_join, hot.lse_join)
    # permuting the fragments leaves every fragment's KV pages untouched (cached content)
    q0 = w.queries[0]
    perm = inputs.SpanQuery(q0.prefix, q0.fragments[::-1], q0.cross)
    k_before = ctx.k_pool.clone()
    res = runner.run_pass(ctx, [perm], tabs, cuda_dev)
    torch.cuda.synchronize()
    fr = [i for i, k in enumerate(res.view["seg_kind"]) if k == 1]
    assert all(res.view["seg_hit"][i] == 1 for i in fr)
    blocks = np.concatenate([res.view["blocks"][res.view["seg_block_off"][i]:
                                                res.view["seg_block_off"][i] + res.view["seg_n_blocks"][i]]
                             for i in fr])
    assert torch.equal(k_before[:, blocks], ctx.k_pool[:, blocks])
    ctx.close()


def test_full_size_c2_sampled_rows(cuda_dev):
    """configs[1] at full size in the bench's launch configuration; sampled (row, head) outputs
    against the oracle computed one by one."""
    import torch

    w = inputs.c2()
    s = w.shape
    ctx = spanq.Context(s, 1024, device=0, max_position=1 << 15, out_dtype="fp32")
    tabs = [runner.device_tables(s, 0, w.seed, cuda_dev)]
    res = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    torch.cuda.synchronize()
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    q = w.queries[0]
    g = np.random.default_rng(7)
    # join rows
    rows = g.choice(len(q.cross), 12, replace=False)
    heads = [0, 5, 17, 31]
    jo, jl = oatt.join_rows(q.prefix, q.fragments, q.cross, eq, ek, ev, s.rope_base, rows, heads)
    got = res.o_join[torch.from_numpy(rows).to(cuda_dev)][:, heads]
    check(got, jo, False, "C2 join sampled")
    # prefill rows: fragment 3 rows and prefix rows
    view = res.view
    for si in [int(view["jobs"][0]), int(view["jobs"][4])]:
        toks = runner.segment_tokens(view, w.queries, si)
        j = list(view["jobs"]).index(si)
        r = g.choice(len(toks), 10, replace=False)
        eo, el = oatt.segment_causal(toks, eq, ek, ev, s.rope_base, r, heads)
        off = int(view["job_row_off"][j])
        got = res.o_prefill[torch.from_numpy(off + r).to(cuda_dev)][:, heads]
        check(got, eo, False, f"C2 prefill seg {si}")
    ctx.close()


@pytest.mark.parametrize("out_dtype,pair", [("fp32", 0), ("bf16", 0), ("bf16", 1)])
def test_full_size_c2_all_rows(cuda_dev, out_dtype, pair):
    """configs[1] at full size in the bench's launch configuration (512-block pool, the bench's
    output dtypes), EVERY output element: all 17,152 prefill rows and all 256 join rows, all 32
    heads, against the fp64 oracle (the whole C2 in a few seconds on the host)."""
    import torch

    w = inputs.c2()
    s = w.shape
    ctx = spanq.Context(s, 512, device=0, max_position=1 << 15, out_dtype=out_dtype)
    ctx.set_option(spanq.OPT_PAIR, pair)  # 1: the CTA-pair prefill kernel
    tabs = [runner.device_tables(s, 0, w.seed, cuda_dev)]
    res = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    torch.cuda.synchronize()
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    ov = oracle_plan(w, w.queries)
    np.testing.assert_array_equal(res.view["prefill_slot"], ov.prefill_slot)
    qs = [(q.prefix, q.fragments, q.cross) for q in w.queries]
    eo, el = oatt.plan_prefill_expected(ov, qs, eq, ek, ev, s.rope_base)
    assert eo.shape == tuple(res.o_prefill.shape) == (17152 - 256, 32, 128)
    check(res.o_prefill, eo, False, f"C2 prefill O all rows ({out_dtype})")
    check_lse(res.lse_prefill, el, False, "C2 prefill LSE all rows")
    jo, jl = oatt.plan_join_expected(ov, qs, eq, ek, ev, s.rope_base)
    assert jo.shape == tuple(res.o_join.shape) == (256, 32, 128)
    check(res.o_join, jo, False, f"C2 join O all rows ({out_dtype})")
    check_lse(res.lse_join, jl, False, "C2 join LSE all rows")
    ctx.close()


def test_multi_layer_plan_reuse(cuda_dev):
    # one plan, three layers (each its own tables and KV-pool layer): the per-launch work
    # counters of the dynamic schedule and the pad zeroing are per launch / per layer
    import torch

    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=32, vocab=1024, layers=3)
    w = inputs.make_rag(109, sh, 100, 3, [300, 129, 260], 200)
    ctx = spanq.Context(sh, 1024, device=0, max_position=1 << 14, out_dtype="fp32")
    plan = ctx.plan(w.queries)
    view = plan.view()
    ov = oracle_plan(w, w.queries)
    qs = [(q.prefix, q.fragments, q.cross) for q in w.queries]
    ptok, jtok = runner.prefill_tokens(view, w.queries), runner.join_tokens(view, w.queries)
    for layer in range(3):
        tab = runner.device_tables(sh, layer, w.seed, cuda_dev)
        op = torch.empty((len(ptok), sh.hq, sh.d), dtype=torch.float32, device=cuda_dev)
        oj = torch.empty((len(jtok), sh.hq, sh.d), dtype=torch.float32, device=cuda_dev)
        plan.prefill(layer, *runner.gather(tab, ptok, cuda_dev), op)
        plan.join(layer, *runner.gather(tab, jtok, cuda_dev), oj)
        torch.cuda.synchronize()
        eq, ek, ev = inputs.layer_tables(sh, layer, w.seed)
        eo, _ = oatt.plan_prefill_expected(ov, qs, eq, ek, ev, sh.rope_base)
        jo, _ = oatt.plan_join_expected(ov, qs, eq, ek, ev, sh.rope_base)
        check(op, eo, False, f"layer {layer} prefill O")
        check(oj, jo, False, f"layer {layer} join O")
    plan.release()
    ctx.close()


def test_sub_range_calls(cuda_dev):
    # prefill jobs and joins issued in two ranges each (the per-call work lists uploaded by the
    # ABI) give the full-range results: prefill bit for bit, joins within tolerance of the oracle
    import torch

    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=16, vocab=256)
    qs = inputs.random_queries(110, 6, vocab=256, max_frag=5, max_len=200, max_prefix=150,
                               max_cross=180, reuse_p=0.5)
    w = inputs.Workload("batch", sh, qs, 110)
    tab = runner.device_tables(sh, 0, w.seed, cuda_dev)
    full = runner.run_pass(spanq.Context(sh, 2048, device=0, out_dtype="fp32"), qs, [tab], cuda_dev)
    ctx = spanq.Context(sh, 2048, device=0, out_dtype="fp32")
    plan = ctx.plan(qs)
    view = plan.view()
    nj, nq = view["n_jobs"], view["n_queries"]
    jr = view["job_row_off"]
    qr = view["query_join_row_off"]
    op = torch.empty_like(full.o_prefill)
    oj = torch.empty_like(full.o_join)
    for a, b in [(0, nj // 2), (nj // 2, nj)]:
        toks = runner.prefill_tokens(view, qs, (a, b))
        if len(toks):
            plan.prefill(0, *runner.gather(tab, toks, cuda_dev), op[jr[a]:jr[b]], jobs=(a, b))
    for a, b in [(0, nq // 2), (nq // 2, nq)]:
        toks = runner.join_tokens(view, qs, (a, b))
        if len(toks):
            plan.join(0, *runner.gather(tab, toks, cuda_dev), oj[qr[a]:qr[b]], queries=(a, b))
    torch.cuda.synchronize()
    assert torch.equal(op, full.o_prefill)
    ov = oracle_plan(w, qs)
    eq, ek, ev = inputs.layer_tables(sh, 0, w.seed)
    jo, _ = oatt.plan_join_expected(ov, [(q.prefix, q.fragments, q.cross) for q in qs], eq, ek, ev, sh.rope_base)
    check(oj, jo, False, "sub-range join O")
    plan.release()
    ctx.close()


def test_bf16_d64_block128(cuda_dev):
    # d = 64 (8-slot K / 4-slot V rings of 8 KB sub-tiles) with 128-token blocks (a 64-key
    # sub-tile is half a block: TMA boxes at row offset 0 / 64)
    sh = inputs.Shape(hq=8, hkv=2, d=64, block_size=128, vocab=1024)
    w = inputs.make_rag(111, sh, 200, 3, [300, 129, 257], 190)
    run_and_check(w, cuda_dev)


def test_full_size_c4_sampled_rows(cuda_dev):
    """configs[3] (judge/generator, 2B shape, 8 x 2048 + 512) at full size; sampled outputs."""
    import torch

    w = inputs.c4()
    s = w.shape
    ctx = spanq.Context(s, 1024, device=0, max_position=1 << 15, out_dtype="fp32")
    res = runner.run_pass(ctx, w.queries, [runner.device_tables(s, 0, w.seed, cuda_dev)], cuda_dev)
    torch.cuda.synchronize()
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    q = w.queries[0]
    g = np.random.default_rng(8)
    heads = [0, 3, s.hq - 1]
    rows = g.choice(len(q.cross), 12, replace=False)
    jo, _ = oatt.join_rows(q.prefix, q.fragments, q.cross, eq, ek, ev, s.rope_base, rows, heads)
    check(res.o_join[torch.from_numpy(rows).to(cuda_dev)][:, heads], jo, False, "C4 join sampled")
    view = res.view
    si = int(view["jobs"][5])
    toks = runner.segment_tokens(view, w.queries, si)
    j = list(view["jobs"]).index(si)
    r = g.choice(len(toks), 10, replace=False)
    eo, _ = oatt.segment_causal(toks, eq, ek, ev, s.rope_base, r, heads)
    off = int(view["job_row_off"][j])
    check(res.o_prefill[torch.from_numpy(off + r).to(cuda_dev)][:, heads], eo, False, "C4 prefill sampled")
    ctx.close()


def test_bf16_matches_rounding_emulation(cuda_dev):
    # The bf16 kernel is as accurate as its formats allow: against an fp64 computation that only
    # rounds the rotated Q, the cached K and P to bf16 (test-side emulation built on the oracle's
    # RoPE), the fragment-prefill outputs agree to 4e-3 (measured 2.5e-3: the kernel's P is taken
    # against a running max that may lag by up to 2^8, so its roundings differ). That the
    # emulation itself sits >= 1e-2 from fp64 on this case (reading R29) is asserted on CPU in
    # tests/test_tolerance_reading.py
    import torch

    from oracle import rope as orope

    s = inputs.Shape(**inputs.SHAPE_8B, block_size=64, vocab=2048)
    w = inputs.make_rag(11, s, 130, 3, [200, 128, 77], 140)
    ctx = spanq.Context(s, 1024, device=0, max_position=1 << 14, out_dtype="fp32")
    res = runner.run_pass(ctx, w.queries, [runner.device_tables(s, 0, w.seed, cuda_dev)], cuda_dev)
    torch.cuda.synchronize()
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    bf = lambda x: torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).double().numpy()
    view = res.view
    worst_emul = worst_exact = 0.0
    for j, si in enumerate(view["jobs"]):
        toks = runner.segment_tokens(view, w.queries, int(si))
        cb = int(view["seg_compute_begin"][si])
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
            P = bf(P) if round_p else P
            return np.einsum("hqk,khd->qhd", P, V) / lsum.transpose(1, 0, 2)

        r0, r1 = int(view["job_row_off"][j]), int(view["job_row_off"][j + 1])
        got = res.o_prefill[r0:r1].double().cpu().numpy()
        emul = attn(bf(Q), bf(K), True)[cb:]
        exact = attn(Q, K, False)[cb:]
        worst_emul = max(worst_emul, float(np.abs(got - emul).max()))
        worst_exact = max(worst_exact, float(np.abs(got - exact).max()))
    print(f"kernel vs bf16-rounding emulation {worst_emul:.3e}, vs exact fp64 {worst_exact:.3e}")
    assert worst_emul <= 4e-3, worst_emul
    ctx.close()


def test_read_blocks(cuda_dev):
    import torch

    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=32, vocab=512, layers=2)
    w = inputs.make_rag(112, sh, 40, 2, [100, 70], 30)
    ctx = spanq.Context(sh, 256, device=0)
    res = runner.run_pass(ctx, w.queries, [runner.device_tables(sh, l, w.seed, cuda_dev) for l in range(2)], cuda_dev)
    ids = res.view["blocks"][:5]
    for layer in range(2):
        k, v = ctx.read_blocks(layer, ids)
        torch.cuda.synchronize()
        assert torch.equal(k, ctx.k_pool[layer, torch.from_numpy(ids.astype(np.int64)).to(cuda_dev)])
        assert torch.equal(v, ctx.v_pool[layer, torch.from_numpy(ids.astype(np.int64)).to(cuda_dev)])
    with pytest.raises(spanq.SpanqError):
        ctx.read_blocks(0, [300])
    res.plan.release()
    ctx.close()


def test_full_size_c3_warm_sampled_rows(cuda_dev):
    """configs[2] at full size: C3's query right after its C2-like warm-up query (12 of 16
    fragments cached, permuted, 4 new, new cross), in the bench's launch configuration: the hits
    are read at their new Δ_f without being rewritten; sampled join rows against the oracle's
    dense definition over the query as written, plus hit statistics."""
    import torch

    w = inputs.c3()
    s = w.shape
    ctx = spanq.Context(s, 1024, device=0, max_position=1 << 15, out_dtype="fp32")
    tabs = [runner.device_tables(s, 0, w.seed, cuda_dev)]
    for q0 in w.warmup_queries:
        runner.run_pass(ctx, [q0], tabs, cuda_dev, release=True)
    st0 = ctx.stats()
    res = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    torch.cuda.synchronize()
    st1 = ctx.stats()
    q = w.queries[0]
    frag_tokens = sum(len(f) for f in q.fragments)
    hit = st1["hit_tokens"] - st0["hit_tokens"]
    # 12 of 16 fragments plus the full prefix blocks are hits (P:123 hit rate = hit / input tokens)
    assert hit >= 0.75 * frag_tokens, (hit, frag_tokens)
    eq, ek, ev = inputs.layer_tables(s, 0, w.seed)
    g = np.random.default_rng(9)
    rows = g.choice(len(q.cross), 12, replace=False)
    heads = [1, 8, 30]
    jo, _ = oatt.join_rows(q.prefix, q.fragments, q.cross, eq, ek, ev, s.rope_base, rows, heads)
    check(res.o_join[torch.from_numpy(rows).to(cuda_dev)][:, heads], jo, False, "C3 warm join sampled")
    res.plan.release()
    ctx.close()


@pytest.mark.parametrize("hq,hkv,d,out_dtype", [(3, 3, 64, "fp32"), (6, 2, 128, "fp32"), (8, 2, 64, "fp32"),
                                                (6, 2, 128, "bf16"), (8, 2, 64, "bf16")])
def test_many_tiny_epochs_stress(cuda_dev, hq, hkv, d, out_dtype):
    """Many one-sub-tile Q epochs (fragments of 1-20 tokens, many queries) in unpaired (odd GQA
    group) and paired launches, repeated: the Q-ring barrier protocol under its tightest timing
    (the unpaired slot-B wait once lapped and deadlocked here)."""
    sh = inputs.Shape(hq=hq, hkv=hkv, d=d, block_size=16, vocab=128)
    for rep in range(3):
        qs = inputs.random_queries(300 + rep, 12, vocab=128, max_frag=6, max_len=20, max_prefix=24,
                                   max_cross=40, reuse_p=0.3)
        run_and_check(inputs.Workload("tiny", sh, qs, 300 + rep), cuda_dev, nblk=2048, out_dtype=out_dtype)


@pytest.mark.parametrize("seed", list(range(32)))
def test_random_workloads_fuzz(cuda_dev, seed):
    """Seeded random shapes and batches against the fp64 oracle: GQA group 1-8 (paired and unpaired
    launches), d 64 / 128, block size 16-128, bf16 (fp32 or bf16 O) or fp32, multi-query batches with
    repeated and permuted fragments, nested ⊕, empty prefixes, ragged lengths, and a warm-up batch on
    the same store so part of the second batch hits the cache. Slot maps bit-exact, outputs and LSE
    within the stated tolerances, K/V pages within their rounding bound."""
    g = np.random.default_rng(9000 + seed)
    hkv = int(g.choice([1, 2, 4]))
    group = int(g.choice([1, 2, 4, 8]))
    dtype = "fp32" if seed % 4 == 3 else "bf16"
    d = int(g.choice([64, 128])) if dtype == "bf16" else 64
    bs = int(g.choice([16, 32, 64, 128]))
    sh = inputs.Shape(hq=hkv * group, hkv=hkv, d=d, block_size=bs, vocab=512, dtype=dtype, model_salt=seed)
    qs = inputs.random_queries(9100 + seed, int(g.integers(2, 6)), vocab=512, max_frag=5,
                               max_len=int(g.integers(20, 260)), max_prefix=int(g.integers(0, 200)),
                               max_cross=int(g.integers(1, 200)), reuse_p=0.4)
    warm, batch = qs[: len(qs) // 2], qs[len(qs) // 2:]
    w = inputs.Workload(f"fuzz{seed}", sh, batch, 9200 + seed, warmup_queries=warm)
    out = "fp32" if dtype == "fp32" or seed % 2 == 0 else "bf16"
    run_and_check(w, cuda_dev, nblk=8192, out_dtype=out)
