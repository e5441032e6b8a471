"""Decode after the join (spq_decode_reserve / spq_decode_step, K9) and plus distribution
(spq_commit_span) on the GPU against the fp64 oracle.

* Each generated token's row equals oracle.attention.decode_row — the plain definition's last
  row of the query whose ordered cross segment is cross ‖ gen[0..t] (pinned on CPU in
  test_oracle_attention.py) — within the bf16 bar of test_gpu_parity (fp32 path: 1e-5).
* Row t reads the K/V that steps 0..t-1 wrote (and its own), so the parity of later rows also
  checks the generated tokens' pages.
* Plus distribution: an inner generate's (input ‖ output) committed as a span and reused as a ⊕
  fragment gives a join bit-identical to recomputing that fragment from scratch, and its pages
  equal the pages a prefill of the span writes.
"""
import numpy as np
import pytest
import torch

from oracle import attention as oatt
from paper_2511_02749_b200 import inputs, runner, spanq
from test_gpu_parity import check, check_lse

pytestmark = pytest.mark.gpu


def run_decode(w, cuda_dev, n_gen, out_dtype="fp32", layers=1, nblk=2048):
    s = inputs.Shape(**{**w.shape.__dict__, "layers": layers})
    fp32 = s.dtype == "fp32"
    ctx = spanq.Context(s, nblk, device=0, max_position=1 << 15, out_dtype=out_dtype)
    tabs = [runner.device_tables(s, l, w.seed, cuda_dev) for l in range(layers)]
    res = runner.run_pass(ctx, w.queries, tabs, cuda_dev)
    plan, view = res.plan, res.view
    rows = [q for q in range(len(w.queries)) if view["query_join_row_off"][q + 1] > view["query_join_row_off"][q]]
    plan.decode_reserve(n_gen)
    g = np.random.default_rng(w.seed + 17)
    gen = [g.integers(0, s.vocab, n_gen).astype(np.int64) for _ in rows]
    odt = torch.float32 if out_dtype == "fp32" else torch.bfloat16
    outs = {}
    for layer in range(layers):
        for t in range(n_gen):
            toks = np.array([gg[t] for gg in gen])
            q, k, v = runner.gather(tabs[layer], toks, cuda_dev)
            o = torch.empty((len(rows), s.hq, s.d), dtype=odt, device=cuda_dev)
            lse = torch.empty((len(rows), s.hq), dtype=torch.float32, device=cuda_dev)
            plan.decode_step(layer, t, q, k, v, o, lse)
            outs[(layer, t)] = (o, lse)
    torch.cuda.synchronize()
    for layer in range(layers):
        eq, ek, ev = inputs.layer_tables(s, layer, w.seed)
        for t in range(n_gen):
            o, lse = outs[(layer, t)]
            for b, qi in enumerate(rows):
                q = w.queries[qi]
                eo, el = oatt.decode_row(q.prefix, q.fragments, q.cross, gen[b], t, eq, ek, ev, s.rope_base)
                check(o[b:b + 1], eo, fp32, f"{w.name} decode L{layer} t{t} q{qi}")
                check_lse(lse[b:b + 1], el, fp32, f"{w.name} decode LSE L{layer} t{t} q{qi}")
    return ctx, plan, view, rows, gen, s


@pytest.mark.parametrize("out_dtype", ["fp32", "bf16"])
def test_decode_8b_shape(cuda_dev, out_dtype):
    # GQA 4 (g = 4 q heads share each K/V tile), d 128, bs 64; the cross (150 tokens) ends inside
    # a block, so generation first fills the partial cross tail block, then new blocks
    w = inputs.make_rag(201, inputs.Shape(**inputs.SHAPE_8B, block_size=64, vocab=2048), 96, 3, [130, 256, 77], 150)
    ctx, *_ = run_decode(w, cuda_dev, 6, out_dtype=out_dtype)
    ctx.close()


def test_decode_multi_query_two_layers_d64(cuda_dev):
    # several queries (shared and repeated fragments), two layers, d 64, bs 16, GQA 4
    sh = inputs.Shape(hq=8, hkv=2, d=64, block_size=16, vocab=256)
    qs = inputs.random_queries(204, 4, vocab=256, max_frag=4, max_len=150, max_prefix=60, max_cross=70, reuse_p=0.5)
    # (row t attends to the K/V the steps before it wrote: later rows check those pages too)
    ctx, *_ = run_decode(inputs.Workload("dq", sh, qs, 204), cuda_dev, 20, layers=2)
    ctx.close()


def test_decode_fp32_gqa2(cuda_dev):
    sh = inputs.Shape(hq=4, hkv=2, d=64, block_size=16, vocab=512, dtype="fp32")
    w = inputs.make_rag(202, sh, 20, 3, [64, 33, 100], 40)
    ctx, *_ = run_decode(w, cuda_dev, 9)
    ctx.close()


def test_decode_mha_d128(cuda_dev):
    sh = inputs.Shape(hq=4, hkv=4, d=128, block_size=32, vocab=512)
    w = inputs.make_rag(203, sh, 0, 2, [300, 129], 64)
    ctx, *_ = run_decode(w, cuda_dev, 3)
    ctx.close()


def test_plus_distribution_commit_equals_recompute(cuda_dev):
    """Inner generate ⋈[input] -> decode n_gen tokens -> commit (input ‖ output) as a span; an
    outer judge query ⋈[prompt, ⊕[span, other], suffix] then hits the span, and its join equals
    (bit for bit) the join of a fresh context that prefilled the span as an ordinary fragment."""
    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=64, vocab=1024)
    s = inputs.Shape(**{**sh.__dict__, "layers": 2})
    g = np.random.default_rng(31)
    inp = g.integers(0, 1024, 150).astype(np.int32)
    n_gen = 40
    gen = g.integers(0, 1024, n_gen).astype(np.int32)
    tabs = [runner.device_tables(s, l, 31, cuda_dev) for l in range(2)]
    ctx = spanq.Context(s, 512, device=0, max_position=1 << 14, out_dtype="fp32")
    inner = inputs.SpanQuery(np.zeros(0, np.int32), [], inp)
    res = runner.run_pass(ctx, [inner], tabs, cuda_dev)  # the input's KV (its cross rows)
    res.plan.decode_reserve(n_gen)
    for layer in range(2):
        for t in range(n_gen):
            q, k, v = runner.gather(tabs[layer], gen[t:t + 1], cuda_dev)
            res.plan.decode_step(layer, t, q, k, v, torch.empty((1, s.hq, s.d), device=cuda_dev))
    n = res.plan.commit_span(0, gen, crop=False)
    span = np.concatenate([inp, gen])
    assert n == len(span)
    res.plan.release()
    other = g.integers(0, 1024, 100).astype(np.int32)
    outer = inputs.SpanQuery(g.integers(0, 1024, 70).astype(np.int32), [span, other], g.integers(0, 1024, 90).astype(np.int32))
    got = runner.run_pass(ctx, [outer], tabs, cuda_dev)
    frag_hits = [int(h) for h, k in zip(got.view["seg_hit"], got.view["seg_kind"]) if k == 1]
    assert frag_hits == [1, 0]
    fresh = spanq.Context(s, 512, device=0, max_position=1 << 14, out_dtype="fp32")
    ref = runner.run_pass(fresh, [outer], tabs, cuda_dev)
    torch.cuda.synchronize()
    assert torch.equal(got.o_join, ref.o_join) and torch.equal(got.lse_join, ref.lse_join)
    # the committed pages are the pages a prefill of the span writes, bit for bit
    def frag_blocks(v):
        i = [j for j, k in enumerate(v["seg_kind"]) if k == 1][0]
        return v["blocks"][v["seg_block_off"][i]:v["seg_block_off"][i] + v["seg_n_blocks"][i]]

    ids_got, ids_ref = frag_blocks(got.view), frag_blocks(ref.view)
    assert len(ids_got) == 3
    for layer in range(2):
        ka, va = ctx.read_blocks(layer, ids_got)
        kb, vb = fresh.read_blocks(layer, ids_ref)
        assert torch.equal(ka, kb) and torch.equal(va, vb)
    ctx.close()
    fresh.close()


@pytest.mark.parametrize("seed", list(range(12)))
def test_decode_random_fuzz(cuda_dev, seed):
    """Seeded random shapes (GQA group 1-8, d 64 / 128, block size 16-128, bf16 / fp32) and
    multi-query batches; a few decode steps per query, each row against the oracle's decode_row."""
    g = np.random.default_rng(7000 + seed)
    hkv = int(g.choice([1, 2, 4]))
    group = int(g.choice([1, 2, 4, 8]))
    dtype = "fp32" if seed % 4 == 3 else "bf16"
    d = int(g.choice([64, 128])) if dtype == "bf16" else 64
    bs = int(g.choice([16, 32, 64, 128]))
    sh = inputs.Shape(hq=hkv * group, hkv=hkv, d=d, block_size=bs, vocab=512, dtype=dtype, model_salt=seed)
    qs = inputs.random_queries(7100 + seed, int(g.integers(1, 4)), vocab=512, max_frag=4,
                               max_len=int(g.integers(20, 200)), max_prefix=int(g.integers(0, 120)),
                               max_cross=int(g.integers(1, 150)), reuse_p=0.4)
    out = "fp32" if dtype == "fp32" or seed % 2 == 0 else "bf16"
    ctx, *_ = run_decode(inputs.Workload(f"dfuzz{seed}", sh, qs, 7200 + seed), cuda_dev, int(g.integers(1, 6)),
                         out_dtype=out, nblk=4096)
    ctx.close()
