"""The k-ary judge reduction on the GPU (§6): every judge of
every ply — its join over the prompt, its ⊕ children and the suffix, and each generated token —
against the fp64 oracle's plain definition with the children's tokens as fragments. Children of
ply >= 2 are the previous judges' outputs, committed by spq_commit_output (K re-encoded to
span-local positions by CIDRA), so those plies also check that plus distribution of an output
gives the KV of the output as a context-free fragment; they must all be cache hits."""
import numpy as np
import pytest
import torch

from oracle import attention as oatt
from paper_2511_02749_b200 import inputs, judge, runner, spanq
from test_gpu_parity import check, check_lse

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,out_dtype", [(4, 2, "fp32"), (5, 2, "bf16"), (6, 3, "fp32")])
def test_judge_tree_vs_oracle(cuda_dev, n, k, out_dtype):
    bs, gen_len = 16, 19
    sh = inputs.Shape(hq=8, hkv=2, d=128, block_size=bs, vocab=512, layers=2)
    g = np.random.default_rng(40 + n)
    cands = [g.integers(0, 512, int(g.integers(20, 90))).astype(np.int32) for _ in range(n)]
    prompt = g.integers(0, 512, 37).astype(np.int32)
    suffix = g.integers(0, 512, 2 * bs).astype(np.int32)  # block-aligned: outputs start a block
    gen_ids = g.integers(0, 512, (n + 8, gen_len))
    tabs = [runner.device_tables(sh, l, 41, cuda_dev) for l in range(sh.layers)]
    ctx = spanq.Context(sh, 1024, device=0, max_position=1 << 12, out_dtype=out_dtype)
    res = judge.run_judge_tree(ctx, cands, prompt, suffix, k, gen_len, tabs, cuda_dev,
                               lambda j, t: int(gen_ids[j, t]), record=True)
    torch.cuda.synchronize()
    assert [len(p) for p in res["plies"]] == [len(p) for p in spanq.reduce_tree(n, k)[0]]
    for p, rec in enumerate(res["records"]):
        view = rec["view"]
        # a child that is an earlier judge's output was committed by spq_commit_output: a cache hit
        # (a candidate that passed up unjudged, R33, is prefilled at its first use)
        kids = [c for j in res["plies"][p] for c in res["children"][j]]
        frag_hits = [int(h) for h, kd in zip(view["seg_hit"], view["seg_kind"]) if kd == 1]
        assert len(kids) == len(frag_hits)
        assert all(h == 1 for c, h in zip(kids, frag_hits) if c >= n)
        for layer in range(sh.layers):
            eq, ek, ev = inputs.layer_tables(sh, layer, 41)
            oj, lj = rec["join"][layer]
            off = view["query_join_row_off"]
            for qi, q in enumerate(rec["queries"]):
                eo, el = oatt.join_rows(q.prefix, q.fragments, q.cross, eq, ek, ev, sh.rope_base)
                check(oj[off[qi]:off[qi + 1]], eo, False, f"ply {p} judge {qi} join L{layer}")
                check_lse(lj[off[qi]:off[qi + 1]], el, False, f"ply {p} judge {qi} join LSE L{layer}")
        ply = res["plies"][p]
        for layer, t, od, ld in rec["decode"]:
            if t % 6 and t != gen_len - 1:
                continue
            eq, ek, ev = inputs.layer_tables(sh, layer, 41)
            for qi, (j, q) in enumerate(zip(ply, rec["queries"])):
                eo, el = oatt.decode_row(q.prefix, q.fragments, q.cross, gen_ids[j], t, eq, ek, ev, sh.rope_base)
                check(od[qi:qi + 1], eo, False, f"ply {p} judge {j} decode t{t} L{layer}")
    ctx.close()
