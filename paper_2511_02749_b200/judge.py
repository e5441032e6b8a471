"""The k-ary judge reduction (§6) executed through the C ABI.

Host orchestration only — every step runs in libspanq.so: the schedule (spq_reduce_tree), each
ply's judges as one multi-query plan ⋈[prompt, ⊕[children], suffix] (spq_plan_create: cache
lookups, misses prefilled as fragments), the joins, token generation (spq_decode_reserve /
spq_decode_step) and plus distribution of each judge's output (spq_commit_output: its blocks
re-encoded to span-local positions by CIDRA and indexed as a fragment), so the next ply's judges
find their children cached. Token ids of the generated outputs are the caller's (there is no
model here: `gen_tokens(judge, t)`), and q/k/v of every token are gathered from the per-layer
synthetic tables (the stand-in for the projections, runner.py).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence

import numpy as np

from . import inputs, runner, spanq


def run_judge_tree(ctx: spanq.Context, candidates: Sequence[np.ndarray], prompt: np.ndarray, suffix: np.ndarray,
                   k: int, gen_len: int, tabs: Sequence[runner.DeviceTables], device,
                   gen_tokens: Callable[[int, int], int], stream=None, record: bool = False,
                   on_ply: Callable = None) -> Dict:
    """Run the reduction over `candidates` (token arrays; cached spans hit, others are prefilled).
    Returns {"plies", "children", "outputs": judge -> generated tokens, "records": per ply
    (queries, view, join O/LSE, decode O/LSE per step) when record=True}."""
    import torch

    shape = ctx.shape
    odt = torch.bfloat16 if ctx.out_dtype == "bf16" else torch.float32
    n = len(candidates)
    plies, children = spanq.reduce_tree(n, k)
    items: Dict[int, np.ndarray] = {i: np.asarray(c, np.int32) for i, c in enumerate(candidates)}
    outputs: Dict[int, np.ndarray] = {}
    records: List[Dict] = []
    for ply in plies:
        queries = [inputs.SpanQuery(prompt, [items[c] for c in children[j]], suffix) for j in ply]
        plan = ctx.plan(queries, stream=stream)
        view = plan.view()
        ptok, jtok = runner.prefill_tokens(view, queries), runner.join_tokens(view, queries)
        op = torch.empty((max(1, len(ptok)), shape.hq, shape.d), dtype=odt, device=device)
        oj = torch.empty((len(jtok), shape.hq, shape.d), dtype=odt, device=device)
        lj = torch.empty((len(jtok), shape.hq), dtype=torch.float32, device=device)
        rec = {"queries": queries, "view": view, "decode": []}
        for layer, tab in enumerate(tabs):
            if len(ptok):
                plan.prefill(layer, *runner.gather(tab, ptok, device), op, stream=stream)
            plan.join(layer, *runner.gather(tab, jtok, device), oj, lj, stream=stream)
            if record:
                rec.setdefault("join", []).append((oj.clone(), lj.clone()))
        plan.decode_reserve(gen_len)
        gen = {j: np.array([gen_tokens(j, t) for t in range(gen_len)], np.int32) for j in ply}
        for t in range(gen_len):  # step-major: token t on every layer, then token t + 1
            toks = np.array([gen[j][t] for j in ply], np.int64)
            for layer, tab in enumerate(tabs):
                od = torch.empty((len(ply), shape.hq, shape.d), dtype=odt, device=device)
                ld = torch.empty((len(ply), shape.hq), dtype=torch.float32, device=device)
                plan.decode_step(layer, t, *runner.gather(tab, toks, device), od, ld, stream=stream)
                if record:
                    rec["decode"].append((layer, t, od, ld))
        for qi, j in enumerate(ply):  # plus distribution: the output becomes a cached span
            plan.commit_output(qi, gen[j], stream=stream)
            items[n + j] = gen[j]
            outputs[j] = gen[j]
        plan.release(stream=stream)
        if on_ply is not None:
            on_ply(ply)
        if record:
            records.append(rec)
    return {"plies": plies, "children": children, "outputs": outputs, "records": records}
