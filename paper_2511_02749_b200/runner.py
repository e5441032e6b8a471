"""Host orchestration around the C ABI: stage a workload's inputs on the GPU and run one pass of
the hot path (plan -> prefill jobs -> join) through `spanq`.

Input staging is plumbing, not the method: a token's pre-RoPE q/k/v are rows of the per-layer
synthetic tables (inputs.layer_tables, the stand-in for the QKV projections), gathered in the
packed row order the plan asks for (job order for prefill, query order for the join). Every
step of the method itself runs inside libspanq.so.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import inputs, spanq


def _torch():
    import torch

    return torch


def segment_tokens(view: Dict, queries: Sequence[inputs.SpanQuery], seg: int) -> np.ndarray:
    q = queries[int(view["seg_query"][seg])]
    kind = int(view["seg_kind"][seg])
    if kind == 0:
        return q.prefix
    if kind == 1:
        return q.fragments[int(view["seg_frag_idx"][seg])]
    return q.cross


def prefill_tokens(view: Dict, queries, jobs=None) -> np.ndarray:
    a, b = (0, int(view["n_jobs"])) if jobs is None else jobs
    parts = []
    for j in range(a, b):
        s = int(view["jobs"][j])
        t = segment_tokens(view, queries, s)
        parts.append(np.asarray(t[int(view["seg_compute_begin"][s]):], np.int64))
    return np.concatenate(parts) if parts else np.zeros(0, np.int64)


def join_tokens(view: Dict, queries, qrange=None) -> np.ndarray:
    """Cross rows of queries [a, b) homed on this rank, in query order (the join's packing)."""
    a, b = (0, int(view["n_queries"])) if qrange is None else qrange
    off = view["query_join_row_off"]
    parts = [np.asarray(queries[i].cross, np.int64) for i in range(a, b) if off[i + 1] > off[i]]
    return np.concatenate(parts) if parts else np.zeros(0, np.int64)


@dataclass
class DeviceTables:
    eq: object
    ek: object
    ev: object


def device_tables(shape: inputs.Shape, layer: int, cfg_seed: int, device, peaky: float = 1.0) -> DeviceTables:
    torch = _torch()
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    eq, ek, ev = inputs.layer_tables(shape, layer, cfg_seed, peaky)
    conv = lambda a: torch.from_numpy(a).to(device=device).to(dt)
    return DeviceTables(conv(eq), conv(ek), conv(ev))


def gather(tab: DeviceTables, tokens: np.ndarray, device):
    torch = _torch()
    idx = torch.from_numpy(np.asarray(tokens, np.int64)).to(device)
    return (tab.eq.index_select(0, idx).contiguous(), tab.ek.index_select(0, idx).contiguous(),
            tab.ev.index_select(0, idx).contiguous())


@dataclass
class PassResult:
    plan: spanq.Plan
    view: Dict
    o_prefill: object
    lse_prefill: object
    o_join: object
    lse_join: object


def run_pass(ctx: spanq.Context, queries: Sequence[inputs.SpanQuery], tabs: Sequence[DeviceTables],
             device, stream=None, release: bool = False, exchange=None) -> PassResult:
    """Plan `queries` and run every layer's prefill jobs and joins (one pass of the hot path).

    With world_size > 1, `exchange(plan, view, layer)` moves the layer's remote fragment KV
    between the prefill and the join (parallel.exchange_layer over NCCL)."""
    torch = _torch()
    shape = ctx.shape
    odt = torch.bfloat16 if ctx.out_dtype == "bf16" else torch.float32
    plan = ctx.plan(queries, stream=stream)
    view = plan.view()
    ptok, jtok = prefill_tokens(view, queries), join_tokens(view, queries)
    op = torch.empty((len(ptok), shape.hq, shape.d), dtype=odt, device=device)
    lp = torch.empty((len(ptok), shape.hq), dtype=torch.float32, device=device)
    oj = torch.empty((len(jtok), shape.hq, shape.d), dtype=odt, device=device)
    lj = torch.empty((len(jtok), shape.hq), dtype=torch.float32, device=device)
    for layer, tab in enumerate(tabs):
        if len(ptok):
            q, k, v = gather(tab, ptok, device)
            plan.prefill(layer, q, k, v, op, lp, stream=stream)
        if exchange is not None:
            exchange(plan, view, layer)
        if not len(jtok):
            continue
        q, k, v = gather(tab, jtok, device)
        plan.join(layer, q, k, v, oj, lj, stream=stream)
    if release:
        plan.release(stream=stream)
    return PassResult(plan, view, op, lp, oj, lj)


def random_tables(shape: inputs.Shape, seed: int, device) -> DeviceTables:
    """Bench-only stand-in tables drawn on the device (torch's CUDA generator, N(0,1) rounded to
    the ctx dtype): per-layer inputs for many layers without the host-side draws of
    inputs.layer_tables (which the parity tests and the oracle use)."""
    torch = _torch()
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    mk = lambda h: torch.randn((shape.vocab, h, shape.d), generator=g, device=device, dtype=torch.float32).to(dt)
    return DeviceTables(mk(shape.hq), mk(shape.hkv), mk(shape.hkv))
