"""Multi-GPU partitioning of a span-query batch — the exchange step.

Each rank plans the same batch with its own (rank, world_size): query q is homed on q mod W (its
prefix, cross rows and join run there) and fragment f is owned by u64le(s_last(f)[0:8]) mod W
(only the owner prefills and caches it). After a layer's prefill jobs, every home rank needs the
KV of the remote-owned fragments its joins read: the plan's exchange lists name them on both sides
in the same order, so one all-to-all per layer moves them:

    pack (K6 gather, per peer)  ->  dist.all_to_all_single (NCCL over NVLink)  ->  unpack (K6 scatter)

Received fragments are indexed on the home rank under their digests (reading R38, digest-keyed
replicas): a later plan there hits them, and once per plan `exchange_needs` tells each owner which
candidate fragments still have to move (one byte each, a tiny all-to-all).

Buffers are laid out [n_blocks][2 (K, V)][Hkv][bs][d] in the pool dtype. Everything here is
argument marshalling around the C ABI (spq_exchange_pack / spq_exchange_unpack) and the collective.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional

import numpy as np


def block_elems(shape) -> int:
    """Elements of one block of one layer, K and V together."""
    return 2 * shape.hkv * shape.block_size * shape.d


def exchange_counts(view: Dict, world: int):
    """Per-peer block counts (send, recv) of a plan view."""
    send = [len(view["send"].get(p, ())) for p in range(world)]
    recv = [len(view["recv"].get(p, ())) for p in range(world)]
    return send, recv


def _a2a(recvbuf, sendbuf, out_splits: List[int], in_splits: List[int], group=None):
    import torch.distributed as dist

    dist.all_to_all_single(recvbuf, sendbuf, out_splits, in_splits, group=group)


def exchange_needs(plan, view: Dict, rank: int, world: int, device="cpu", group=None,
                   transport: Optional[Callable] = None) -> Dict:
    """Replica protocol (DESIGN reading R38), once per plan before its first exchange: every home
    rank sends each owner one byte per candidate fragment (1 = send its KV, 0 = a replica is
    resident here); each owner narrows its send lists accordingly. Returns the refreshed view."""
    import torch

    out_n = [len(view["need"].get(p, ())) for p in range(world)]  # flags this rank sends to owner p
    in_n = list(view["n_cand_send"])                                # flags home p sends here
    assert out_n[rank] == 0 and in_n[rank] == 0, "a rank never exchanges with itself"
    sendbuf = torch.zeros(sum(out_n), dtype=torch.uint8, device=device)
    off = 0
    for p in range(world):
        if out_n[p]:
            sendbuf[off:off + out_n[p]] = torch.from_numpy(view["need"][p].astype(np.uint8)).to(device)
        off += out_n[p]
    recvbuf = torch.zeros(sum(in_n), dtype=torch.uint8, device=device)
    (transport or (lambda r, s_, o, i: _a2a(r, s_, o, i, group)))(recvbuf, sendbuf, in_n, out_n)
    flags = recvbuf.cpu().numpy()
    off = 0
    for p in range(world):
        if in_n[p]:
            plan.exchange_set_need(p, flags[off:off + in_n[p]])
        off += in_n[p]
    return plan.view()


def exchange_layer(plan, view: Dict, layer: int, shape, device, dtype, rank: int, world: int,
                   group=None, stream=None, transport: Optional[Callable] = None) -> Dict[str, int]:
    """Move one layer's remote fragment KV to the home ranks. Returns the bytes sent/received.

    `transport(recvbuf, sendbuf, out_splits, in_splits)` defaults to an all-to-all on `group`.
    """
    import torch

    be = block_elems(shape)
    send, recv = exchange_counts(view, world)
    assert send[rank] == 0 and recv[rank] == 0, "a rank never exchanges with itself"
    sendbuf = torch.empty(sum(send) * be, dtype=dtype, device=device)
    recvbuf = torch.empty(sum(recv) * be, dtype=dtype, device=device)
    off = 0
    for p in range(world):
        if send[p]:
            plan.exchange_pack(layer, p, sendbuf[off:off + send[p] * be], stream=stream)
        off += send[p] * be
    (transport or (lambda r, s, o, i: _a2a(r, s, o, i, group)))(
        recvbuf, sendbuf, [c * be for c in recv], [c * be for c in send])
    off = 0
    for p in range(world):
        if recv[p]:
            plan.exchange_unpack(layer, p, recvbuf[off:off + recv[p] * be], stream=stream)
        off += recv[p] * be
    elt = sendbuf.element_size()
    return {"sent_bytes": sum(send) * be * elt, "recv_bytes": sum(recv) * be * elt}


# ---------------------------------------------------------------- owner-side split join (f1)
def split_rows(view: Dict, world: int):
    """Rows per peer of the two split-join exchanges: (qsend[w] = rows of the home queries whose Q
    goes to owner w = partial rows coming back from w, qrecv[h] = rows of this rank's tasks homed
    on h = partial rows going back to h)."""
    off = view["query_join_row_off"]
    qsend = [sum(int(off[q + 1] - off[q]) for q in view["xq"].get(w, [])) for w in range(world)]
    qrecv = [0] * world
    for (query, home, n_rows, _pos0, _b, _e) in view["tasks"]:
        qrecv[home] += n_rows
    return qsend, qrecv


def split_exchange_layer(plan, view: Dict, layer: int, shape, device, q_join, rank: int, world: int,
                         group=None, stream=None, transport: Optional[Callable] = None,
                         local_join: Optional[Callable] = None) -> Dict[str, int]:
    """One layer of the owner-side split join around the C-ABI calls: pack Q -> all-to-all ->
    task join (owner) -> all-to-all of the fp32 partials -> the caller's merge input. Returns the
    partial buffers to pass to spq_split_merge (and the bytes moved). `local_join()` (the home's
    spq_split_join_local) is issued right after the Q exchange so it overlaps the task joins of
    the owners."""
    import torch

    qsend_rows, qrecv_rows = split_rows(view, world)
    hq, d = shape.hq, shape.d
    send = torch.empty((sum(qsend_rows), hq, d), dtype=q_join.dtype, device=device)
    recv = torch.empty((sum(qrecv_rows), hq, d), dtype=q_join.dtype, device=device)
    plan.split_pack_q(q_join, send, stream=stream)
    tr = transport or (lambda r, s_, o, i: _a2a(r, s_, o, i, group))
    tr(recv.view(-1), send.view(-1), [n * hq * d for n in qrecv_rows], [n * hq * d for n in qsend_rows])
    if local_join is not None:
        local_join()
    po = torch.empty((sum(qrecv_rows), hq, d), dtype=torch.float32, device=device)
    pl = torch.empty((sum(qrecv_rows), hq), dtype=torch.float32, device=device)
    plan.split_task_join(layer, recv, po, pl, stream=stream)
    ro = torch.empty((sum(qsend_rows), hq, d), dtype=torch.float32, device=device)
    rl = torch.empty((sum(qsend_rows), hq), dtype=torch.float32, device=device)
    tr(ro.view(-1), po.view(-1), [n * hq * d for n in qsend_rows], [n * hq * d for n in qrecv_rows])
    tr(rl.view(-1), pl.view(-1), [n * hq for n in qsend_rows], [n * hq for n in qrecv_rows])
    qb = send.numel() * send.element_size()
    pb = po.numel() * 4 + pl.numel() * 4
    return {"part_o": ro, "part_lse": rl, "q_bytes": qb, "partial_bytes": pb}
