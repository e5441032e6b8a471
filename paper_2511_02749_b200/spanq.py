"""Thin Python binding of the C ABI (include/spanq.h) — argument marshalling only.

Every step of the hot path runs inside libspanq.so (C++ planner/store, CUDA kernels). This
module converts numpy arrays / torch tensors to pointers and back; it never computes any part
of the method and has no CPU fallback: if the library is missing it raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import inputs as _inputs

# SPANQ_LIB (tuning / A/B only) points at an alternative build of the same library
_LIB_PATH = os.environ.get("SPANQ_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                        "libspanq.so")
_lib = None

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ESTATE = range(6)
BF16, FP32 = 0, 1
# spq_option keys (include/spanq.h)
OPT_EXP2, OPT_RESCALE_THRESHOLD, OPT_PDL, OPT_HASH_SCALAR, OPT_PAIR = 1, 2, 3, 4, 5


class SpanqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"spanq status {status}: {msg}")
        self.status = status


class spq_config(C.Structure):
    _fields_ = [
        ("num_q_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
        ("num_layers", C.c_int32), ("block_size", C.c_int32), ("num_blocks", C.c_int64),
        ("dtype", C.c_int32), ("rope_base", C.c_double), ("max_position", C.c_int32),
        ("model_salt", C.c_uint64), ("k_pool", C.c_void_p), ("v_pool", C.c_void_p),
        ("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
        ("out_dtype", C.c_int32), ("split_join", C.c_int32),
    ]


class spq_node(C.Structure):
    _fields_ = [("op", C.c_int32), ("num_children", C.c_int32), ("tok_begin", C.c_int64),
                ("tok_len", C.c_int64)]


class spq_query(C.Structure):
    _fields_ = [("nodes", C.POINTER(spq_node)), ("num_nodes", C.c_int32),
                ("tokens", C.POINTER(C.c_int32)), ("num_tokens", C.c_int64)]


_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_U8P = C.POINTER(C.c_uint8)


class spq_plan_view(C.Structure):
    _fields_ = [
        ("n_queries", C.c_int32), ("n_segments", C.c_int32), ("n_jobs", C.c_int32),
        ("n_blocks_total", C.c_int64),
        ("seg_query", _I32P), ("seg_kind", _I32P), ("seg_frag_idx", _I32P), ("seg_tok_len", _I32P),
        ("seg_pos0", _I32P), ("seg_hit", _I32P), ("seg_compute_begin", _I32P),
        ("seg_block_off", _I32P), ("seg_n_blocks", _I32P),
        ("blocks", _I32P), ("block_write", _U8P), ("digests", _U8P), ("join_digests", _U8P),
        ("jobs", _I32P), ("job_row_off", _I64P),
        ("n_prefill_rows", C.c_int64), ("prefill_pos", _I32P), ("prefill_slot", _I64P),
        ("n_join_rows", C.c_int64), ("query_join_row_off", _I64P), ("join_pos", _I32P),
        ("join_slot", _I64P), ("n_pad_slots", C.c_int64), ("pad_slots", _I64P),
        ("prefill_flops", C.c_double), ("join_flops", C.c_double),
        ("prefill_kv_bytes", C.c_int64), ("join_kv_bytes", C.c_int64),
        ("n_join_queries", C.c_int32), ("world_size", C.c_int32),
        ("send_off", _I64P), ("send_blocks", _I32P), ("recv_off", _I64P), ("recv_blocks", _I32P),
        ("n_tasks", C.c_int32), ("tasks", _I32P), ("xq_off", _I32P), ("xq_queries", _I32P),
        ("cand_recv_off", _I64P), ("cand_recv_need", _U8P), ("cand_send_off", _I64P),
    ]


class spq_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "lookups", "hit_blocks", "miss_blocks", "hit_tokens", "input_tokens", "evictions",
        "inserted_blocks", "resident_blocks", "free_blocks", "pinned_blocks", "plans")]


class spq_cidra_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "moves", "components", "cycles", "duplicates", "ops", "max_component_ops")]


# name -> (restype, argtypes) for every entry point of include/spanq.h
SIGNATURES = {
    "spq_create": (C.c_int, [C.POINTER(spq_config), C.POINTER(C.c_void_p)]),
    "spq_destroy": (None, [C.c_void_p]),
    "spq_last_error": (C.c_char_p, []),
    "spq_version": (C.c_char_p, []),
    "spq_block_hashes": (C.c_int, [C.c_void_p, C.POINTER(spq_query), C.c_void_p, C.c_int64, _I64P]),
    "spq_lookup": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "spq_insert": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "spq_plan_create": (C.c_int, [C.c_void_p, C.POINTER(spq_query), C.c_int32, C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
    "spq_plan_view_get": (C.c_int, [C.c_void_p, C.POINTER(spq_plan_view)]),
    "spq_prefill_jobs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "spq_join": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spq_join_phase": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spq_exchange_set_need": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, _U8P, C.c_int64, C.c_void_p]),
    "spq_exchange_pack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                    C.c_void_p]),
    "spq_exchange_unpack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                      C.c_void_p]),
    "spq_plan_release": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "spq_get_stats": (C.c_int, [C.c_void_p, C.POINTER(spq_stats)]),
    "spq_evict_all": (C.c_int, [C.c_void_p]),
    "spq_read_blocks": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "spq_reposition": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                 C.c_int32, C.c_void_p, C.POINTER(spq_cidra_stats)]),
    "spq_cidra_schedule": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_int64, _I64P, C.c_void_p, C.c_int64, _I64P,
                                     C.POINTER(spq_cidra_stats)]),
    "spq_launch_count": (C.c_int, [C.c_void_p, _I64P]),
    "spq_last_attn_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "spq_set_timing": (C.c_int, [C.c_void_p, C.c_int32]),
    "spq_decode_reserve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "spq_decode_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spq_commit_span": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                  _I32P]),
    "spq_commit_output": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, _I32P]),
    "spq_reduce_tree": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
                                  _I32P, _I32P]),
    "spq_bulk_order": (C.c_int, [C.c_void_p, C.POINTER(spq_query), C.c_int32, C.c_int64, C.c_void_p]),
    "spq_split_pack_q": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "spq_split_task_join": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "spq_split_join_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]),
    "spq_split_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "spq_set_option": (C.c_int, [C.c_void_p, C.c_int32, C.c_double]),
    "spq_set_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
}


def lib():
    """Load libspanq.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise FileNotFoundError(
                f"{_LIB_PATH} not built; run `python -m paper_2511_02749_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(_LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        raise SpanqError(status, lib().spq_last_error().decode())


def _ptr(x) -> Optional[int]:
    """torch tensor / numpy array / None -> raw address."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def _stream_ptr(stream, device: int = -1) -> Optional[int]:
    """Stream handle for the ABI. None means torch's current stream of the ctx's device (so the
    kernels are ordered after the torch work that produced their inputs), never the legacy
    default stream; host-only contexts pass NULL."""
    if stream is None:
        if device < 0:
            return None
        import torch

        return torch.cuda.current_stream(device).cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)



class _QueryBuf:
    """Keeps the ctypes arrays of one spq_query alive."""

    def __init__(self, nodes: np.ndarray, tokens: np.ndarray):
        nodes = np.asarray(nodes, dtype=np.int64).reshape(-1, 4)
        # spq_node = {int32 op, int32 num_children, int64 tok_begin, int64 tok_len}: three
        # little-endian int64 words per node (op | num_children << 32, tok_begin, tok_len)
        assert C.sizeof(spq_node) == 24
        self.nodes = np.empty((max(1, len(nodes)), 3), dtype=np.int64)
        self.nodes[: len(nodes), 0] = (nodes[:, 0] & 0xFFFFFFFF) | (nodes[:, 1] << 32)
        self.nodes[: len(nodes), 1:] = nodes[:, 2:]
        self.tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        self.q = spq_query(self.nodes.ctypes.data_as(C.POINTER(spq_node)), len(nodes),
                           self.tokens.ctypes.data_as(_I32P), len(self.tokens))


class _FlatQueryBuf(_QueryBuf):
    """The common ⋈[prefix?, ⊕[f…]?, cross] tree encoded straight into the ABI layout (the same
    nodes as inputs.query_to_tree builds for a non-nested query, without its intermediate arrays)."""

    def __init__(self, q):  # noqa: super().__init__ not called: the arrays are built here
        parts = ([q.prefix] if len(q.prefix) else []) + list(q.fragments) + [q.cross]
        lens = np.fromiter((len(p) for p in parts), dtype=np.int64, count=len(parts))
        offs = np.zeros(len(parts), np.int64)
        np.cumsum(lens[:-1], out=offs[1:])
        nf = len(q.fragments)
        n_top = (1 if len(q.prefix) else 0) + (1 if nf else 0) + 1
        nodes = np.zeros((1 + len(parts) + (1 if nf else 0), 3), np.int64)
        nodes[0, 0] = _inputs.OP_CROSS | (n_top << 32)
        r, k = 1, 0
        if len(q.prefix):
            nodes[r] = (_inputs.OP_TOKENS, offs[0], lens[0])
            r, k = r + 1, 1
        if nf:
            nodes[r, 0] = _inputs.OP_PLUS | (nf << 32)
            r += 1
            nodes[r:r + nf, 0] = _inputs.OP_TOKENS
            nodes[r:r + nf, 1] = offs[k:k + nf]
            nodes[r:r + nf, 2] = lens[k:k + nf]
            r, k = r + nf, k + nf
        nodes[r] = (_inputs.OP_TOKENS, offs[k], lens[k])
        self.nodes = nodes
        self.tokens = np.ascontiguousarray(np.concatenate(parts), dtype=np.int32)
        self.q = spq_query(self.nodes.ctypes.data_as(C.POINTER(spq_node)), len(nodes),
                           self.tokens.ctypes.data_as(_I32P), len(self.tokens))


def to_query(q) -> _QueryBuf:
    if isinstance(q, _inputs.SpanQuery):
        if not q.nest or len(q.fragments) < 3:
            return _FlatQueryBuf(q)
        return _QueryBuf(*_inputs.query_to_tree(q))
    nodes, toks = q
    return _QueryBuf(nodes, toks)


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class Plan:
    def __init__(self, ctx: "Context", handle: int):
        self.ctx = ctx
        self.handle = handle
        self.released = False
        v = spq_plan_view()
        _check(lib().spq_plan_view_get(self.handle, C.byref(v)))
        self.n_jobs, self.n_queries = v.n_jobs, v.n_queries

    def view(self) -> Dict[str, object]:
        v = spq_plan_view()
        _check(lib().spq_plan_view_get(self.handle, C.byref(v)))
        ns, nb, nq = v.n_segments, v.n_blocks_total, v.n_queries
        out = dict(
            n_queries=nq, n_segments=ns, n_jobs=v.n_jobs,
            seg_query=_arr(v.seg_query, ns, np.int32), seg_kind=_arr(v.seg_kind, ns, np.int32),
            seg_frag_idx=_arr(v.seg_frag_idx, ns, np.int32),
            seg_tok_len=_arr(v.seg_tok_len, ns, np.int32), seg_pos0=_arr(v.seg_pos0, ns, np.int32),
            seg_hit=_arr(v.seg_hit, ns, np.int32),
            seg_compute_begin=_arr(v.seg_compute_begin, ns, np.int32),
            seg_block_off=_arr(v.seg_block_off, ns, np.int32),
            seg_n_blocks=_arr(v.seg_n_blocks, ns, np.int32),
            blocks=_arr(v.blocks, nb, np.int32), block_write=_arr(v.block_write, nb, np.uint8),
            digests=_arr(v.digests, nb * 16, np.uint8).reshape(nb, 16),
            join_digests=_arr(v.join_digests, nq * 16, np.uint8).reshape(nq, 16),
            jobs=_arr(v.jobs, v.n_jobs, np.int32),
            job_row_off=_arr(v.job_row_off, v.n_jobs + 1, np.int64),
            prefill_pos=_arr(v.prefill_pos, v.n_prefill_rows, np.int32),
            prefill_slot=_arr(v.prefill_slot, v.n_prefill_rows, np.int64),
            query_join_row_off=_arr(v.query_join_row_off, nq + 1, np.int64),
            join_pos=_arr(v.join_pos, v.n_join_rows, np.int32),
            join_slot=_arr(v.join_slot, v.n_join_rows, np.int64),
            pad_slots=_arr(v.pad_slots, v.n_pad_slots, np.int64),
            prefill_flops=v.prefill_flops, join_flops=v.join_flops,
            prefill_kv_bytes=v.prefill_kv_bytes, join_kv_bytes=v.join_kv_bytes,
            n_join_queries=v.n_join_queries, world_size=v.world_size,
        )
        w = v.world_size
        so, ro = _arr(v.send_off, w + 1, np.int64), _arr(v.recv_off, w + 1, np.int64)
        sb, rb = _arr(v.send_blocks, int(so[-1]), np.int32), _arr(v.recv_blocks, int(ro[-1]), np.int32)
        out["send"] = {p: sb[so[p]:so[p + 1]] for p in range(w) if so[p + 1] > so[p]}
        out["recv"] = {p: rb[ro[p]:ro[p + 1]] for p in range(w) if ro[p + 1] > ro[p]}
        out["tasks"] = [tuple(int(x) for x in r) for r in _arr(v.tasks, 6 * v.n_tasks, np.int32).reshape(-1, 6)]
        xo = _arr(v.xq_off, w + 1, np.int32) if v.xq_off else np.zeros(w + 1, np.int32)
        xqq = _arr(v.xq_queries, int(xo[-1]), np.int32)
        out["xq"] = {p: xqq[xo[p]:xo[p + 1]].tolist() for p in range(w) if xo[p + 1] > xo[p]}
        # replica need flags (R38): per owner peer (home side) / candidate counts per home peer
        co = _arr(v.cand_recv_off, w + 1, np.int64) if v.cand_recv_off else np.zeros(w + 1, np.int64)
        cn = _arr(v.cand_recv_need, int(co[-1]), np.uint8)
        out["need"] = {p: cn[co[p]:co[p + 1]] for p in range(w) if co[p + 1] > co[p]}
        cs = _arr(v.cand_send_off, w + 1, np.int64) if v.cand_send_off else np.zeros(w + 1, np.int64)
        out["n_cand_send"] = [int(cs[p + 1] - cs[p]) for p in range(w)]
        return out

    def exchange_set_need(self, peer, need, stream=None):
        """Owner side (R38): keep in the send list to `peer` only the fragments it flagged."""
        flags = np.ascontiguousarray(np.asarray(need, dtype=np.uint8))
        _check(lib().spq_exchange_set_need(self.ctx.handle, self.handle, int(peer),
                                           flags.ctypes.data_as(_U8P), int(flags.size),
                                           _stream_ptr(stream, self.ctx.device)))

    def exchange_pack(self, layer, peer, buf, stream=None):
        """Gather this plan's send blocks for `peer` (one layer) into buf [n, 2, Hkv, bs, d]."""
        _check(lib().spq_exchange_pack(self.ctx.handle, self.handle, layer, peer, _ptr(buf),
                                       _stream_ptr(stream, self.ctx.device)))

    def exchange_unpack(self, layer, peer, buf, stream=None):
        """Scatter buf [n, 2, Hkv, bs, d] into this plan's recv blocks from `peer` (one layer)."""
        _check(lib().spq_exchange_unpack(self.ctx.handle, self.handle, layer, peer, _ptr(buf),
                                         _stream_ptr(stream, self.ctx.device)))

    def prefill(self, layer, q, k, v, o, lse=None, jobs=None, stream=None):
        a, b = (0, self.n_jobs) if jobs is None else jobs
        _check(lib().spq_prefill_jobs(self.ctx.handle, self.handle, layer, a, b, _ptr(q), _ptr(k),
                                      _ptr(v), _ptr(o), _ptr(lse), _stream_ptr(stream, self.ctx.device)))

    def join(self, layer, q, k, v, o, lse=None, queries=None, stream=None):
        a, b = (0, self.n_queries) if queries is None else queries
        _check(lib().spq_join(self.ctx.handle, self.handle, layer, a, b, _ptr(q), _ptr(k), _ptr(v),
                              _ptr(o), _ptr(lse), _stream_ptr(stream, self.ctx.device)))

    def join_phase(self, layer, phase, q, k, v, o, lse=None, stream=None):
        """Phase 0 / 1 of the join of all home queries (W > 1: around the fragment-KV exchange)."""
        _check(lib().spq_join_phase(self.ctx.handle, self.handle, layer, phase, _ptr(q), _ptr(k), _ptr(v),
                                    _ptr(o), _ptr(lse), _stream_ptr(stream, self.ctx.device)))

    def decode_reserve(self, max_new: int):
        """Reserve generation blocks for max_new tokens per home query (rows in query order)."""
        _check(lib().spq_decode_reserve(self.ctx.handle, self.handle, int(max_new)))
        self.max_new = int(max_new)

    def decode_step(self, layer, t, q, k, v, o, lse=None, stream=None):
        """Generated token t of every home query: K1 of its k/v, then its row over the whole span."""
        _check(lib().spq_decode_step(self.ctx.handle, self.handle, layer, t, _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                     _ptr(lse), _stream_ptr(stream, self.ctx.device)))

    def commit_span(self, query: int, gen_tokens, crop: bool = False) -> int:
        """Plus distribution: index the query's (cross ‖ generated) tokens as a cached fragment;
        returns the tokens committed (the trailing partial block is dropped with crop=True)."""
        g = np.ascontiguousarray(gen_tokens, dtype=np.int32)
        n = C.c_int32()
        _check(lib().spq_commit_span(self.ctx.handle, self.handle, int(query), g.ctypes.data if len(g) else None,
                                     len(g), 1 if crop else 0, C.byref(n)))
        return n.value

    def commit_output(self, query: int, gen_tokens, stream=None) -> int:
        """Commit only the query's generated tokens as a span (K re-encoded to 0.. by CIDRA)."""
        g = np.ascontiguousarray(gen_tokens, dtype=np.int32)
        n = C.c_int32()
        _check(lib().spq_commit_output(self.ctx.handle, self.handle, int(query), g.ctypes.data, len(g),
                                       _stream_ptr(stream, self.ctx.device), C.byref(n)))
        return n.value

    # ---- owner-side split join (W > 1, split_join=True)
    def split_pack_q(self, q_join, qsend, stream=None):
        _check(lib().spq_split_pack_q(self.ctx.handle, self.handle, _ptr(q_join), _ptr(qsend),
                                      _stream_ptr(stream, self.ctx.device)))

    def split_task_join(self, layer, qrecv, part_o, part_lse, stream=None):
        _check(lib().spq_split_task_join(self.ctx.handle, self.handle, layer, _ptr(qrecv), _ptr(part_o),
                                         _ptr(part_lse), _stream_ptr(stream, self.ctx.device)))

    def split_join_local(self, layer, q, k, v, stream=None):
        _check(lib().spq_split_join_local(self.ctx.handle, self.handle, layer, _ptr(q), _ptr(k), _ptr(v),
                                          _stream_ptr(stream, self.ctx.device)))

    def split_merge(self, part_o_recv, part_lse_recv, o, lse=None, stream=None):
        _check(lib().spq_split_merge(self.ctx.handle, self.handle, _ptr(part_o_recv), _ptr(part_lse_recv), _ptr(o),
                                     _ptr(lse), _stream_ptr(stream, self.ctx.device)))

    def release(self, stream=None):
        if not self.released:
            _check(lib().spq_plan_release(self.ctx.handle, self.handle, _stream_ptr(stream, self.ctx.device)))
            self.released = True


class Context:
    """One ctx per GPU (or host-only with device=-1: planner and store only).

    For a GPU ctx the KV pools are allocated here with torch (caller-owned memory in ABI terms):
    k_pool/v_pool [L, num_blocks, Hkv, bs, d].
    """

    def __init__(self, shape: _inputs.Shape, num_blocks: int, device: int = 0,
                 max_position: int = 1 << 15, pools=None, out_dtype: Optional[str] = None,
                 rank: int = 0, world_size: int = 1, split_join: bool = False):
        self.shape = shape
        self.device = device
        self.num_blocks = num_blocks
        self.k_pool = self.v_pool = None
        self.out_dtype = out_dtype or shape.dtype
        self.rank, self.world_size = rank, world_size
        if device >= 0:
            import torch

            dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
            if pools is None:
                sz = (shape.layers, num_blocks, shape.hkv, shape.block_size, shape.d)
                self.k_pool = torch.zeros(sz, dtype=dt, device=f"cuda:{device}")
                self.v_pool = torch.zeros(sz, dtype=dt, device=f"cuda:{device}")
            else:
                self.k_pool, self.v_pool = pools
        cfg = spq_config(shape.hq, shape.hkv, shape.d, shape.layers, shape.block_size, num_blocks,
                         BF16 if shape.dtype == "bf16" else FP32, float(shape.rope_base),
                         int(max_position), int(shape.model_salt), _ptr(self.k_pool),
                         _ptr(self.v_pool), device, int(rank), int(world_size),
                         BF16 if self.out_dtype == "bf16" else FP32, 1 if split_join else 0)
        h = C.c_void_p()
        _check(lib().spq_create(C.byref(cfg), C.byref(h)))
        self.handle = h.value

    def close(self):
        if self.handle:
            lib().spq_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def plan(self, queries: Sequence, stream=None) -> Plan:
        bufs = [to_query(q) for q in queries]
        arr = (spq_query * len(bufs))(*[b.q for b in bufs])
        h = C.c_void_p()
        _check(lib().spq_plan_create(self.handle, arr, len(bufs), _stream_ptr(stream, self.device), C.byref(h)))
        return Plan(self, h.value)

    def block_hashes(self, query) -> np.ndarray:
        b = to_query(query)
        n = C.c_int64()
        cap = 1 << 16
        out = np.zeros((cap, 16), np.uint8)
        _check(lib().spq_block_hashes(self.handle, C.byref(b.q), out.ctypes.data, cap, C.byref(n)))
        return out[: n.value].copy()

    def lookup(self, digests: np.ndarray) -> np.ndarray:
        d = np.ascontiguousarray(digests, dtype=np.uint8).reshape(-1, 16)
        ids = np.zeros(len(d), np.int32)
        _check(lib().spq_lookup(self.handle, d.ctypes.data, len(d), ids.ctypes.data))
        return ids

    def insert(self, digests: np.ndarray, ntok: Sequence[int]) -> np.ndarray:
        d = np.ascontiguousarray(digests, dtype=np.uint8).reshape(-1, 16)
        nt = np.ascontiguousarray(ntok, dtype=np.int32)
        ids = np.zeros(len(d), np.int32)
        _check(lib().spq_insert(self.handle, d.ctypes.data, nt.ctypes.data, len(d), ids.ctypes.data))
        return ids

    def read_blocks(self, layer: int, block_ids, stream=None):
        """K and V pages of the given blocks of one layer: two device tensors [n, Hkv, bs, d]."""
        import torch

        ids = np.ascontiguousarray(block_ids, dtype=np.int32)
        s = self.shape
        dt = torch.bfloat16 if s.dtype == "bf16" else torch.float32
        k = torch.empty((len(ids), s.hkv, s.block_size, s.d), dtype=dt, device=f"cuda:{self.device}")
        v = torch.empty_like(k)
        _check(lib().spq_read_blocks(self.handle, layer, ids.ctypes.data, len(ids), _ptr(k), _ptr(v),
                                     _stream_ptr(stream, self.device)))
        return k, v

    @staticmethod
    def _moves(src, dst, delta):
        a = [np.ascontiguousarray(x, dtype=np.int32) for x in (src, dst, delta)]
        if not (len(a[0]) == len(a[1]) == len(a[2])):
            raise ValueError("src, dst, delta must have the same length")
        return a

    def reposition(self, src, dst, delta, layers=None, stream=None) -> Dict[str, int]:
        """CIDRA: block dst[i] <- block src[i] with K re-encoded delta[i] positions
        later, V copied, in place on the ctx's pools for layers [begin, end). Returns the stats."""
        s_, d_, dl = self._moves(src, dst, delta)
        lb, le = layers if layers is not None else (0, self.shape.layers)
        st = spq_cidra_stats()
        _check(lib().spq_reposition(self.handle, s_.ctypes.data, d_.ctypes.data, dl.ctypes.data, len(s_), lb, le,
                                    _stream_ptr(stream, self.device), C.byref(st)))
        return {n: getattr(st, n) for n, _ in spq_cidra_stats._fields_}

    def cidra_schedule(self, src, dst, delta):
        """The in-place schedule spq_reposition would run: (ops [n_ops, 4] = dst, src, delta, mode;
        comp_off [n_comp + 1]; stats)."""
        s_, d_, dl = self._moves(src, dst, delta)
        cap = 2 * len(s_) + 8
        ops = np.zeros((cap, 4), np.int32)
        off = np.zeros(len(s_) + 2, np.int32)
        n_ops, n_comp = C.c_int64(), C.c_int64()
        st = spq_cidra_stats()
        _check(lib().spq_cidra_schedule(self.handle, s_.ctypes.data, d_.ctypes.data, dl.ctypes.data, len(s_),
                                        ops.ctypes.data, cap, C.byref(n_ops), off.ctypes.data, len(off),
                                        C.byref(n_comp), C.byref(st)))
        return (ops[: n_ops.value].copy(), off[: n_comp.value + 1].copy(),
                {n: getattr(st, n) for n, _ in spq_cidra_stats._fields_})

    def stats(self) -> Dict[str, int]:
        s = spq_stats()
        _check(lib().spq_get_stats(self.handle, C.byref(s)))
        return {n: getattr(s, n) for n, _ in spq_stats._fields_}

    def evict_all(self):
        _check(lib().spq_evict_all(self.handle))

    def bulk_order(self, queries: Sequence, window_blocks: int = 0) -> np.ndarray:
        """spq_bulk_order: the greedy locality order of a bulk of queries (a permutation)."""
        bufs = [to_query(q) for q in queries]
        arr = (spq_query * max(1, len(bufs)))(*[b.q for b in bufs])
        order = np.zeros(len(bufs), np.int32)
        _check(lib().spq_bulk_order(self.handle, arr, len(bufs), int(window_blocks), order.ctypes.data))
        return order

    def set_option(self, key: int, value: float):
        """spq_set_option (OPT_EXP2, OPT_RESCALE_THRESHOLD, OPT_PDL, OPT_HASH_SCALAR, OPT_PAIR)."""
        _check(lib().spq_set_option(self.handle, int(key), float(value)))

    def set_trace(self, buf, mode: int = 0):
        """Profiling builds only (SPANQ_LIB=.../libspanq_prof.so): CTA-0 timeline buffer + mode."""
        _check(lib().spq_set_trace(self.handle, _ptr(buf), int(mode)))

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().spq_launch_count(self.handle, C.byref(n)))
        return n.value

    def set_timing(self, on: bool):
        _check(lib().spq_set_timing(self.handle, 1 if on else 0))

    def last_attn_ms(self):
        a, b = C.c_float(), C.c_float()
        _check(lib().spq_last_attn_ms(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value


def reduce_tree(n: int, k: int):
    """spq_reduce_tree: the k-ary judge reduction schedule. Returns (plies, children) where
    plies[p] = the judge ids of ply p (judge j is item n + j) and children[j] = the items judge j
    reads (candidates 0..n-1, judges n..)."""
    np_, nj = C.c_int32(), C.c_int32()
    cap = 2 * n + 8
    po, co, ch = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(2 * cap, np.int32)
    _check(lib().spq_reduce_tree(int(n), int(k), po.ctypes.data, cap, co.ctypes.data, ch.ctypes.data, cap,
                                 C.byref(np_), C.byref(nj)))
    plies = [list(range(po[p], po[p + 1])) for p in range(np_.value)]
    children = [ch[co[j]:co[j + 1]].tolist() for j in range(nj.value)]
    return plies, children
