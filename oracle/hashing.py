"""Block digest chains — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Paper: vLLM's block hash depends on the previous block's hash (§2, P:97-98,
"The hash code for a block B_i … depends on the hash code of block B_{i−1}"); span queries
"suspend the accumulation logic" at a span start and "resume" it at the span end (§5.4).
The paper names no hash function or byte layout; this file writes out the contract of
SURVEY.md §8(c) (readings R5-R7 in DESIGN.md) with CPython's hashlib BLAKE2b, digest_size 16:

  ROOT = B("SPQv1" ‖ u32 Hq ‖ u32 Hkv ‖ u32 d ‖ u32 bs ‖ f64 rope_base ‖ u64 model_salt)
  prefix  h_i = B('P' ‖ h_{i−1} ‖ u32 n ‖ n×u32 tok),  h_{−1} = ROOT
  fragment s_i = B('F' ‖ s_{i−1} ‖ u32 n ‖ tok…),       s_{−1} = ROOT   (restart = suspension)
  join    J   = B('J' ‖ h_last or ROOT ‖ u32 n_frag ‖ s_last(f_1) ‖ … ‖ s_last(f_n))  (⊕ order)
  cross   x_i = B('X' ‖ x_{i−1} ‖ u32 n ‖ tok…),        x_{−1} = J

All integers little-endian; ``n`` is the number of tokens actually in the block (< bs for a
tail).
"""
from __future__ import annotations

import hashlib
import struct
from typing import List, Sequence

import numpy as np


def b2(data: bytes) -> bytes:
    return hashlib.blake2b(data, digest_size=16).digest()


def root_digest(hq: int, hkv: int, d: int, bs: int, rope_base: float, model_salt: int) -> bytes:
    return b2(b"SPQv1" + struct.pack("<IIIIdQ", hq, hkv, d, bs, float(rope_base), model_salt))


def _blocks(tokens: np.ndarray, bs: int) -> List[np.ndarray]:
    t = np.asarray(tokens, dtype=np.int64)
    return [t[i : i + bs] for i in range(0, len(t), bs)]


def _chain(tag: bytes, seed: bytes, tokens: np.ndarray, bs: int) -> List[bytes]:
    out = []
    prev = seed
    for blk in _blocks(tokens, bs):
        payload = tag + prev + struct.pack("<I", len(blk)) + b"".join(
            struct.pack("<I", int(t) & 0xFFFFFFFF) for t in blk
        )
        prev = b2(payload)
        out.append(prev)
    return out


def prefix_chain(tokens: np.ndarray, bs: int, root: bytes) -> List[bytes]:
    """Chained digests of the ordered prefix."""
    return _chain(b"P", root, tokens, bs)


def fragment_chain(tokens: np.ndarray, bs: int, root: bytes) -> List[bytes]:
    """Chain restarted from ROOT at the fragment start: accumulation suspended."""
    return _chain(b"F", root, tokens, bs)


def join_fold(h_last: bytes, frag_lasts: Sequence[bytes]) -> bytes:
    """Resume after the ⊕ span: ordered fold of the fragment identities (reading R6)."""
    return b2(b"J" + h_last + struct.pack("<I", len(frag_lasts)) + b"".join(frag_lasts))


def cross_chain(tokens: np.ndarray, bs: int, j: bytes) -> List[bytes]:
    return _chain(b"X", j, tokens, bs)


def owner_rank(frag_last: bytes, world_size: int) -> int:
    """Fragment owner for multi-GPU partitioning: u64le(s_last[0:8]) mod W."""
    return struct.unpack("<Q", frag_last[:8])[0] % world_size
