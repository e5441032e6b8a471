"""Content-hash KV block store and planner mirror — TEST INFRASTRUCTURE ONLY (oracle/__init__).

What it follows, step by step:
  * blocks of ``bs`` tokens are the unit of insert/lookup/evict (§2);
  * chained digests, prefix scan that "stops scanning for cache hits after the first miss"
    (P:97-98); the trailing partial block of an ordered span is not cached;
  * hash accumulation suspended inside ⊕ fragments so a fragment hits wherever it appears
    (§5.4), fragments are "prepared" independently of context (§5.1 footnote);
  * hit rate = hit tokens / input tokens (fig. 2 caption);
  * the readings the paper leaves open (restated in DESIGN.md):
      R8  fragment tail block stored with its true n, pad slots zeroed;
      R9  prefix: full blocks prefix-scanned and inserted, partial tail plan-private;
          cross: always computed; full blocks inserted under the X chain (a resident X
          digest is referenced, not rewritten), partial tail plan-private;
      R10 fragment hit is all-or-nothing; on a miss the whole fragment is recomputed and
          its resident blocks are read but not rewritten (slot −1);
      R11 a fragment repeated in one plan is prefilled once, at its first occurrence;
      R12 allocation takes the lowest free block id, in the order queries → prefix blocks →
          fragments in ⊕ order → cross blocks;
      R13 with no free block, evict the unpinned resident block with the smallest
          (last-use plan number, block id); none → ENOMEM and the plan is rolled back.

The plan view produced here is compared bit-for-bit with the C++ planner's (spq_plan_view).
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import hashing

KIND_PREFIX, KIND_FRAG, KIND_CROSS = 0, 1, 2


class OracleENOMEM(RuntimeError):
    pass


@dataclass
class Segment:
    query: int
    kind: int
    frag_idx: int  # -1 for prefix / cross
    tok_len: int
    pos0: int  # global position of the first token in the query (Δ for fragments)
    blocks: List[int]
    digests: List[bytes]
    hit: int  # prefix: #hit blocks (prefix scan); fragment: 1 if all-or-nothing hit; cross: 0
    compute_begin: int  # first row whose attention is computed (tok_len = none)
    write: List[bool]  # per block: newly written by this plan


@dataclass
class PlanView:
    segments: List[Segment]
    join_digests: List[bytes]
    prefill_pos: np.ndarray  # int32, packed job order
    prefill_slot: np.ndarray  # int64, -1 = not written
    prefill_seg: np.ndarray  # int32 segment index per packed row
    join_pos: np.ndarray
    join_slot: np.ndarray
    join_seg: np.ndarray
    pad_slots: np.ndarray  # int64
    jobs: List[int]  # segment indices of prefill jobs, plan order
    stats: Dict[str, int]
    pinned: List[int]
    private: List[int]
    # multi-rank exchange: blocks this rank sends to / receives from each peer,
    # fragments in first-occurrence order, each fragment's blocks in order
    send: Dict[int, List[int]] = field(default_factory=dict)
    recv: Dict[int, List[int]] = field(default_factory=dict)
    n_join_queries: int = 0
    # owner-side split join (split=True): tasks this rank computes for other
    # homes, (home, query) order: (query, home, n_rows, pos0 of the cross rows, first and end
    # segment index of the query's fragments owned here); per peer owner, the home queries whose
    # cross Q this rank sends to it and whose partial (O, LSE) comes back (query order)
    tasks: List[Tuple[int, int, int, int, int, int]] = field(default_factory=list)
    xq: Dict[int, List[int]] = field(default_factory=dict)
    # digest-keyed replicas (R38): home side, per owner peer, one flag per remote fragment its joins
    # read (first-occurrence order; 1 = its KV must be sent, 0 = a replica is resident); owner side,
    # per home peer, the candidate fragments' block lists in the same order (`send` holds them all
    # until `select_send` narrows it by the home's flags)
    need: Dict[int, List[int]] = field(default_factory=dict)
    send_candidates: Dict[int, List[List[int]]] = field(default_factory=dict)


class Store:
    def __init__(self, num_blocks: int, hq: int, hkv: int, d: int, bs: int,
                 rope_base: float = 10000.0, model_salt: int = 0):
        self.num_blocks = num_blocks
        self.bs = bs
        self.root = hashing.root_digest(hq, hkv, d, bs, rope_base, model_salt)
        self.index: Dict[bytes, int] = {}
        self.meta: Dict[int, Tuple[bytes, int, int]] = {}  # id -> (digest, ntok, last_use)
        self.free = set(range(num_blocks))
        self.pins = [0] * num_blocks
        self.plan_no = 0
        self.stats = dict(lookups=0, hit_blocks=0, miss_blocks=0, hit_tokens=0,
                          input_tokens=0, evictions=0, inserted_blocks=0)

    # -------------------------------------------------------------- primitives
    def _alloc(self) -> int:
        if self.free:
            b = min(self.free)
            self.free.remove(b)
            return b
        victims = [b for b in self.meta if self.pins[b] == 0]
        if not victims:
            raise OracleENOMEM("no free or evictable block")
        b = min(victims, key=lambda x: (self.meta[x][2], x))
        dig = self.meta[b][0]
        del self.index[dig]
        del self.meta[b]
        self.stats["evictions"] += 1
        return b

    def lookup(self, digests: Sequence[bytes]) -> List[int]:
        """Low-level lookup (SPEC kv_cache.lookup S:301): block id or -1 per digest, no scan."""
        return [self.index.get(d, -1) for d in digests]

    def insert(self, digests: Sequence[bytes], ntok: Sequence[int]) -> List[int]:
        """Low-level insert (SPEC kv_cache.insert S:310): resident digests keep their block;
        others get a new unpinned block (lowest free id, else LRU eviction). All-or-nothing."""
        saved = copy.deepcopy((self.index, self.meta, self.free, self.stats))
        out = []
        try:
            for dig, n in zip(digests, ntok):
                if dig in self.index:
                    out.append(self.index[dig])
                    continue
                b = self._alloc()
                self.index[dig] = b
                self.meta[b] = (dig, int(n), self.plan_no)
                self.stats["inserted_blocks"] += 1
                out.append(b)
        except OracleENOMEM:
            (self.index, self.meta, self.free, self.stats) = saved
            raise
        return out

    # -------------------------------------------------------------- planner
    def plan(self, queries: Sequence[Tuple[np.ndarray, List[np.ndarray], np.ndarray]],
             rank: int = 0, world: int = 1, split: bool = False) -> PlanView:
        """Plan a batch. With world > 1 this is rank `rank`'s share: query q is
        homed on q mod W (its prefix, join and cross run there), fragment f is owned by
        u64le(s_last[0:8]) mod W (it is prefilled and cached only there); a home rank receives
        remote-owned fragments, in first-occurrence order, into blocks indexed under their
        digests (R38 replicas: a later plan here hits them and nothing moves).

        split=True (owner-side split join; §4.3, parallel
        sub-trees): no KV moves. An owner keeps each owned fragment's segment at its place in the
        query (pos0 = Δ_f) and computes the home query's cross rows over its owned fragments as a
        task; the home rank keeps only its local segments and merges the owners' partials."""
        saved = copy.deepcopy((self.index, self.meta, self.free, self.pins, self.plan_no,
                               self.stats))
        try:
            return self._plan(queries, rank, world, split)
        except OracleENOMEM:
            (self.index, self.meta, self.free, self.pins, self.plan_no, self.stats) = saved
            raise

    def _plan(self, queries, rank: int = 0, world: int = 1, split: bool = False) -> PlanView:
        bs = self.bs
        self.plan_no += 1
        p = self.plan_no
        pinned: List[int] = []
        pinned_set = set()
        private: List[int] = []
        pad_slots: List[int] = []

        def pin(b):
            if b not in pinned_set:
                pinned_set.add(b)
                pinned.append(b)
                self.pins[b] += 1

        def touch(b):
            dig, n, _ = self.meta[b]
            self.meta[b] = (dig, n, p)

        def insert_new(dig, ntok) -> int:
            b = self._alloc()
            self.index[dig] = b
            self.meta[b] = (dig, ntok, p)
            self.stats["inserted_blocks"] += 1
            pin(b)
            if ntok < bs:
                pad_slots.extend(range(b * bs + ntok, b * bs + bs))
            return b

        # R38: blocks whose KV this plan receives (digest-keyed replicas). An owned fragment of the
        # same plan that shares one (common token prefix) recomputes and writes it: the exchange
        # fills it only after the prefill and after the owner's own sends are packed
        pending = set()

        def insert_replica(dig, ntok) -> int:
            b = self._alloc()
            self.index[dig] = b
            self.meta[b] = (dig, ntok, p)
            self.stats["inserted_blocks"] += 1
            pin(b)
            pending.add(b)  # no pad slots: the owner's pages carry their zeroed pads
            return b

        def new_private(ntok, pad=True) -> int:
            b = self._alloc()
            private.append(b)
            pin(b)
            if pad:
                pad_slots.extend(range(b * bs + ntok, b * bs + bs))
            return b

        send: Dict[int, List[bytes]] = {}
        recv: Dict[int, List[bytes]] = {}
        owned_blocks: Dict[bytes, List[int]] = {}
        recv_blocks: Dict[bytes, List[int]] = {}
        recv_hit: Dict[bytes, bool] = {}
        cand_recv: Dict[int, List[bytes]] = {}

        segs: List[Segment] = []
        joins: List[bytes] = []
        n_home = 0
        tasks: List[Tuple[int, int, int, int, int, int]] = []
        xq: Dict[int, List[int]] = {}
        for qi, (prefix, frags, cross) in enumerate(queries):
            prefix = np.asarray(prefix)
            cross = np.asarray(cross)
            home = qi % world
            is_home = home == rank
            h = hashing.prefix_chain(prefix, bs, self.root)
            if not is_home:
                joins.append(bytes(16))  # join digests are per query; zero where homed elsewhere
                # only the fragments this rank owns: prefill/cache them and send them home (split:
                # keep them at their offset in the query for this rank's task)
                first = len(segs)
                off = len(prefix)
                for fi, f in enumerate(frags):
                    sf = hashing.fragment_chain(f, bs, self.root)
                    delta = off
                    off += len(f)
                    if hashing.owner_rank(sf[-1], world) != rank:
                        continue
                    seg = self._frag_segment(qi, fi, f, sf, delta if split else 0, touch, pin, insert_new,
                                             pending)
                    segs.append(seg)
                    owned_blocks.setdefault(sf[-1], seg.blocks)
                    if split:
                        continue
                    lst = send.setdefault(home, [])
                    if sf[-1] not in lst:
                        lst.append(sf[-1])
                if split and len(segs) > first:
                    tasks.append((qi, home, len(cross), off, first, len(segs)))
                continue
            n_home += 1
            self.stats["input_tokens"] += len(prefix) + sum(len(f) for f in frags) + len(cross)
            # ---- prefix: chained digests, prefix scan
            blocks, write = [], []
            hit_run, n_hit = True, 0
            for i, dig in enumerate(h):
                ntok = min(bs, len(prefix) - i * bs)
                full = ntok == bs
                self.stats["lookups"] += 1 if full else 0
                if full and dig in self.index:
                    b = self.index[dig]
                    touch(b)
                    pin(b)
                    blocks.append(b)
                    write.append(False)
                    if hit_run:
                        n_hit += 1
                        self.stats["hit_blocks"] += 1
                        self.stats["hit_tokens"] += bs
                    else:  # resident after the first miss: read, not rewritten, recomputed
                        self.stats["miss_blocks"] += 1
                    continue
                if full:
                    self.stats["miss_blocks"] += 1
                    hit_run = False
                    blocks.append(insert_new(dig, bs))
                else:
                    hit_run = False
                    blocks.append(new_private(ntok))
                write.append(True)
            if len(prefix):
                segs.append(Segment(qi, KIND_PREFIX, -1, len(prefix), 0, blocks, h, n_hit,
                                    min(n_hit * bs, len(prefix)), write))
            h_last = h[-1] if h else self.root
            # ---- fragments: suspended chains, all-or-nothing (R10, R11)
            off = len(prefix)
            lasts = []
            for fi, f in enumerate(frags):
                sf = hashing.fragment_chain(f, bs, self.root)
                lasts.append(sf[-1])
                owner = hashing.owner_rank(sf[-1], world)
                if owner == rank:
                    seg = self._frag_segment(qi, fi, f, sf, off, touch, pin, insert_new, pending)
                    owned_blocks.setdefault(sf[-1], seg.blocks)
                elif split:  # computed by its owner (a task there); this rank merges its partial
                    if qi not in xq.setdefault(owner, []):
                        xq[owner].append(qi)
                    off += len(f)
                    continue
                else:
                    # remote-owned (R38): all-or-nothing lookup of a replica kept from an earlier
                    # exchange; a miss is received whole into its resident blocks (pinned first,
                    # R24) and newly indexed ones; no prefill here
                    if sf[-1] not in recv_blocks:
                        self.stats["lookups"] += 1
                        resident = [self.index.get(dig, -1) for dig in sf]
                        for b in resident:
                            if b >= 0:
                                touch(b)
                                pin(b)
                        hit = all(b >= 0 for b in resident)
                        if hit:
                            self.stats["hit_blocks"] += len(sf)
                            self.stats["hit_tokens"] += len(f)
                        else:
                            self.stats["miss_blocks"] += len(sf)
                            resident = [b if b >= 0 else insert_replica(dig, min(bs, len(f) - i * bs))
                                        for i, (b, dig) in enumerate(zip(resident, sf))]
                            recv.setdefault(owner, []).append(sf[-1])
                        recv_blocks[sf[-1]] = resident
                        recv_hit[sf[-1]] = hit
                        cand_recv.setdefault(owner, []).append(sf[-1])
                    seg = Segment(qi, KIND_FRAG, fi, len(f), off, recv_blocks[sf[-1]], sf,
                                  int(recv_hit[sf[-1]]), len(f), [False] * len(sf))
                segs.append(seg)
                off += len(f)
            j = hashing.join_fold(h_last, lasts)
            joins.append(j)
            # ---- cross: always computed (R9)
            x = hashing.cross_chain(cross, bs, j)
            blocks, write = [], []
            for i, dig in enumerate(x):
                ntok = min(bs, len(cross) - i * bs)
                if ntok == bs and dig in self.index:
                    b = self.index[dig]
                    touch(b)
                    pin(b)
                    blocks.append(b)
                    write.append(False)
                elif ntok == bs:
                    blocks.append(insert_new(dig, bs))
                    write.append(True)
                else:
                    blocks.append(new_private(ntok))
                    write.append(True)
            segs.append(Segment(qi, KIND_CROSS, -1, len(cross), off, blocks, x, 0, 0, write))

        # ---- packed rows
        def rows(seg: Segment, begin: int):
            pos, slot = [], []
            for t in range(begin, seg.tok_len):
                b, o = divmod(t, bs)
                pos.append(seg.pos0 + t if seg.kind == KIND_CROSS else t)
                slot.append(seg.blocks[b] * bs + o if seg.write[b] else -1)
            return pos, slot

        jobs = [i for i, s in enumerate(segs) if s.kind != KIND_CROSS and s.compute_begin < s.tok_len]
        pp, ps, pg = [], [], []
        for i in jobs:
            a, b = rows(segs[i], segs[i].compute_begin)
            pp += a
            ps += b
            pg += [i] * len(a)
        jp, js, jg = [], [], []
        for i, s in enumerate(segs):
            if s.kind == KIND_CROSS:
                a, b = rows(s, 0)
                jp += a
                js += b
                jg += [i] * len(a)
        send_b = {d: [b for dig in lst for b in owned_blocks[dig]] for d, lst in send.items()}
        recv_b = {o: [b for dig in lst for b in recv_blocks[dig]] for o, lst in recv.items()}
        view = PlanView(segs, joins, np.asarray(pp, np.int32), np.asarray(ps, np.int64),
                        np.asarray(pg, np.int32), np.asarray(jp, np.int32),
                        np.asarray(js, np.int64), np.asarray(jg, np.int32),
                        np.asarray(pad_slots, np.int64), jobs, dict(self.stats), pinned, private,
                        send_b, recv_b, n_home, sorted(tasks, key=lambda t: (t[1], t[0])), xq)
        # R38 need flags (home side, per owner) and the owner's candidates (per home peer)
        view.need = {o: [0 if recv_hit[d] else 1 for d in lst] for o, lst in cand_recv.items()}
        view.send_candidates = {d: [list(owned_blocks[dig]) for dig in lst] for d, lst in send.items()}
        return view

    @staticmethod
    def select_send(view: PlanView, peer: int, need: Sequence[int]) -> None:
        """Owner side of R38: the send list to `peer` keeps the candidates it flagged."""
        cands = view.send_candidates.get(peer, [])
        assert len(need) == len(cands), "one flag per candidate fragment"
        view.send[peer] = [b for blocks, n in zip(cands, need) if n for b in blocks]

    def _frag_segment(self, qi, fi, f, s, off, touch, pin, insert_new, pending=frozenset()) -> Segment:
        """All-or-nothing fragment lookup (R10, R11) with pin-before-alloc (R24); a block this plan
        only receives (R38 `pending`) counts as missing and is written by this fragment's prefill."""
        bs = self.bs
        self.stats["lookups"] += 1
        resident = [self.index.get(dig, -1) for dig in s]
        if all(b >= 0 and b not in pending for b in resident):
            for b in resident:
                touch(b)
                pin(b)
            self.stats["hit_blocks"] += len(s)
            self.stats["hit_tokens"] += len(f)
            return Segment(qi, KIND_FRAG, fi, len(f), off, resident, s, 1, len(f), [False] * len(s))
        self.stats["miss_blocks"] += len(s)
        # resident blocks are pinned before any allocation of this fragment, so an eviction
        # cannot reclaim a block the fragment is about to read
        for b in resident:
            if b >= 0:
                touch(b)
                pin(b)
        blocks, write = [], []
        for i, dig in enumerate(s):
            if resident[i] >= 0:
                blocks.append(resident[i])
                write.append(resident[i] in pending)
            else:
                blocks.append(insert_new(dig, min(bs, len(f) - i * bs)))
                write.append(True)
        return Segment(qi, KIND_FRAG, fi, len(f), off, blocks, s, 0, 0, write)

    def release(self, view: PlanView) -> None:
        """Unpin the plan's blocks and free its plan-private blocks."""
        for b in view.pinned:
            self.pins[b] -= 1
        for b in view.private:
            self.free.add(b)

    def evict_all(self) -> None:
        """Drop every unpinned resident block (cold-cache reset)."""
        for b in [b for b in self.meta if self.pins[b] == 0]:
            del self.index[self.meta[b][0]]
            del self.meta[b]
            self.free.add(b)


def hit_rate(stats: Dict[str, int]) -> float:
    """hit tokens / input tokens."""
    return stats["hit_tokens"] / max(1, stats["input_tokens"])
