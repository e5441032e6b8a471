"""Multi-rank partitioning of a span-query batch, host side, CPU only.

* The C++ planner in partitioned mode (ctx rank r of W) is bit-exact against the oracle's
  `Store.plan(rank=r, world=W)` — segments, block tables, slot maps, stats and exchange lists.
* The exchange lists agree across ranks: what rank r sends to p is, block for block, the
  fragment KV that p's plan expects from r (same digests, same order).
* Partitioning covers the batch exactly once: every join runs on one rank, every distinct
  fragment (cold cache) is prefilled on exactly one rank, its owner.
* The exchange step itself (parallel.exchange_layer) over a real world-2 gloo group moves the
  right blocks into the right places (pack/unpack emulated on CPU pools; the CUDA K6 kernel is
  covered by tests/test_gpu_parity.py).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from oracle import hashing
from oracle.store import OracleENOMEM, Store
from paper_2511_02749_b200 import inputs, parallel, spanq

from test_abi_host import STAT_KEYS, assert_same, flat


def seg_digest_map(view):
    """block id -> digest (bytes) for every block referenced by the view's segments."""
    m = {}
    for b, d in zip(view["blocks"], view["digests"]):
        m.setdefault(int(b), bytes(d))
    return m


def test_owner_rank_definition():
    d = bytes(range(16))
    v = sum(d[i] << (8 * i) for i in range(8))  # u64 little-endian of the first 8 bytes
    for w in (1, 2, 3, 8):
        assert hashing.owner_rank(d, w) == v % w


@pytest.mark.parametrize("world,seed,bs,nblk", [(2, 11, 4, 4096), (3, 12, 8, 4096), (4, 13, 2, 160),
                                                (2, 14, 16, 64)])
def test_partitioned_planner_bit_exact_vs_oracle(world, seed, bs, nblk):
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=bs, dtype="fp32", rope_base=5000.0, model_salt=seed)
    qs = inputs.random_queries(seed, 48, vocab=12, max_len=30)
    for rank in range(world):
        ctx = spanq.Context(shape, nblk, device=-1, rank=rank, world_size=world)
        ost = Store(nblk, 4, 2, 64, bs, 5000.0, seed)
        g = np.random.default_rng(seed * 10 + rank)
        live, i, n_plans = [], 0, 0
        while i < len(qs):
            k = int(g.integers(1, 6))
            batch = qs[i:i + k]
            i += k
            try:
                ov = ost.plan([flat(q) for q in batch], rank=rank, world=world)
            except OracleENOMEM:
                with pytest.raises(spanq.SpanqError) as e:
                    ctx.plan(batch)
                assert e.value.status == spanq.ENOMEM
                continue
            cp = ctx.plan(batch)
            cv = cp.view()
            assert_same(cv, ov)
            assert cv["n_join_queries"] == ov.n_join_queries
            assert cv["world_size"] == world
            for name, od in (("send", ov.send), ("recv", ov.recv)):
                assert sorted(cv[name]) == sorted(p for p, b in od.items() if b), name
                for p, b in od.items():
                    np.testing.assert_array_equal(cv[name].get(p, np.zeros(0, np.int32)), b, err_msg=name)
            cs = ctx.stats()
            for key in STAT_KEYS:
                assert cs[key] == ost.stats[key], key
            live.append((cp, ov))
            n_plans += 1
            while live and g.random() < 0.5:
                cp, ov = live.pop(int(g.integers(0, len(live))))
                cp.release()
                ost.release(ov)
        assert n_plans >= 4
        for cp, ov in live:
            cp.release()
        ctx.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_exchange_lists_agree_and_cover_batch(world):
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=8, dtype="fp32")
    qs = inputs.random_queries(21 + world, 40, vocab=16, max_len=40, reuse_p=0.5)
    views = []
    for rank in range(world):
        ctx = spanq.Context(shape, 1 << 14, device=-1, rank=rank, world_size=world)
        views.append(ctx.plan(qs).view())
    maps = [seg_digest_map(v) for v in views]
    for r in range(world):
        for p in range(world):
            sent = [maps[r][int(b)] for b in views[r]["send"].get(p, [])]
            got = [maps[p][int(b)] for b in views[p]["recv"].get(r, [])]
            assert sent == got, (r, p)
        assert r not in views[r]["send"] and r not in views[r]["recv"]
    # every join on exactly one rank (its home), all queries covered
    homes = [set(np.nonzero(np.diff(v["query_join_row_off"]))[0].tolist()) for v in views]
    assert sum(len(h) for h in homes) == len(qs)
    for r, h in enumerate(homes):
        assert h == {q for q in range(len(qs)) if q % world == r and len(qs[q].cross)}
        assert views[r]["n_join_queries"] == len([q for q in range(len(qs)) if q % world == r])
    # cold cache: every distinct fragment prefilled exactly once, on its owner
    frag_jobs = {}
    for r, v in enumerate(views):
        for j in v["jobs"]:
            if v["seg_kind"][j] == 1:
                blk0 = v["seg_block_off"][j]
                nb = v["seg_n_blocks"][j]
                last = bytes(v["digests"][blk0 + nb - 1])
                frag_jobs.setdefault(last, []).append(r)
    distinct = {hashing.fragment_chain(np.asarray(f), 8, Store(1, 4, 2, 64, 8).root)[-1]
                for q in qs for f in q.fragments}
    assert set(frag_jobs) == distinct
    for last, ranks in frag_jobs.items():
        assert ranks == [hashing.owner_rank(last, world)]


# ---------------------------------------------------------------- exchange over a gloo group
class _CpuPlan:
    """pack/unpack of K6 emulated on CPU pools [nblk, 2, E] (E = block elems / 2); the need-flag
    step goes to the real (host-only) plan."""

    def __init__(self, plan, pool):
        self.plan, self.pool = plan, pool
        self.cur = plan.view()

    def exchange_set_need(self, peer, need):
        self.plan.exchange_set_need(peer, need)

    def view(self):
        self.cur = self.plan.view()
        return self.cur

    def exchange_pack(self, layer, peer, buf, stream=None):
        blocks = self.cur["send"][peer]
        buf.view(len(blocks), -1).copy_(self.pool[blocks].reshape(len(blocks), -1))

    def exchange_unpack(self, layer, peer, buf, stream=None):
        blocks = self.cur["recv"][peer]
        self.pool[blocks] = buf.view(len(blocks), *self.pool.shape[1:])


def _fill_from_digest(pool, dmap):
    import torch

    for b, d in dmap.items():
        g = np.random.default_rng(int.from_bytes(d[:8], "little"))
        pool[b] = torch.from_numpy(g.standard_normal(pool.shape[1:]).astype(np.float32))


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shape = inputs.Shape(hq=4, hkv=2, d=16, block_size=4, dtype="fp32")
        qs = inputs.random_queries(77, 24, vocab=16, max_len=20, reuse_p=0.5)
        ctx = spanq.Context(shape, 4096, device=-1, rank=rank, world_size=world)
        be = parallel.block_elems(shape)
        pool = torch.zeros(4096, 2, be // 2)
        hits = 0
        # two batches: the second re-reads fragments the first received (R38 replicas: their
        # blocks keep the first exchange's KV and need no transfer)
        for batch in (qs[:12], qs[6:24]):
            plan = _CpuPlan(ctx.plan(batch), pool)
            view = parallel.exchange_needs(plan, plan.cur, rank, world)
            hits += sum(int(x == 0) for v in view["need"].values() for x in v)
            dmap = seg_digest_map(view)
            recv_blocks = {int(b) for bl in view["recv"].values() for b in bl}
            # fill only the blocks this rank computes (owned fragments written by this plan);
            # received ones come from the exchange, replica hits from the previous batch
            _fill_from_digest(pool, {int(b): dmap[int(b)] for b, w in zip(view["blocks"], view["block_write"])
                                     if w and int(b) not in recv_blocks})
            stats = parallel.exchange_layer(plan, view, 0, shape, "cpu", torch.float32, rank, world)
            ref = torch.zeros_like(pool)
            _fill_from_digest(ref, dmap)
            for s in range(len(view["seg_kind"])):
                if view["seg_kind"][s] != 1:
                    continue
                for b in view["blocks"][view["seg_block_off"][s]:][:view["seg_n_blocks"][s]]:
                    assert torch.equal(pool[int(b)], ref[int(b)]), f"rank {rank}: block {b} holds the wrong fragment KV"
            counts = [None] * world
            dist.all_gather_object(counts, (stats["sent_bytes"], stats["recv_bytes"], len(recv_blocks)))
            assert sum(c[0] for c in counts) == sum(c[1] for c in counts)
            assert sum(c[2] for c in counts) > 0
            plan.plan.release()
        all_hits = [None] * world
        dist.all_gather_object(all_hits, hits)
        assert sum(all_hits) > 0, "no replica was re-read"
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback

        q.put((rank, traceback.format_exc()))


def test_exchange_layer_gloo_world2():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


# ---------------------------------------------------------------- owner-side split join (f1)
@pytest.mark.parametrize("world,seed,bs", [(2, 31, 4), (3, 32, 8), (5, 33, 2)])
def test_split_planner_bit_exact_vs_oracle(world, seed, bs):
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=bs, dtype="fp32", model_salt=seed)
    qs = inputs.random_queries(seed, 30, vocab=12, max_len=30, reuse_p=0.5)
    for rank in range(world):
        ctx = spanq.Context(shape, 4096, device=-1, rank=rank, world_size=world, split_join=True)
        ost = Store(4096, 4, 2, 64, bs, shape.rope_base, seed)
        for i in range(0, len(qs), 7):
            batch = qs[i:i + 7]
            ov = ost.plan([flat(q) for q in batch], rank=rank, world=world, split=True)
            cv = ctx.plan(batch).view()
            assert_same(cv, ov)
            np.testing.assert_array_equal(cv["seg_pos0"], [s.pos0 for s in ov.segments])
            assert cv["tasks"] == ov.tasks
            assert cv["xq"] == {p: q for p, q in ov.xq.items() if q}
            assert not cv["send"] and not cv["recv"]  # no KV moves in split mode
        ctx.close()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_split_lists_agree_and_cover_batch(world):
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=8, dtype="fp32")
    qs = inputs.random_queries(41 + world, 40, vocab=16, max_len=40, reuse_p=0.5)
    views = [spanq.Context(shape, 1 << 14, device=-1, rank=r, world_size=world, split_join=True).plan(qs).view()
             for r in range(world)]
    root = Store(1, 4, 2, 64, 8).root
    for h in range(world):
        for w in range(world):
            # what home h sends to owner w is what w's tasks homed on h read, in the same order
            mine = views[h]["xq"].get(w, [])
            theirs = [t[0] for t in views[w]["tasks"] if t[1] == h]
            assert mine == theirs, (h, w)
            rows_h = sum(int(views[h]["query_join_row_off"][q + 1] - views[h]["query_join_row_off"][q]) for q in mine)
            assert rows_h == sum(t[2] for t in views[w]["tasks"] if t[1] == h)
    # every (query, fragment occurrence) attended exactly once: on the home (a local segment) or
    # by the owner's task for that query, at the fragment's offset Δ_f in the query
    for qi, q in enumerate(qs):
        h = qi % world
        want, off = [], len(q.prefix)
        for f in q.fragments:
            want.append((hashing.fragment_chain(np.asarray(f), 8, root)[-1], off))
            off += len(f)
        got = []
        v = views[h]
        for s in range(len(v["seg_kind"])):
            if v["seg_query"][s] == qi and v["seg_kind"][s] == 1:
                blk = v["seg_block_off"][s] + v["seg_n_blocks"][s] - 1
                got.append((bytes(v["digests"][blk]), int(v["seg_pos0"][s])))
        for w in range(world):
            for (tq, th, n_rows, pos0, sb, se) in views[w]["tasks"]:
                if tq != qi:
                    continue
                assert th == h and n_rows == len(q.cross) and pos0 == off
                for s in range(sb, se):
                    vw = views[w]
                    assert vw["seg_query"][s] == qi and vw["seg_kind"][s] == 1
                    blk = vw["seg_block_off"][s] + vw["seg_n_blocks"][s] - 1
                    d = bytes(vw["digests"][blk])
                    assert hashing.owner_rank(d, world) == w
                    got.append((d, int(vw["seg_pos0"][s])))
        assert sorted(got) == sorted(want), qi


class _CpuSplitPlan:
    """split_pack_q / split_task_join emulated on CPU: the 'partial' of a task row is the received
    q row itself (fp32) and its LSE the task's query id, so the home can check that every row came
    back from the right owner in the right order."""

    def __init__(self, view):
        self.view = view

    def split_pack_q(self, q_join, qsend, stream=None):
        off = self.view["query_join_row_off"]
        rows = [r for w in sorted(self.view["xq"]) for q in self.view["xq"][w] for r in range(off[q], off[q + 1])]
        qsend.copy_(q_join[rows])

    def split_task_join(self, layer, qrecv, part_o, part_lse, stream=None):
        import torch

        part_o.copy_(qrecv.float())
        qid = [t[0] for t in self.view["tasks"] for _ in range(t[2])]
        part_lse.copy_(torch.tensor(qid, dtype=torch.float32)[:, None].expand_as(part_lse))


def _gloo_split_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        shape = inputs.Shape(hq=2, hkv=1, d=8, block_size=4, dtype="fp32")
        qs = inputs.random_queries(88, 20, vocab=16, max_len=20, reuse_p=0.5)
        ctx = spanq.Context(shape, 4096, device=-1, rank=rank, world_size=world, split_join=True)
        view = ctx.plan(qs).view()
        n = int(view["query_join_row_off"][-1])
        q_join = torch.arange(n * 2 * 8, dtype=torch.float32).reshape(n, 2, 8) + 1000 * rank
        out = parallel.split_exchange_layer(_CpuSplitPlan(view), view, 0, shape, "cpu", q_join, rank, world)
        off = view["query_join_row_off"]
        r = 0
        for w in sorted(view["xq"]):
            for qq in view["xq"][w]:
                k = off[qq + 1] - off[qq]
                assert torch.equal(out["part_o"][r:r + k], q_join[off[qq]:off[qq + 1]]), (rank, w, qq)
                assert (out["part_lse"][r:r + k] == qq).all()
                r += k
        assert r == out["part_o"].shape[0]
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported by the parent
        import traceback

        q.put((rank, traceback.format_exc()))


def test_split_exchange_gloo_world2():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


# ---------------------------------------------------------------- digest-keyed replicas (R38)
def _need_round(views, plans, world, ostores=None, oviews=None):
    """The need-flag exchange among W host-only ranks: home h's flags for owner w go to w."""
    for w in range(world):
        for h in range(world):
            if h == w:
                continue
            flags = views[h]["need"].get(w, np.zeros(0, np.uint8))
            assert len(flags) == views[w]["n_cand_send"][h], (h, w)
            plans[w].exchange_set_need(h, flags)
            if oviews is not None:
                Store.select_send(oviews[w], h, list(flags))
    return [p.view() for p in plans]


def _digest_lists(view, key, peer):
    m = seg_digest_map(view)
    return [m[int(b)] for b in view[key].get(peer, [])]


@pytest.mark.parametrize("world,seed", [(2, 51), (3, 52), (4, 53)])
def test_replicas_hit_in_later_plans_and_need_flags_prune_the_sends(world, seed):
    """A fragment received once is indexed on the home rank under its digests: a later plan there
    hits it (need flag 0, segment hit, nothing in the recv list), and once the owners apply the
    homes' flags, what each owner sends is exactly what each home receives. C++ and the oracle
    agree on every list, flag and stat along the way."""
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=4, dtype="fp32", model_salt=seed)
    qs = inputs.random_queries(seed, 36, vocab=10, max_len=24, reuse_p=0.6)
    ctxs = [spanq.Context(shape, 8192, device=-1, rank=r, world_size=world) for r in range(world)]
    ost = [Store(8192, 4, 2, 64, 4, shape.rope_base, seed) for _ in range(world)]
    replica_hits = 0
    for i in range(0, len(qs), 6):
        batch = qs[i:i + 6]
        plans = [c.plan(batch) for c in ctxs]
        oviews = [ost[r].plan([flat(q) for q in batch], rank=r, world=world) for r in range(world)]
        views = [p.view() for p in plans]
        for r in range(world):
            assert_same(views[r], oviews[r])
            assert {p: list(v) for p, v in views[r]["need"].items()} == {p: v for p, v in oviews[r].need.items() if v}
            assert views[r]["n_cand_send"] == [len(oviews[r].send_candidates.get(p, [])) for p in range(world)]
            for key in STAT_KEYS:
                assert ctxs[r].stats()[key] == ost[r].stats[key], key
            replica_hits += sum(int(x == 0) for v in views[r]["need"].values() for x in v)
            # a need-0 fragment's segment is a hit and none of its blocks is received
            recv = {int(b) for bl in views[r]["recv"].values() for b in bl}
            for s in range(len(views[r]["seg_kind"])):
                if views[r]["seg_kind"][s] == 1 and views[r]["seg_hit"][s] == 1:
                    blk = views[r]["blocks"][views[r]["seg_block_off"][s]:][:views[r]["seg_n_blocks"][s]]
                    last = bytes(views[r]["digests"][views[r]["seg_block_off"][s] + views[r]["seg_n_blocks"][s] - 1])
                    if hashing.owner_rank(last, world) != r:
                        assert not recv.intersection(int(b) for b in blk)
        views = _need_round(views, plans, world, ost, oviews)
        for r in range(world):
            for p in range(world):
                np.testing.assert_array_equal(views[r]["send"].get(p, np.zeros(0, np.int32)),
                                              oviews[r].send.get(p, []))
                assert _digest_lists(views[r], "send", p) == _digest_lists(views[p], "recv", r), (r, p)
        for r in range(world):
            plans[r].release()
            ost[r].release(oviews[r])
    assert replica_hits > 0, "the batch sequence never re-read a received fragment"
    for c in ctxs:
        c.close()


def test_owned_fragment_sharing_a_received_block_writes_it():
    """R38 hazard: a remote fragment B received by this plan and a locally owned fragment A that
    shares B's first block (a common token prefix). The block's KV arrives only with the exchange
    (after the prefill and after this rank packs its own sends), so A must not treat it as cached:
    A is a miss and its prefill writes that block. Checked on C++ and the oracle."""
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=4, dtype="fp32", model_salt=5)
    root = Store(1, 4, 2, 64, 4, shape.rope_base, 5).root
    head = np.array([1, 2, 3, 4], np.int32)  # one full shared block
    g = np.random.default_rng(0)
    a = b = None
    while a is None or b is None:
        f = np.concatenate([head, g.integers(0, 50, 5).astype(np.int32)])
        own = hashing.owner_rank(hashing.fragment_chain(f, 4, root)[-1], 2)
        if own == 0 and a is None:
            a = f
        elif own == 1 and b is None:
            b = f
    q = inputs.SpanQuery(np.zeros(0, np.int32), [b, a], np.array([7, 8], np.int32))
    ctx = spanq.Context(shape, 256, device=-1, rank=0, world_size=2)
    v = ctx.plan([q]).view()
    ov = Store(256, 4, 2, 64, 4, shape.rope_base, 5).plan([flat(q)], rank=0, world=2)
    assert_same(v, ov)
    segs = [s for s in range(len(v["seg_kind"])) if v["seg_kind"][s] == 1]
    sb, sa = segs  # B (received), A (owned)
    blk_b0 = int(v["blocks"][v["seg_block_off"][sb]])
    blk_a0 = int(v["blocks"][v["seg_block_off"][sa]])
    assert blk_a0 == blk_b0  # one block, indexed once
    assert v["seg_hit"][sa] == 0 and v["block_write"][v["seg_block_off"][sa]] == 1
    assert blk_b0 in v["recv"][1].tolist()
    ctx.close()


def test_exchange_set_need_rejects_bad_input():
    """spq_exchange_set_need (R38): the flag count must equal the peer's candidate count, the
    peer must exist, and a released plan is refused."""
    shape = inputs.Shape(hq=4, hkv=2, d=64, block_size=4, dtype="fp32")
    qs = inputs.random_queries(61, 12, vocab=10, max_len=20, reuse_p=0.5)
    ctx = spanq.Context(shape, 4096, device=-1, rank=1, world_size=2)
    plan = ctx.plan(qs)
    v = plan.view()
    n = v["n_cand_send"][0]
    assert n > 0
    with pytest.raises(spanq.SpanqError) as e:
        plan.exchange_set_need(0, np.ones(n + 1, np.uint8))
    assert e.value.status == spanq.EINVAL
    with pytest.raises(spanq.SpanqError) as e:
        plan.exchange_set_need(2, np.ones(n, np.uint8))
    assert e.value.status == spanq.ESTATE
    plan.exchange_set_need(0, np.zeros(n, np.uint8))  # nothing to send to rank 0
    assert 0 not in plan.view()["send"]
    plan.exchange_set_need(0, np.ones(n, np.uint8))  # flags can be re-applied: all again
    np.testing.assert_array_equal(plan.view()["send"][0], v["send"][0])
    plan.release()
    with pytest.raises(spanq.SpanqError) as e:
        plan.exchange_set_need(0, np.ones(n, np.uint8))
    assert e.value.status == spanq.ESTATE
    ctx.close()
