"""GPU parity of the partitioned (world_size > 1) path on one GPU.

Two contexts stand for ranks 0 and 1 of W = 2 (each its own KV pool, as on two GPUs). Each plans
the same batch for its rank and runs its prefill jobs (its home queries' prefixes plus the
fragments it owns); the K6 pack/unpack kernels then move the remote-owned fragment KV between
the pools through device buffers (the role NCCL's all-to-all plays across GPUs); each rank then
runs the joins of its home queries. Checked against the oracle:
  * each rank's plan is the oracle's `plan(rank, world)` bit for bit (slot maps, exchange lists);
  * received blocks are bit-identical to the owner's blocks (K and V, pads included);
  * prefill and join outputs match the fp64 oracle at the north_star tolerances.
"""
import numpy as np
import pytest

from oracle import attention as oatt
from oracle.store import Store
from paper_2511_02749_b200 import inputs, parallel, runner, spanq

from test_gpu_parity import check, check_lse

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,world,phased,out", [("bf16", 2, False, "fp32"), ("fp32", 2, False, "fp32"),
                                                    ("bf16", 3, False, "fp32"), ("bf16", 2, True, "fp32"),
                                                    ("bf16", 3, True, "fp32"), ("fp32", 2, True, "fp32"),
                                                    ("bf16", 2, True, "bf16")])
def test_partitioned_exchange_parity(cuda_dev, dtype, world, phased, out):
    # phased: each home rank runs join phase 0 (held segments) BEFORE the exchange — with its
    # received blocks poisoned with NaN, so reading one early would show — then phase 1 after it
    import torch

    fp32 = dtype == "fp32"
    sh = inputs.Shape(hq=8, hkv=2, d=128 if not fp32 else 64, block_size=16, vocab=512, dtype=dtype)
    qs = inputs.random_queries(205 + world, 9, vocab=512, max_frag=5, max_len=150, max_prefix=100,
                               max_cross=120, reuse_p=0.5)
    seed = 205
    eq, ek, ev = inputs.layer_tables(sh, 0, seed)
    tab = runner.device_tables(sh, 0, seed, cuda_dev)
    flat = [(q.prefix, q.fragments, q.cross) for q in qs]
    ctxs, plans, views, outs = [], [], [], []
    for r in range(world):
        ctx = spanq.Context(sh, 2048, device=0, max_position=1 << 14, out_dtype=out, rank=r, world_size=world)
        plan = ctx.plan(qs)
        view = plan.view()
        ov = Store(2048, sh.hq, sh.hkv, sh.d, sh.block_size, sh.rope_base, sh.model_salt).plan(flat, rank=r,
                                                                                                   world=world)
        np.testing.assert_array_equal(view["prefill_slot"], ov.prefill_slot)
        np.testing.assert_array_equal(view["join_slot"], ov.join_slot)
        for p in range(world):
            np.testing.assert_array_equal(view["send"].get(p, np.zeros(0, np.int32)), ov.send.get(p, []))
            np.testing.assert_array_equal(view["recv"].get(p, np.zeros(0, np.int32)), ov.recv.get(p, []))
        ptok = runner.prefill_tokens(view, qs)
        odt = torch.bfloat16 if out == "bf16" else torch.float32
        op = torch.empty((len(ptok), sh.hq, sh.d), dtype=odt, device=cuda_dev)
        lp = torch.empty((len(ptok), sh.hq), dtype=torch.float32, device=cuda_dev)
        if len(ptok):
            q, k, v = runner.gather(tab, ptok, cuda_dev)
            plan.prefill(0, q, k, v, op, lp)
        if len(ov.jobs):
            eo, el = oatt.plan_prefill_expected(ov, flat, eq, ek, ev, sh.rope_base)
            check(op, eo, fp32, f"rank {r} prefill O")
            check_lse(lp, el, fp32, f"rank {r} prefill LSE")
        ctxs.append(ctx)
        plans.append(plan)
        views.append(view)
    joins = []
    for r in range(world):
        jtok = runner.join_tokens(views[r], qs)
        oj = torch.empty((len(jtok), sh.hq, sh.d), dtype=torch.bfloat16 if out == "bf16" else torch.float32,
                         device=cuda_dev)
        lj = torch.empty((len(jtok), sh.hq), dtype=torch.float32, device=cuda_dev)
        joins.append((*runner.gather(tab, jtok, cuda_dev), oj, lj))
        if phased:
            rid = [views[r]["recv"].get(p, np.zeros(0, np.int32)) for p in range(world)]
            rid = torch.from_numpy(np.concatenate(rid).astype(np.int64)).to(cuda_dev)
            if len(rid):
                ctxs[r].k_pool[0, rid] = float("nan")
                ctxs[r].v_pool[0, rid] = float("nan")
            plans[r].join_phase(0, 0, *joins[r])
    # exchange: rank r packs for p, p unpacks from r (device buffers stand in for NCCL)
    dt = ctxs[0].k_pool.dtype
    be = parallel.block_elems(sh)
    n_moved = 0
    for r in range(world):
        for p in range(world):
            sb = views[r]["send"].get(p, np.zeros(0, np.int32))
            rb = views[p]["recv"].get(r, np.zeros(0, np.int32))
            assert len(sb) == len(rb)
            if not len(sb):
                continue
            buf = torch.full((len(sb) * be,), float("nan"), dtype=dt, device=cuda_dev)
            plans[r].exchange_pack(0, p, buf)
            plans[p].exchange_unpack(0, r, buf)
            torch.cuda.synchronize()
            for a, b in zip(sb.tolist(), rb.tolist()):
                assert torch.equal(ctxs[r].k_pool[0, a], ctxs[p].k_pool[0, b])
                assert torch.equal(ctxs[r].v_pool[0, a], ctxs[p].v_pool[0, b])
            n_moved += len(sb)
    assert n_moved > 0, "workload exchanged nothing"
    # joins of each rank's home queries
    n_join = 0
    for r in range(world):
        q, k, v, oj, lj = joins[r]
        if phased:
            plans[r].join_phase(0, 1, q, k, v, oj, lj)
        else:
            plans[r].join(0, q, k, v, oj, lj)
        torch.cuda.synchronize()
        home = [i for i in range(len(qs)) if i % world == r]
        exp = [oatt.join_rows(*flat[i], eq, ek, ev, sh.rope_base) for i in home]
        check(oj, np.concatenate([e[0] for e in exp]), fp32, f"rank {r} join O")
        check_lse(lj, np.concatenate([e[1] for e in exp]), fp32, f"rank {r} join LSE")
        n_join += len(q)
    assert n_join == sum(len(q.cross) for q in qs)
    for p, c in zip(plans, ctxs):
        p.release()
        c.close()


@pytest.mark.parametrize("dtype,world,out", [("bf16", 2, "fp32"), ("bf16", 3, "bf16"), ("fp32", 2, "fp32"),
                                             ("bf16", 4, "fp32")])
def test_split_join_parity(cuda_dev, dtype, world, out):
    """Owner-side split join (f1) with W contexts on one GPU: each home packs its queries' cross Q
    for their fragments' owners, each owner runs its tasks (the home query's rows over its
    fragments at Δ_f) into fp32 partials, each home merges them with its local join; the
    device-to-device copies stand in for the two NCCL all-to-alls. Every home query's join
    output must match the oracle's plain join (no KV moved: the owners' pages never leave)."""
    fp32 = dtype == "fp32"
    sh = inputs.Shape(hq=8, hkv=2, d=128 if not fp32 else 64, block_size=16, vocab=512, dtype=dtype)
    qs = inputs.random_queries(305 + world, 10, vocab=512, max_frag=6, max_len=170, max_prefix=90,
                               max_cross=140, reuse_p=0.5)
    _split_run(cuda_dev, sh, qs, world, out, 305, fp32)


@pytest.mark.parametrize("seed", list(range(8)))
def test_split_join_random_fuzz(cuda_dev, seed):
    """The owner-side split join on seeded random shapes (GQA 1-4, d 64 / 128, bs 16-64, bf16 /
    fp32, W = 2-4) against the oracle's plain join."""
    g = np.random.default_rng(6000 + seed)
    hkv = int(g.choice([1, 2, 4]))
    group = int(g.choice([1, 2, 4]))
    dtype = "fp32" if seed % 4 == 3 else "bf16"
    d = int(g.choice([64, 128])) if dtype == "bf16" else 64
    sh = inputs.Shape(hq=hkv * group, hkv=hkv, d=d, block_size=int(g.choice([16, 32, 64])), vocab=512,
                      dtype=dtype, model_salt=seed)
    qs = inputs.random_queries(6100 + seed, 9, vocab=512, max_frag=5, max_len=int(g.integers(20, 170)),
                               max_prefix=int(g.integers(0, 90)), max_cross=int(g.integers(1, 140)), reuse_p=0.5)
    out = "fp32" if dtype == "fp32" or seed % 2 == 0 else "bf16"
    _split_run(cuda_dev, sh, qs, int(g.integers(2, 5)), out, 6200 + seed, dtype == "fp32", require_tasks=False)


def _split_run(cuda_dev, sh, qs, world, out, seed, fp32, require_tasks=True):
    import torch

    eq, ek, ev = inputs.layer_tables(sh, 0, seed)
    tab = runner.device_tables(sh, 0, seed, cuda_dev)
    flat = [(q.prefix, q.fragments, q.cross) for q in qs]
    odt = torch.bfloat16 if out == "bf16" else torch.float32
    ctxs, plans, views, qjoin = [], [], [], []
    for r in range(world):
        ctx = spanq.Context(sh, 2048, device=0, max_position=1 << 14, out_dtype=out, rank=r, world_size=world,
                            split_join=True)
        plan = ctx.plan(qs)
        view = plan.view()
        ptok = runner.prefill_tokens(view, qs)
        if len(ptok):
            plan.prefill(0, *runner.gather(tab, ptok, cuda_dev), torch.empty((len(ptok), sh.hq, sh.d), dtype=odt,
                                                                             device=cuda_dev))
        jtok = runner.join_tokens(view, qs)
        qjoin.append(runner.gather(tab, jtok, cuda_dev))
        ctxs.append(ctx)
        plans.append(plan)
        views.append(view)
    rows = [parallel.split_rows(v, world) for v in views]
    # Q exchange: home h packs (owner-major); owner w receives the chunks of every home (rank order)
    qsend = []
    for h in range(world):
        buf = torch.full((sum(rows[h][0]), sh.hq, sh.d), float("nan"), dtype=qjoin[h][0].dtype, device=cuda_dev)
        plans[h].split_pack_q(qjoin[h][0], buf)
        qsend.append(buf)
    chunks = lambda x, counts: list(torch.split(x, counts)) if len(counts) else []
    qrecv = [torch.cat([chunks(qsend[h], rows[h][0])[w] for h in range(world)]) for w in range(world)]
    for w in range(world):
        assert qrecv[w].shape[0] == sum(rows[w][1])
    # homes: K1 + local join (before the owners' partials exist); owners: task joins
    for h in range(world):
        plans[h].split_join_local(0, *qjoin[h])
    parts = []
    for w in range(world):
        po = torch.full((qrecv[w].shape[0], sh.hq, sh.d), float("nan"), device=cuda_dev)
        pl = torch.full((qrecv[w].shape[0], sh.hq), float("nan"), device=cuda_dev)
        plans[w].split_task_join(0, qrecv[w], po, pl)
        parts.append((po, pl))
    torch.cuda.synchronize()
    n_tasks = sum(len(v["tasks"]) for v in views)
    assert n_tasks > 0 or not require_tasks, "no remote work"
    # partials back: owner w's rows homed on h -> h, which lays them out owner-major
    for h in range(world):
        ro = torch.cat([chunks(parts[w][0], rows[w][1])[h] for w in range(world)])
        rl = torch.cat([chunks(parts[w][1], rows[w][1])[h] for w in range(world)])
        n = int(views[h]["query_join_row_off"][-1])
        oj = torch.empty((n, sh.hq, sh.d), dtype=odt, device=cuda_dev)
        lj = torch.empty((n, sh.hq), dtype=torch.float32, device=cuda_dev)
        plans[h].split_merge(ro, rl, oj, lj)
        torch.cuda.synchronize()
        home = [i for i in range(len(qs)) if i % world == h]
        exp = [oatt.join_rows(*flat[i], eq, ek, ev, sh.rope_base) for i in home]
        check(oj, np.concatenate([e[0] for e in exp]), fp32, f"rank {h} split join O")
        check_lse(lj, np.concatenate([e[1] for e in exp]), fp32, f"rank {h} split join LSE")
    for p, c in zip(plans, ctxs):
        p.release()
        c.close()


@pytest.mark.parametrize("dtype,world,phased", [("bf16", 2, False), ("bf16", 3, False), ("fp32", 2, False),
                                                ("bf16", 2, True), ("bf16", 3, True)])
def test_replica_hits_across_batches(cuda_dev, dtype, world, phased):
    """Digest-keyed replicas (reading R38) on one GPU with W contexts standing in for ranks: batch 1
    moves remote fragments to their home ranks, where they are indexed; batch 2 re-reads some of
    them. After the need-flag round (home flags -> owners' spq_exchange_set_need) the owners send
    only what has no replica, the received blocks equal the owners' bit for bit, the replica
    blocks still hold batch 1's KV, and every join of batch 2 matches the fp64 oracle. phased: the
    join runs in two phases around the exchange, phase 0 with the blocks being received poisoned
    (NaN) — replica hits belong to phase 0 and must not read a poisoned block."""
    fp32 = dtype == "fp32"
    sh = inputs.Shape(hq=8, hkv=2, d=128 if not fp32 else 64, block_size=16, vocab=512, dtype=dtype)
    qs = inputs.random_queries(405 + world, 16, vocab=512, max_frag=5, max_len=120, max_prefix=80,
                               max_cross=100, reuse_p=0.6)
    _replica_run(cuda_dev, sh, [qs[:8], qs[4:16]], world, phased, 405, fp32)


@pytest.mark.parametrize("seed", list(range(8)))
def test_partition_random_fuzz(cuda_dev, seed):
    """Seeded random shapes, W = 2-4 contexts, two overlapping batches (replicas hit in the
    second), plain or phased join: plans bit-exact vs the oracle, moved blocks bit-identical, joins
    vs the fp64 oracle."""
    g = np.random.default_rng(8000 + seed)
    hkv = int(g.choice([1, 2, 4]))
    group = int(g.choice([1, 2, 4]))
    dtype = "fp32" if seed % 4 == 3 else "bf16"
    d = int(g.choice([64, 128])) if dtype == "bf16" else 64
    bs = int(g.choice([16, 32, 64]))
    sh = inputs.Shape(hq=hkv * group, hkv=hkv, d=d, block_size=bs, vocab=512, dtype=dtype, model_salt=seed)
    qs = inputs.random_queries(8100 + seed, 12, vocab=512, max_frag=5, max_len=int(g.integers(20, 160)),
                               max_prefix=int(g.integers(0, 100)), max_cross=int(g.integers(1, 120)), reuse_p=0.6)
    _replica_run(cuda_dev, sh, [qs[:7], qs[3:12]], int(g.integers(2, 5)), bool(seed % 2), 8200 + seed,
                 dtype == "fp32", require_hits=False)


def _replica_run(cuda_dev, sh, batches, world, phased, seed, fp32, require_hits=True):
    import torch

    eq, ek, ev = inputs.layer_tables(sh, 0, seed)
    tab = runner.device_tables(sh, 0, seed, cuda_dev)
    ctxs = [spanq.Context(sh, 4096, device=0, max_position=1 << 14, out_dtype="fp32", rank=r, world_size=world)
            for r in range(world)]
    osts = [Store(4096, sh.hq, sh.hkv, sh.d, sh.block_size, sh.rope_base, sh.model_salt) for _ in range(world)]
    be = parallel.block_elems(sh)
    hits = 0
    for batch in batches:
        flat = [(q.prefix, q.fragments, q.cross) for q in batch]
        plans = [c.plan(batch) for c in ctxs]
        oviews = [osts[r].plan(flat, rank=r, world=world) for r in range(world)]
        views = [p.view() for p in plans]
        for r in range(world):  # prefill of what each rank computes
            ptok = runner.prefill_tokens(views[r], batch)
            if len(ptok):
                q, k, v = runner.gather(tab, ptok, cuda_dev)
                op = torch.empty((len(ptok), sh.hq, sh.d), dtype=torch.float32, device=cuda_dev)
                plans[r].prefill(0, q, k, v, op)
        # need flags: home h -> owner w
        for w in range(world):
            for h in range(world):
                if h != w:
                    flags = views[h]["need"].get(w, np.zeros(0, np.uint8))
                    hits += int((flags == 0).sum())
                    plans[w].exchange_set_need(h, flags)
                    oviews[w].send[h] = [b for bl, n in zip(oviews[w].send_candidates.get(h, []), flags) if n
                                         for b in bl]
        views = [p.view() for p in plans]
        for r in range(world):
            for p in range(world):
                np.testing.assert_array_equal(views[r]["send"].get(p, np.zeros(0, np.int32)), oviews[r].send.get(p, []))
                np.testing.assert_array_equal(views[r]["recv"].get(p, np.zeros(0, np.int32)), oviews[r].recv.get(p, []))
        joins = {}
        for r in range(world):
            jtok = runner.join_tokens(views[r], batch)
            if not len(jtok):
                continue
            q, k, v = runner.gather(tab, jtok, cuda_dev)
            oj = torch.empty((len(jtok), sh.hq, sh.d), dtype=torch.float32, device=cuda_dev)
            lj = torch.empty((len(jtok), sh.hq), dtype=torch.float32, device=cuda_dev)
            joins[r] = (q, k, v, oj, lj)
            if phased:
                rid = [views[r]["recv"].get(p, np.zeros(0, np.int32)) for p in range(world)]
                rid = torch.from_numpy(np.concatenate(rid).astype(np.int64)).to(cuda_dev)
                saved = (ctxs[r].k_pool[0, rid].clone(), ctxs[r].v_pool[0, rid].clone()) if len(rid) else None
                if len(rid):
                    ctxs[r].k_pool[0, rid] = float("nan")
                    ctxs[r].v_pool[0, rid] = float("nan")
                plans[r].join_phase(0, 0, q, k, v, oj, lj)
                torch.cuda.synchronize()
                if saved is not None:  # blocks shared with an owned fragment keep their own KV
                    ctxs[r].k_pool[0, rid], ctxs[r].v_pool[0, rid] = saved
        for r in range(world):
            for p in range(world):
                sb = views[r]["send"].get(p, np.zeros(0, np.int32))
                rb = views[p]["recv"].get(r, np.zeros(0, np.int32))
                assert len(sb) == len(rb)
                if not len(sb):
                    continue
                buf = torch.full((len(sb) * be,), float("nan"), dtype=ctxs[0].k_pool.dtype, device=cuda_dev)
                plans[r].exchange_pack(0, p, buf)
                plans[p].exchange_unpack(0, r, buf)
                torch.cuda.synchronize()
                for a, b in zip(sb.tolist(), rb.tolist()):
                    assert torch.equal(ctxs[r].k_pool[0, a], ctxs[p].k_pool[0, b])
                    assert torch.equal(ctxs[r].v_pool[0, a], ctxs[p].v_pool[0, b])
        for r in range(world):
            if r not in joins:
                continue
            q, k, v, oj, lj = joins[r]
            if phased:
                plans[r].join_phase(0, 1, q, k, v, oj, lj)
            else:
                plans[r].join(0, q, k, v, oj, lj)
            torch.cuda.synchronize()
            home = [i for i in range(len(batch)) if i % world == r]
            exp = [oatt.join_rows(*flat[i], eq, ek, ev, sh.rope_base) for i in home]
            check(oj, np.concatenate([e[0] for e in exp]), fp32, f"rank {r} join O")
            check_lse(lj, np.concatenate([e[1] for e in exp]), fp32, f"rank {r} join LSE")
        for r in range(world):
            plans[r].release()
            osts[r].release(oviews[r])
    assert hits > 0 or not require_hits, "batch 2 re-read no replica"
    for c in ctxs:
        c.close()
