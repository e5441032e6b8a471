"""CIDRA host schedule (spq_cidra_schedule): executing its ops IN PLACE on symbolic
block contents must give every destination its source's ORIGINAL content with the move's shift —
the out-of-place definition (oracle/cidra.py) — for chains, cycles, self-moves,
duplicated sources and random move graphs. Labels are exact, so this is bit-exact. CPU only."""
import numpy as np
import pytest

from oracle.cidra import out_degree_duplicates
from paper_2511_02749_b200 import inputs, spanq

NBLK = 512


@pytest.fixture(scope="module")
def ctx():
    c = spanq.Context(inputs.Shape(hq=2, hkv=1, d=64, block_size=16, dtype="fp32"), NBLK, device=-1,
                      max_position=1 << 15)
    yield c
    c.close()


def run_symbolic(ops, off):
    """Execute the schedule in place on labels: block b holds (origin block, accumulated shift)."""
    content = {b: (b, 0) for b in range(NBLK)}
    for c in range(len(off) - 1):
        tmp = None
        for dst, src, delta, mode in ops[off[c]: off[c + 1]]:
            if mode == 1:
                tmp = content[src]
            elif mode == 2:
                content[dst] = (tmp[0], tmp[1] + delta)
            else:
                o, sh = content[src]
                content[dst] = (o, sh + delta)
    return content


def expected(moves):
    out = {b: (b, 0) for b in range(NBLK)}
    for s, d, dl in moves:
        out[d] = (s, dl)
    return out


def check(ctx, moves):
    src, dst, dl = (np.array([m[i] for m in moves], np.int32) for i in range(3))
    ops, off, st = ctx.cidra_schedule(src, dst, dl)
    assert run_symbolic(ops, off) == expected(moves)
    # every move runs exactly once; per component one scratch save per cycle
    assert st["moves"] == len(moves) and st["ops"] == len(moves) + st["cycles"]
    assert st["duplicates"] == out_degree_duplicates([(s, d, 0, 0) for s, d, _ in moves])
    assert st["components"] == len(off) - 1
    # reads precede writes block by block, so op i+1 never reads what op i writes (a kernel may
    # issue op i+1's loads before op i's stores)
    for c in range(len(off) - 1):
        seq = ops[off[c]: off[c + 1]]
        for a, b in zip(seq[:-1], seq[1:]):
            if a[3] != 1 and b[3] != 2:
                assert b[1] != a[0], (a, b)
    # components touch disjoint blocks (they run in parallel)
    seen = {}
    for c in range(len(off) - 1):
        for dsti, srci, _, mode in ops[off[c]: off[c + 1]]:
            for b in (dsti, srci):
                if b >= 0:
                    assert seen.setdefault(int(b), c) == c
    return st


def test_swap_is_one_cycle(ctx):  # SPEC S:396 "A<->B swap -> one 2-cycle, zero duplications"
    st = check(ctx, [(3, 7, 100), (7, 3, -40)])
    assert st["cycles"] == 1 and st["duplicates"] == 0 and st["components"] == 1


def test_chain_self_move_and_duplicates(ctx):
    # chain 1 -> 2 -> 3 -> 4 (in place: 4 first), a self-move, a source feeding 3 destinations
    st = check(ctx, [(1, 2, 5), (2, 3, 6), (3, 4, 7), (9, 9, 11), (20, 21, 1), (20, 22, 2), (20, 23, 3)])
    assert st["cycles"] == 1 and st["duplicates"] == 2 and st["components"] == 3


def test_cycle_with_trees(ctx):
    # 3-cycle 10 -> 11 -> 12 -> 10 with trees hanging off it (they must read before the rotation)
    check(ctx, [(10, 11, 1), (11, 12, 2), (12, 10, 3), (10, 30, 4), (30, 31, 5), (12, 32, 6), (31, 33, 7)])


@pytest.mark.parametrize("seed", range(20))
def test_random_move_graphs(ctx, seed):
    # random functional graphs over a small block range (dense conflicts: cycles, trees, chains,
    # duplicated sources), SPEC S:416 style instances
    g = np.random.default_rng(seed)
    nb = int(g.integers(2, 80))
    n = int(g.integers(1, nb + 1))
    dsts = g.choice(nb, size=n, replace=False)
    srcs = g.integers(0, nb, size=n)
    moves = [(int(s), int(d), int(x)) for s, d, x in zip(srcs, dsts, g.integers(-5000, 5000, size=n))]
    check(ctx, moves)


def test_errors(ctx):
    with pytest.raises(spanq.SpanqError) as e:
        ctx.cidra_schedule([1, 2], [5, 5], [0, 0])  # block 5 written twice
    assert e.value.status == spanq.EINVAL
    with pytest.raises(spanq.SpanqError):
        ctx.cidra_schedule([NBLK], [0], [0])
    with pytest.raises(spanq.SpanqError):
        ctx.cidra_schedule([0], [1], [1 << 15])  # no RoPE table row for |delta|
    with pytest.raises(spanq.SpanqError) as e:
        ctx.reposition([0], [1], [3])  # host-only ctx: no pool
    assert e.value.status == spanq.ESTATE
    ops, off, st = ctx.cidra_schedule([], [], [])
    assert len(ops) == 0 and list(off) == [0] and st["components"] == 0
