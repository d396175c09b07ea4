"""Multi-rank exhaustive re-plan: item sharding + tuple arg-min reduction.

CPU: world_size 2 over gloo, each rank's shard evaluated by the oracle (the
engine needs a GPU); the reduced winner must equal the reference's
exhaustive_plan winner.  GPU: engine item ranges vs the golden costs.
"""

import math
import os
import random

import numpy as np
import pytest
import torch.multiprocessing as mp

from cases import enumerate_encoded, golden_costs, load_case
from paper_2505_15536_b200 import distributed as DI
from paper_2505_15536_b200.layout import PackedInstance


def _oracle_items(O, packed, lo, hi):
    """Rank-local (cost, tie, first error) over items [lo, hi), oracle-evaluated."""
    k = packed.n_fgs
    NC, NP, n_items = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    nm = len(packed.micros)
    best, err = DI.NO_KEY, None
    for bi in range(len(packed.batches)):
        a, b = (bi * nm * NP + lo) * NC, (bi * nm * NP + hi) * NC
        cost, status = O.eval_range(packed, a, b, threads=1)
        bad = np.nonzero(status)[0]
        if bad.size:
            if err is None or a + int(bad[0]) < err[0]:
                err = (a + int(bad[0]), int(status[bad[0]]))
            continue
        for j in range(cost.size):
            best = min(best, (float(cost[j]), DI.tie_of_index(a + j, NC, NP, nbm)))
    return best[0], best[1], err


def _worker(rank, world, port, name, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    k = packed.n_fgs
    NC, NP, n_items = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    try:
        out[rank] = DI.sharded_argmin(lambda lo, hi: _oracle_items(O, packed, lo, hi), n_items)
    except Exception as e:  # every rank must raise the same error, none may hang
        out[rank] = type(e).__name__
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = 29500 + random.randint(0, 2000)
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (out,))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    return dict(out)


@pytest.mark.parametrize("name", ["err_gateway", "err_intra_bw"])
def test_gloo_two_ranks_raise_reference_error(name):
    """A rank whose shard raises does not leave the others in the collective:
    all ranks raise the error of the smallest index, as the reference does."""
    out = _spawn(_worker, 2, name)
    doc, model, topo, groups = load_case(name)
    exp = doc["exhaustive"]["error"]
    assert out[0] == out[1] == exp


def _snap_worker(rank, world, port, n_snap, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2505_15536_b200 import instances as I
    spec = I.config("c1")
    lo, hi = DI.shard_items(n_snap, world, rank)
    rec = np.zeros((hi - lo, 3), np.int64)
    for i, j in enumerate(range(lo, hi)):
        m, t, g = I.build(spec, I.snapshot_multipliers(spec, j))
        p = PackedInstance(m, t, g, 1.25)
        st, b = O.argmin_range(p, 0, O.space_size(p), threads=1)
        rec[i] = (DI._cost_bits(b.cost), b.index, st)
    allrec = DI.gather_snapshot_records(rec, n_snap, device=torch.device("cpu"))
    m, t, g = I.build(spec)
    out[rank] = list(DI.decode_snapshot_records(PackedInstance(m, t, g, 1.25), allrec))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_snapshot_shards_gather_every_result(world):
    """Snapshots partitioned by index; every rank ends with all results,
    each equal to the single-process re-plan of that snapshot."""
    from oracle import oracle as O
    from paper_2505_15536_b200 import instances as I
    n_snap = 7
    out = _spawn(_snap_worker, world, n_snap)
    spec = I.config("c1")
    for r in range(1, world):
        assert out[r] == out[0]
    for j in range(n_snap):
        m, t, g = I.build(spec, I.snapshot_multipliers(spec, j))
        p = PackedInstance(m, t, g, 1.25)
        st, b = O.argmin_range(p, 0, O.space_size(p), threads=1)
        cost, order, counts, bb, mm = out[0][j]
        assert cost == b.cost
        assert [p.fg_pos[f] for f in order] == list(b.order[:b.k])
        assert counts == list(b.counts[:b.k])
        assert (bb, mm) == (p.batches[b.batch_index], p.micros[b.micro_index])


@pytest.mark.parametrize("name", ["c2", "c2j", "rand10", "small"])
def test_gloo_two_ranks_match_exhaustive(name):
    out = _spawn(_worker, 2, name)
    assert out[0] == out[1]
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    k = packed.n_fgs
    NC, NP, _ = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    cost, tie = out[0]
    order, counts, bm = DI.decode_candidate(tie, NC, NP, nbm, packed.n_layers, k)
    exp = doc["exhaustive"]["result"]
    stages = exp["plan"]["stages"]
    assert cost == exp["breakdown"]["plan_cost"]
    assert [packed.fg_ids[x] for x in order] == [s[0] for s in stages]
    assert counts == [s[2] - s[1] for s in stages]
    assert packed.bm_pairs()[bm] == (exp["plan"]["batch_b"], exp["plan"]["microbatch_m"])


def test_shards_cover_items_exactly():
    for n in (1, 5, 72, 1000):
        for w in (1, 2, 3, 8):
            spans = [DI.shard_items(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_tie_index_roundtrip():
    rng = random.Random(0)
    for _ in range(200):
        NC, NP, nbm = rng.randint(1, 500), rng.choice([1, 2, 6, 24]), rng.randint(1, 6)
        idx = rng.randrange(NC * NP * nbm)
        assert DI.index_of_tie(DI.tie_of_index(idx, NC, NP, nbm), NC, NP, nbm) == idx


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c2j", "rand5", "rand10", "small", "c1j"])
def test_engine_item_ranges(engine, name):
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    gc, gs = golden_costs(name)
    order, counts, bm = enumerate_encoded(packed)
    k = packed.n_fgs
    NC, NP, n_items = DI.space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    nm = len(packed.micros)
    ties = np.array([DI.tie_of_index(i, NC, NP, nbm) for i in range(gc.size)])
    items = np.array([((i // NC) // NP % nm) * NP + (i // NC) % NP for i in range(gc.size)])
    rng = random.Random(3)
    for _ in range(8):
        lo, hi = sorted(rng.sample(range(n_items + 1), 2))
        if hi <= lo:
            continue
        sel = np.nonzero((items >= lo) & (items < hi))[0]
        exp = min((gc[i], ties[i]) for i in sel)
        got = engine.argmin_items(lo, hi)
        assert got.cost == exp[0]
        assert DI.tie_of_index(got.index, NC, NP, nbm) == exp[1]
        assert got.evaluated == sel.size
