"""Randomised parity sweep: 60 seeded random instances (3-5 groups, 12-40
layers, mixed tiers, memory budgets that make part of the space infeasible,
several bottleneck factors and (batch, micro-batch) sets) - the engine's
exhaustive arg-min (K1 + K3), explicit batches (K2) and winner detail
against the pinned C oracle, bit for bit."""

import random

import numpy as np
import pytest

from paper_2505_15536_b200 import instances as I
from paper_2505_15536_b200.layout import PackedInstance

SEEDS = list(range(60))


def _instance(seed):
    rng = random.Random(1000 + seed)
    k = rng.randint(3, 5)
    n = rng.randint(max(k, 12), 40)
    regions = []
    for _ in range(k):
        tiers = [[(rng.choice([3.5e13, 7.1e13, 1.65e14, 9.89e14]),
                   rng.choice([6e9, 16e9, 24e9, 80e9]))] * rng.randint(1, 3)]
        if rng.random() < 0.6:
            tiers.append([(rng.choice([2.0e13, 3.12e14, 2.25e15]), rng.choice([8e9, 24e9]))]
                         * rng.randint(1, 2))
        regions.append(tiers)
    layers = I.transformer_layers(n, rng.choice([1024, 2048, 4096]), rng.choice([4096, 5504]),
                                  rng.choice([512, 1024, 2048]), 32000,
                                  d_kv=rng.choice([512, 1024, 2048]), jitter_seed=seed)
    batches = rng.choice([(64, 128), (128,), (32, 64, 256)])
    micros = rng.choice([(8, 16), (4, 8, 16), (16,)])
    spec = I.InstanceSpec(f"fz{seed}", layers, batches, micros, regions,
                          intra_bw=[rng.uniform(1e9, 5e10) for _ in range(k)],
                          intra_lat=[rng.uniform(1e-5, 1e-3) for _ in range(k)],
                          cross_bw=rng.choice([1.25e7, 1.25e8]), cross_lat=0.03, jitter_seed=seed)
    model, topo, groups = I.build(spec)
    return model, topo, groups, rng.choice([1.05, 1.25, 2.0])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_random_instance_parity(engine, oracle_lib, seed):
    model, topo, groups, bf = _instance(seed)
    packed = PackedInstance(model, topo, groups, bf)
    engine.load(packed)
    total = engine.space_size()
    assert total == oracle_lib.space_size(packed)
    got = engine.argmin_range(0, total)
    st, exp = oracle_lib.argmin_range(packed, 0, total, threads=8)
    assert st == 0
    assert (got.cost, got.index) == (exp.cost, exp.index)
    rng = np.random.default_rng(seed)
    idx = rng.choice(total, size=min(total, 2000), replace=False)
    dec = [oracle_lib.decode(packed, int(i)) for i in idx]
    order = np.stack([d[0] for d in dec]); counts = np.stack([d[1] for d in dec])
    bm = np.array([d[2] for d in dec], np.uint8)
    cost, status = engine.eval_batch(order, counts, bm)
    ocost, ostatus = oracle_lib.eval_batch(packed, order, counts, bm)
    assert (status == ostatus).all()
    assert (cost.view(np.uint64) == ocost.view(np.uint64)).all()
    # winner detail (splits + per-stage breakdown) against the oracle's
    o, c, b = oracle_lib.decode(packed, int(exp.index))
    info = engine.plan_detail(o, c, b)
    st2, ocost2, oinfo = oracle_lib.evaluate(packed, o, c, b, detail=True)
    assert st2 == 0 and info.plan_cost == oinfo.plan_cost == exp.cost
    for s in range(len(o)):
        a_, b_ = info.stage[s], oinfo.stage[s]
        assert (a_.kind, a_.n_parts, a_.fill_seconds, a_.run_seconds, a_.residual_seconds,
                a_.collective_seconds) == (b_.kind, b_.n_parts, b_.fill_seconds, b_.run_seconds,
                                           b_.residual_seconds, b_.collective_seconds)
