"""Bandwidth-snapshot re-plan (K6) vs the reference's CS4 composition.

Golden tests/golden/c3_snapshots.json: C2 under App. D C3 snapshots 0..199,
each rebuilt with the reference constructors + grouping; arg-min from the
pinned oracle (checked against the reference exhaustive_plan on 3 of them).
"""

import numpy as np
import pytest

import golden_io as G
from paper_2505_15536_b200 import instances as I
from paper_2505_15536_b200.layout import PackedInstance
from paper_2505_15536_b200 import replan as R

SNAP = G.load("c3_snapshots.json")


def _setup(n=200):
    spec = I.config("c2")
    model, topo, groups = I.build(spec)
    packed = PackedInstance(model, topo, groups, 1.25)
    mults = [I.snapshot_multipliers(spec, j) for j in range(n)]
    return spec, model, topo, groups, packed, R.bandwidth_matrices(packed, mults)


def test_snapshot_matrices_and_min_bw_match_reference_rebuild():
    spec, model, topo, groups, packed, bws = _setup(50)
    for j in range(50):
        m2, t2, g2 = I.build(spec, I.snapshot_multipliers(spec, j))
        p2 = PackedInstance(m2, t2, g2, 1.25)
        assert (p2.bw == bws[j]).all()
        exp = SNAP["snapshots"][j]["min_bw"]
        for f in sorted(g2.fgs):
            assert g2.fgs[f].min_intra_bandwidth == exp[f]


@pytest.mark.gpu
def test_k6_replan_200_snapshots(engine):
    spec, model, topo, groups, packed, bws = _setup(200)
    engine.load(packed)
    bests, status = engine.replan_snapshots(bws)
    assert (status == 0).all()
    for j, rec in enumerate(SNAP["snapshots"]):
        assert bests[j].cost == rec["cost"], j
        assert bests[j].index == rec["index"], j
    # the context's own instance is left unchanged
    total = engine.space_size()
    assert engine.argmin_range(0, total).cost == G.load("c2.json")["exhaustive"]["result"]["breakdown"]["plan_cost"]


@pytest.mark.gpu
def test_k6_replan_pinned_matrices_read_in_place(engine):
    """Pinned (mapped) host matrices are read in place by the patch kernels
    (zero-copy) - same winners as the golden composition."""
    import torch
    spec, model, topo, groups, packed, bws = _setup(60)
    pinned = torch.from_numpy(bws).pin_memory().numpy()
    engine.load(packed)
    bests, status = engine.replan_snapshots(pinned)
    assert (status == 0).all()
    for j, rec in enumerate(SNAP["snapshots"][:60]):
        assert bests[j].cost == rec["cost"], j
        assert bests[j].index == rec["index"], j


@pytest.mark.gpu
def test_k6_replan_detail_matches_reference(engine):
    from paper_2505_15536_b200 import SearchConfig
    spec, model, topo, groups, packed, bws = _setup(3)
    res = R.replan_snapshots(model, topo, groups, SearchConfig(seed=0), bws, engine=engine,
                             detail=True)
    for j in range(3):
        assert G.normalize_result(res[j]) == SNAP["snapshots"][j]["reference"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 3])
def test_k6_variants(engine, mode):
    spec, model, topo, groups, packed, bws = _setup(20)
    engine.load(packed)
    try:
        engine.set_k3_mode(mode)
        bests, status = engine.replan_snapshots(bws)
    finally:
        engine.set_k3_mode(-1)
    for j in range(20):
        assert bests[j].index == SNAP["snapshots"][j]["index"]


@pytest.mark.gpu
def test_graph_replan_over_same_shape_instances(engine):
    """gp_replan replays one captured CUDA graph for every same-shape instance."""
    spec = I.config("c2")
    for j in list(range(12)) + [0, 5]:
        m2, t2, g2 = I.build(spec, I.snapshot_multipliers(spec, j))
        best, info = engine.replan(PackedInstance(m2, t2, g2, 1.25))
        assert best.cost == SNAP["snapshots"][j]["cost"], j
        assert best.index == SNAP["snapshots"][j]["index"], j
        assert info.plan_cost == best.cost
