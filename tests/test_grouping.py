"""Two-level grouping (K7) vs the reference's group_first_level /
group_second_level (src/grouping.py:146-228).

Golden: tests/golden/grouping.json (scripts/make_golden.py dump_grouping) =
the reference's groups for every topology of tests/grouping_cases.py.
"""

import math

import numpy as np
import pytest

import golden_io as G
import grouping_cases as GC
from paper_2505_15536_b200 import domain as D
from paper_2505_15536_b200 import grouping as GR

GOLD = G.load("grouping.json")
NAMES = GC.names()


def _bits(x):
    return np.float64(x).view(np.uint64)


def _check(h, rows):
    assert len(h.fg_capacity) == len(rows)
    base = 0
    for f, (members, intra, cap, minbw, sgs) in enumerate(rows):
        assert list(np.nonzero(h.fg_of == f)[0]) == members
        assert _bits(h.fg_capacity[f]) == _bits(cap)
        if intra is None:
            assert math.isnan(h.fg_intra[f]) and math.isnan(h.fg_min_bw[f])
        else:
            assert _bits(h.fg_intra[f]) == _bits(intra)
            assert _bits(h.fg_min_bw[f]) == _bits(minbw)
        mem = np.array(members)
        for j, (sm, scap) in enumerate(sgs):
            assert list(mem[h.sg_of[mem] == j]) == sm
            assert _bits(h.sg_capacity[base + j]) == _bits(scap)
        assert int(h.sg_of[mem].max()) == len(sgs) - 1
        base += len(sgs)
    assert len(h.sg_capacity) == base


def test_golden_covers_ties_and_scale():
    assert len(GOLD) == len(NAMES)
    sizes = [len(GC.build(n)[2]) for n in ("big0", "big1", "c4")]
    assert sizes == [160, 256, 64]
    assert any(len(rows) > 3 for rows in GOLD.values())


@pytest.mark.parametrize("name", NAMES)
def test_oracle_grouping_matches_reference(oracle_lib, name):
    pt, bw, pc, tn, tc = GC.build(name)
    st, h = oracle_lib.group_hierarchy(pt, bw, pc, tn, tc)
    assert st == 0
    _check(h, GOLD[name])


def test_oracle_rejects_bad_thresholds(oracle_lib):
    pt, bw, pc, _, _ = GC.build("rand0")
    assert oracle_lib.group_hierarchy(pt, bw, pc, 0.0, 0.3)[0] != 0
    assert oracle_lib.group_hierarchy(pt, bw, pc, 0.3, 1.0)[0] != 0


@pytest.mark.gpu
def test_k7_matches_reference(engine):
    # one launch per threshold pair, every case of that pair batched by size
    by = {}
    for name in NAMES:
        pt, bw, pc, tn, tc = GC.build(name)
        by.setdefault((len(pc), tn, tc, pc.tobytes()), []).append((name, pt, bw, pc))
    for (n, tn, tc, _), cases in by.items():
        pts = np.stack([c[1] for c in cases])
        bws = np.stack([c[2] for c in cases])
        hs = GR.group_hierarchies(pts, bws, cases[0][3], tn, tc, engine=engine)
        for (name, *_), h in zip(cases, hs):
            _check(h, GOLD[name])


@pytest.mark.gpu
def test_k7_snapshot_batch(engine):
    names = [f"c4snap{s}" for s in range(12)]
    built = [GC.build(n) for n in names]
    hs = GR.group_hierarchies(np.stack([b[0] for b in built]), np.stack([b[1] for b in built]),
                              built[0][2], 0.3, 0.3, engine=engine)
    for name, h in zip(names, hs):
        _check(h, GOLD[name])
    assert len({len(h.fg_capacity) for h in hs}) > 1  # regrouping changes k


@pytest.mark.gpu
def test_k7_drop_in_hierarchy_equals_instance_groups(engine):
    from paper_2505_15536_b200 import instances as I
    for name in ("c1", "c2", "c4"):
        _, topo, groups = I.load(name, True)
        fgs, sgs, gi = GR.build_hierarchy(topo, 0.3, 0.3, engine=engine)
        assert [fg for fg in fgs] == [groups.fgs[f] for f in sorted(groups.fgs)]
        assert {k: tuple(v) for k, v in sgs.items()} == dict(groups.sgs_by_fg)
        assert gi == groups


@pytest.mark.gpu
def test_k7_errors(engine):
    pt, bw, pc, _, _ = GC.build("rand1")
    with pytest.raises(D.InputFileError):
        engine.group_snapshots(pt, bw, pc, 1.5, 0.3)
    with pytest.raises(D.InputFileError):
        engine.group_snapshots(np.zeros((1, 0, 0)), None, np.zeros(0), 0.3, 0.3)


REPLAN = G.load("regroup_replan.json")


@pytest.mark.gpu
def test_regroup_then_replan_matches_reference(engine):
    """p_t snapshots of C2: K7 regrouping (k changes between 3 and 4 groups)
    then the exact re-plan equal the reference's group_first_level +
    group_second_level + exhaustive_plan on the rebuilt topology."""
    from paper_2505_15536_b200 import instances as I
    from paper_2505_15536_b200.replan import replan_regrouped
    model, topo, _ = I.load("c2")
    names = sorted(REPLAN)
    pts = np.stack([GC.build(n)[0] for n in names])
    res = replan_regrouped(model, topo, D.SearchConfig(seed=0), pts, engine=engine)
    ks = set()
    for name, (r, gi) in zip(names, res):
        exp = REPLAN[name]
        assert "result" in exp
        got = G.normalize_result(r)
        assert got["plan"] == exp["result"]["plan"]
        assert got["breakdown"] == exp["result"]["breakdown"]
        ks.add(len(gi.fgs))
    assert ks == {3, 4}


# ------------------------------------------------ C2 region-grouping sweep --
SWEEP = G.load("region_sweep.json")


def _sweep_arrays():
    from paper_2505_15536_b200 import instances as I
    _, topo, _ = I.load("c2")
    ids, pt, bw, pc = GR.topology_arrays(topo)
    return topo, ids, pt, bw, pc


def test_set_partitions_order():
    from paper_2505_15536_b200.replan import set_partitions
    assert set_partitions(3) == [[0, 0, 0], [0, 0, 1], [0, 1, 0], [0, 1, 1], [0, 1, 2]]
    assert len(set_partitions(4)) == 15 and [g["rgs"] for g in SWEEP["groupings"]] == set_partitions(3)


@pytest.mark.parametrize("gi", range(5))
def test_oracle_fixed_partition_matches_reference(oracle_lib, gi):
    topo, ids, pt, bw, pc = _sweep_arrays()
    g = SWEEP["groupings"][gi]
    pos = {d: i for i, d in enumerate(ids)}
    fg_of = np.zeros(len(ids), np.uint16)
    for f, (_, members, *_r) in enumerate(g["fgs"]):
        for d in members:
            fg_of[pos[d]] = f
    st, h = oracle_lib.group_fixed(pt, bw, pc, fg_of, len(g["fgs"]))
    assert st == 0
    fgs, sgs, _ = GR.to_groups(ids, h)
    for fg, (fid, members, intra, cap, mb) in zip(fgs, g["fgs"]):
        assert (fg.id, list(fg.member_device_ids), fg.aggregate_capacity) == (fid, members, cap)
        assert (fg.intra_metric, fg.min_intra_bandwidth) == (intra, mb)
        assert [[s.id, list(s.member_device_ids), s.aggregate_capacity] for s in sgs[fid]] == \
            g["sgs"][fid]


@pytest.mark.gpu
def test_region_grouping_sweep_matches_reference(engine):
    from paper_2505_15536_b200 import instances as I
    from paper_2505_15536_b200.replan import region_grouping_sweep
    model, topo, _ = I.load("c2")
    results, best = region_grouping_sweep(model, topo, SWEEP["regions"], D.SearchConfig(seed=0),
                                          engine=engine)
    evaluated = 0
    for (blocks, r), g in zip(results, SWEEP["groupings"]):
        assert blocks == g["blocks"]
        if "error" in g:
            assert type(r).__name__ == g["error"]
            continue
        got = G.normalize_result(r)
        assert got["plan"] == g["result"]["plan"]
        assert got["breakdown"] == g["result"]["breakdown"]
        assert r.evaluated == g["result"]["evaluated"]
        evaluated += r.evaluated
    assert evaluated == 3 * 372 + 16740
    costs = [(g["result"]["breakdown"]["plan_cost"], i) for i, g in enumerate(SWEEP["groupings"])
             if "result" in g]
    assert best == min(costs)[1]
