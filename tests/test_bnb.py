"""K4 branch-and-bound == exhaustive arg-min (same cost, same winner index)."""

import pytest

from cases import CASES_ALL, load_case
from paper_2505_15536_b200 import instances as I
from paper_2505_15536_b200.layout import PackedInstance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", CASES_ALL + ["c4", "c4j"])
def test_bnb_equals_exhaustive_golden(engine, name):
    doc, model, topo, groups = load_case(name)
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    total = engine.space_size()
    if total == 0:
        return
    try:
        ex = engine.argmin_range(0, total)
    except Exception as e:
        with pytest.raises(type(e)):
            engine.argmin_bnb()
        return
    bb = engine.argmin_bnb()
    assert bb.cost == ex.cost
    assert bb.index == ex.index


def _many_group_instance(k, n, seed, jitter=True):
    return I.build(I.many_group_config(k, n, seed, jitter=jitter))


@pytest.mark.parametrize("k,n,seed", [(5, 20, 1), (5, 24, 2), (6, 16, 3), (6, 20, 4), (6, 40, 5),
                                      (7, 20, 11), (7, 24, 12), (8, 16, 13)])
def test_bnb_equals_sweep_many_groups(engine, k, n, seed):
    model, topo, groups = _many_group_instance(k, n, seed)
    assert len(groups.fgs) == k
    packed = PackedInstance(model, topo, groups, 1.25)
    engine.load(packed)
    total = engine.space_size()
    ex = engine.argmin_range(0, total)
    bb = engine.argmin_bnb()
    assert bb.cost == ex.cost
    assert bb.index == ex.index


@pytest.mark.parametrize("name", ["c1j", "c2", "c2j", "small", "rand10", "err_memory", "c4"])
def test_exhaustive_plan_via_bnb_matches_reference(engine, name, monkeypatch):
    import golden_io as G
    import paper_2505_15536_b200 as P
    from paper_2505_15536_b200 import planner as PL
    monkeypatch.setattr(PL, "BNB_THRESHOLD", 0)
    doc, model, topo, groups = load_case(name)
    cfg = P.SearchConfig(seed=0)
    if "error" in doc.get("exhaustive", {}):
        with pytest.raises(P.GeopipeError):
            P.exhaustive_plan(model, topo, groups, cfg, engine=engine)
        return
    res = P.exhaustive_plan(model, topo, groups, cfg, engine=engine)
    if "exhaustive" in doc:
        assert G.normalize_result(res) == doc["exhaustive"]["result"]
    else:
        exp = doc["oracle_argmin"]
        assert res.breakdown.plan_cost == exp["cost"]
