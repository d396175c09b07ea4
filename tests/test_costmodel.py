"""Explicit-plan cost and timing (k_plan_cost) vs the reference's plan_cost /
build_plan_timing (src/costmodel.py:92-100, src/timing.py:176-231).

Golden: tests/golden/plan_costs.json (scripts/make_golden.py dump_plan_costs)
= 40 random plans per golden instance with arbitrary split kinds and
pipeline parts (incl. empty and degenerate ones), the reference's
CostBreakdown and PlanTiming, or the exception it raised.
"""

import json
import tempfile

import numpy as np
import pytest

import golden_io as G
from cases import load_case
from paper_2505_15536_b200 import domain as D
from paper_2505_15536_b200 import fileio
from paper_2505_15536_b200.costmodel import build_plan_timing, plan_cost

GOLD = G.load("plan_costs.json")
ERR = {"DegenerateGroupError": D.DegenerateGroupError,
       "InvalidTopologyError": D.InvalidTopologyError}


def _plan(d):
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as fh:
        json.dump(d, fh)
    return fileio.read_plan(fh.name)


def test_golden_has_every_split_kind_and_errors():
    kinds = {st["split"]["kind"] for rows in GOLD.values() for r in rows
             for st in r["plan"]["stages"] if "cost" in r}
    assert kinds == {"uniform", "asymmetric_pp", "asymmetric_dp", "asymmetric_tp_dp"}
    errs = {r["error"] for rows in GOLD.values() for r in rows if "error" in r}
    assert errs == set(ERR)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
def test_plan_cost_matches_reference(engine, name):
    _, model, topo, groups = load_case(name)
    for r in GOLD[name]:
        plan = _plan(r["plan"])
        if "error" in r:
            with pytest.raises(ERR[r["error"]]):
                plan_cost(plan, topo, model, groups, r["opt_seconds"], engine=engine)
            continue
        bd = plan_cost(plan, topo, model, groups, r["opt_seconds"], engine=engine)
        assert G.breakdown_to_dict(bd) == r["cost"]
        t = build_plan_timing(plan, topo, model, groups, r["opt_seconds"], engine=engine)
        got = {"batch": t.batch, "microbatch": t.microbatch,
               "stages": [[s.fwd_per_sample, s.bwd_per_sample, s.wgt_per_sample,
                           s.sync_seconds, s.opt_seconds] for s in t.stages],
               "boundaries": [[b.latency_seconds, b.bandwidth_bytes_per_s,
                               b.act_bytes_per_sample, b.grad_bytes_per_sample]
                              for b in t.boundaries]}
        assert got == r["timing"]


@pytest.mark.gpu
def test_plan_cost_of_planner_plans_equals_search_breakdown(engine):
    from paper_2505_15536_b200 import search_plan
    for name in ("c1j", "c2j", "rand3"):
        _, model, topo, groups = load_case(name)
        res = search_plan(model, topo, groups, D.SearchConfig(seed=0), engine=engine)
        assert plan_cost(res.plan, topo, model, groups, engine=engine) == res.breakdown
