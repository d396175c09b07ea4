"""Cost and timing of explicit plans on the GPU - ``plan_cost`` and
``build_plan_timing`` of the reference (src/costmodel.py:92-100,
src/timing.py:176-231), plus ``simulate(plan, ...)`` (src/simulator.py:116-128).

Unlike the search path (whose splits come from ``choose_intra_split``), a
plan here carries its own splits: the kernel (``k_plan_cost``) takes each
stage's split kind and ``ASYMMETRIC_PP`` parts, which are the only split
data that enter the cost (``effective_capacity`` and the collective
volume).  Memory is not checked, as in the reference.
"""

from __future__ import annotations

from typing import Optional

from . import abi
from . import domain as D
from .engine import Engine, default_engine
from .layout import PackedInstance, packed_instance


def _stages(plan, packed: PackedInstance):
    arr = (abi.GpPlanStage * len(plan.stages))()
    for s, st in enumerate(plan.stages):
        if st.fg_id not in packed.fg_pos:
            raise KeyError(st.fg_id)
        f = packed.fg_pos[st.fg_id]
        r = arr[s]
        r.fg, r.layer_start, r.layer_end = f, st.layer_start, st.layer_end
        kind = getattr(st.intra_split.kind, "value", st.intra_split.kind)
        r.kind = abi.KIND_CODE[D.SplitKind(kind)]
        parts = st.intra_split.parts if r.kind == abi.GP_ASYM_PP else ()
        if len(parts) > abi.GP_MAX_SGS:
            raise D.InputFileError(f"stage {s}: more than {abi.GP_MAX_SGS} pipeline parts")
        r.n_parts = len(parts)
        sg_ids = packed.sg_ids[f]
        for j, (sg, a, b) in enumerate(parts):
            if sg not in sg_ids:
                raise KeyError(sg)
            r.pp_sg[j], r.pp_start[j], r.pp_end[j] = sg_ids.index(sg), int(a), int(b)
    return arr


def _evaluate(plan, topology, model, groups, opt_seconds, engine, timing):
    packed = packed_instance(model, topology, groups, 1.25)
    eng = (engine if engine is not None else default_engine()).load(packed)
    return eng.plan_cost(_stages(plan, packed), plan.batch_b, plan.microbatch_m, opt_seconds,
                         timing)


def plan_cost(plan, topology, model, groups, opt_seconds: float = 0.0,
              engine: Optional[Engine] = None) -> D.CostBreakdown:
    """``plan_cost`` (src/costmodel.py:92-100) of a plan with its own splits."""
    info, _ = _evaluate(plan, topology, model, groups, opt_seconds, engine, False)
    per_stage = tuple(D.StageCost(fill_seconds=info.stage[s].fill_seconds,
                                  run_seconds=info.stage[s].run_seconds,
                                  residual_seconds=info.stage[s].residual_seconds,
                                  collective_seconds=info.stage[s].collective_seconds)
                      for s in range(len(plan.stages)))
    return D.CostBreakdown(per_stage=per_stage, plan_cost=info.plan_cost)


def build_plan_timing(plan, topology, model, groups, opt_seconds: float = 0.0,
                      engine: Optional[Engine] = None):
    """``build_plan_timing`` (src/timing.py:176-231) as simulate.PlanTiming
    (``al_seconds`` carries the sync value; the event engine never reads it)."""
    from .simulate import BoundaryTiming, PlanTiming, StageTiming
    _, t = _evaluate(plan, topology, model, groups, opt_seconds, engine, True)
    S = int(t.n_stages)
    stages = tuple(StageTiming(t.fwd[s], t.bwd[s], t.wgt[s], t.sync[s], t.sync[s], t.opt[s], 1.0)
                   for s in range(S))
    bounds = tuple(BoundaryTiming(f"{b}-{b + 1}", t.lat[b], t.bw[b], t.act[b], t.grad[b])
                   for b in range(S - 1))
    return PlanTiming(stages, bounds, int(t.batch), int(t.microbatch))


def simulate(plan, topology, model, groups, policy="1f1b", trace=None,
             adapter_enabled: bool = False, config=None, engine: Optional[Engine] = None):
    """``simulate`` (src/simulator.py:116-128): build_plan_timing then the
    full event engine; returns simulate.SimSummary."""
    from .simulate import SimConfig, simulate_timing
    config = config if config is not None else SimConfig()
    timing = build_plan_timing(plan, topology, model, groups,
                               getattr(config, "opt_seconds", 0.0), engine)
    return simulate_timing(timing, policy, trace, adapter_enabled, config, engine)
