"""Drop-in ``search_plan`` / ``exhaustive_plan`` backed by the CUDA engine.

Signatures, results and exceptions follow the reference
(``src/planner.py:330-403``, src/ = /root/reference/pkg/src/geopipe/):

* :func:`exhaustive_plan` is one K3 launch: the arg-min over every
  ``(b, m, order, cuts)`` index under the reference key ``(cost, (order,
  cuts))`` with earliest-``(b, m)`` tie-break (src/planner.py:389-399).
* :func:`search_plan` keeps the reference's host-side beam driver - Python
  ``random.Random(f"{seed}:{b}:{m}")`` streams, candidate expansion, stable
  sort on ``(cost, (order, counts))`` and the monotone trace - but advances the
  independent ``(b, m)`` passes in lock-step so each beam iteration is ONE K2
  batch on the GPU instead of ``|B||M|`` Python ``_evaluate`` loops.  The
  per-pass RNG streams are independent, so the lock-step order does not change
  any draw; best/trace are replayed afterwards in the reference's pass order.

All costs come from the engine (:mod:`.engine`).  Nothing here evaluates a
plan on the CPU.
"""

from __future__ import annotations

import logging
import math
import random
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import abi
from . import domain as D
from .engine import Engine, default_engine
from .layout import PackedInstance, packed_instance

log = logging.getLogger(__name__)

INFEASIBLE = math.inf
# exhaustive spaces above this many candidates go to the K4 branch-and-bound
BNB_THRESHOLD = 500_000_000


# --------------------------------------------------------------------------
# host-side beam driver pieces (integer / RNG logic only)
# --------------------------------------------------------------------------

def proportional_split(total: int, weights: Sequence[float], minimum: int = 0) -> List[int]:
    """Largest-remainder shares (src/planner.py:65-87); used by the beam's
    initial candidates on the host.  Same arithmetic as the device copy in
    csrc/device_math.cuh."""
    wsum = sum(weights)
    raw = [total * w / wsum for w in weights]
    shares = [int(math.floor(r)) for r in raw]
    rem = [r - s for r, s in zip(raw, shares)]
    leftover = total - sum(shares)
    for idx in sorted(range(len(weights)), key=lambda i: (-rem[i], i))[:leftover]:
        shares[idx] += 1
    if minimum > 0:
        for i in range(len(shares)):
            while shares[i] < minimum:
                donor = max(range(len(shares)), key=lambda j: shares[j])
                if shares[donor] <= minimum:
                    raise D.InfeasibleSplitError(
                        f"cannot give {minimum} unit(s) to each of {len(shares)} "
                        f"parts out of {total}")
                shares[donor] -= 1
                shares[i] += 1
    return shares


def initial_candidates(model, fgs, l: int, seed: int) -> List[D.Candidate]:
    """Random orders with capacity-proportional cuts (src/planner.py:256-282)."""
    n = len(model.layers)
    if len(fgs) > n:
        raise D.InfeasibleSplitError(f"{len(fgs)} groups cannot each take a layer of {n}")
    rng = random.Random(seed)
    ids = sorted(fg.id for fg in fgs)
    caps = {fg.id: fg.aggregate_capacity for fg in fgs}
    out = []
    for i in range(l):
        order = list(ids)
        rng.shuffle(order)
        counts = proportional_split(n, [caps[f] for f in order], minimum=1)
        if i > 0 and len(counts) > 1:
            j = rng.randrange(len(counts) - 1)
            if rng.random() < 0.5 and counts[j] > 1:
                counts[j] -= 1
                counts[j + 1] += 1
            elif counts[j + 1] > 1:
                counts[j + 1] -= 1
                counts[j] += 1
        out.append(D.Candidate(order=tuple(order), counts=tuple(counts)))
    return out


def expand_candidates(cands, rng: random.Random) -> List[D.Candidate]:
    """Self + one random transposition + every +-1 cut shift, deduplicated in
    first-seen order (src/planner.py:285-310)."""
    seen: Dict[tuple, D.Candidate] = {}
    for cand in cands:
        variants = [cand]
        k = len(cand.order)
        if k > 1:
            i, j = rng.sample(range(k), 2)
            order = list(cand.order)
            order[i], order[j] = order[j], order[i]
            variants.append(D.Candidate(order=tuple(order), counts=cand.counts))
        for b in range(k - 1):
            if cand.counts[b] > 1:
                c = list(cand.counts)
                c[b] -= 1
                c[b + 1] += 1
                variants.append(D.Candidate(cand.order, tuple(c)))
            if cand.counts[b + 1] > 1:
                c = list(cand.counts)
                c[b + 1] -= 1
                c[b] += 1
                variants.append(D.Candidate(cand.order, tuple(c)))
        for v in variants:
            seen.setdefault((v.order, v.counts), v)
    return list(seen.values())


def _expand_keys(cands, rng: random.Random) -> List[tuple]:
    """expand_candidates on ``(order, counts)`` tuples (the beam driver's
    internal form): the same variants in the same first-seen order and the
    same RNG draws (one ``rng.sample(range(k), 2)`` per candidate with k > 1),
    without building a Candidate per variant."""
    seen: Dict[tuple, None] = {}
    add = seen.setdefault
    for order, counts in cands:
        k = len(order)
        add((order, counts), None)
        if k > 1:
            i, j = rng.sample(range(k), 2)
            o = list(order)
            o[i], o[j] = o[j], o[i]
            add((tuple(o), counts), None)
        for b in range(k - 1):
            if counts[b] > 1:
                c = list(counts)
                c[b] -= 1
                c[b + 1] += 1
                add((order, tuple(c)), None)
            if counts[b + 1] > 1:
                c = list(counts)
                c[b + 1] -= 1
                c[b] += 1
                add((order, tuple(c)), None)
    return list(seen)


# --------------------------------------------------------------------------
# result assembly from the engine's plan detail
# --------------------------------------------------------------------------

def _engine_for(packed: PackedInstance, engine: Engine = None) -> Engine:
    eng = engine if engine is not None else default_engine()
    return eng.load(packed)


def assemble(packed: PackedInstance, eng: Engine, order_idx, counts, bm: int, info=None):
    """(plan, breakdown|None, feasible) of one candidate, from gp_plan_detail."""
    if info is None:
        info = eng.plan_detail(order_idx, counts, bm)
    b, m = packed.bm_pairs()[bm]
    stages = []
    pos = 0
    group_cache: Dict[int, abi.GpGroupInfo] = {}
    for s, f in enumerate(order_idx):
        f = int(f)
        fid = packed.fg_ids[f]
        st = info.stage[s]
        kind = abi.KIND_OF[st.kind]
        end = pos + int(counts[s])
        if st.kind == abi.GP_ASYM_PP:
            parts = tuple((packed.sg_ids[f][st.pp_sg[j]], int(st.pp_start[j]),
                           int(st.pp_end[j])) for j in range(st.n_parts))
        elif st.kind in (abi.GP_ASYM_TP_DP, abi.GP_ASYM_DP):
            g = group_cache.get(f)
            if g is None:
                g = group_cache[f] = eng.group_splits(f)
            if st.kind == abi.GP_ASYM_TP_DP:
                members = packed.groups.fgs[fid].member_device_ids
                parts = tuple((d, g.tp_row[x], g.tp_col[x]) for x, d in enumerate(members))
            else:
                parts = tuple((sid, g.dp_fraction[j])
                              for j, sid in enumerate(packed.sg_ids[f]))
        else:
            parts = ()
        stages.append(D.StageAssignment(fg_id=fid, layer_start=pos, layer_end=end,
                                        intra_split=D.IntraSplit(kind, parts)))
        pos = end
    plan = D.ParallelPlan(stages=tuple(stages), batch_b=b, microbatch_m=m)
    if not info.feasible:
        return plan, None, False
    per_stage = tuple(D.StageCost(fill_seconds=info.stage[s].fill_seconds,
                                  run_seconds=info.stage[s].run_seconds,
                                  residual_seconds=info.stage[s].residual_seconds,
                                  collective_seconds=info.stage[s].collective_seconds)
                      for s in range(len(order_idx)))
    breakdown = D.CostBreakdown(per_stage=per_stage, plan_cost=info.plan_cost)
    return plan, breakdown, True


# --------------------------------------------------------------------------
# drop-in entry points
# --------------------------------------------------------------------------

def exhaustive_plan(model, topology, groups, config, engine: Engine = None) -> D.SearchResult:
    """GPU replacement for ``exhaustive_plan`` (src/planner.py:374-403)."""
    packed = packed_instance(model, topology, groups, config.bottleneck_factor)
    eng = engine if engine is not None else default_engine()
    k, n = packed.n_fgs, packed.n_layers
    space = (len(packed.batches) * len(packed.micros) * math.factorial(k) *
             math.comb(n - 1, k - 1)) if k <= n else 0
    if space > BNB_THRESHOLD:
        # large spaces: exact branch-and-bound with DP bounds (K4), same winner
        eng.load(packed)
        best = eng.argmin_bnb()
        info = None
    else:
        best, info = eng.replan(packed)   # H2D + K1 + K3 + detail as one CUDA graph
    total = int(best.evaluated)
    k = best.k
    order = np.array(best.order[:k], dtype=np.uint8)
    counts = np.array(best.counts[:k], dtype=np.uint8)
    bm = best.batch_index * len(packed.micros) + best.micro_index
    plan, breakdown, feasible = assemble(packed, eng, order, counts, bm, info)
    if breakdown is None:
        raise D.NoFeasiblePlanError("no feasible plan in exhaustive sweep")
    return D.SearchResult(plan=plan, breakdown=breakdown,
                          best_cost_trace=[best.cost], evaluated=int(total))


def search_plan(model, topology, groups, config, engine: Engine = None) -> D.SearchResult:
    """GPU-batched replacement for ``search_plan`` (src/planner.py:330-371).

    The (b, m) passes advance in lock-step (one K2 batch per beam iteration
    over every active pass); what the caller observes is then replayed in the
    reference's sequential pass order: the per-plan memory warnings
    (src/planner.py:321) and per-pass "no feasible plan" warnings (:367) in
    that order, and - if a candidate raises - the exception of the first
    erroring candidate in sequential (pass, iteration, position) order.  A
    pass that errors stops; passes after it in the sequential order are not
    needed any more, passes before it run on until they finish or error.
    """
    packed = packed_instance(model, topology, groups, config.bottleneck_factor)
    eng = _engine_for(packed, engine)
    fgs = sorted(groups.fgs.values(), key=lambda g: g.id)
    pairs = packed.bm_pairs()
    # one beam state per (b, m) pass, in the reference's pass order
    passes = []
    for bm, (b, m) in enumerate(pairs):
        rng = random.Random(f"{config.seed}:{b}:{m}")
        beam = [(c.order, c.counts) for c in
                initial_candidates(model, fgs, config.beam_width, rng.randrange(2 ** 30))]
        passes.append({"bm": bm, "rng": rng, "beam": beam, "tops": [], "iters": [],
                       "err": None})
    cache: Dict[tuple, float] = {}
    errors: Dict[tuple, int] = {}  # key -> status of candidates that raise
    first_err = len(passes)        # smallest pass index that raised so far
    for _ in range(config.max_iter):
        live = [ps for ps in passes[:first_err] if ps["err"] is None]
        if not live:
            break
        expanded = []
        todo_c, todo_bm, todo_keys = [], [], []
        for ps in live:
            ex = _expand_keys(ps["beam"], ps["rng"])
            expanded.append(ex)
            b, m = pairs[ps["bm"]]
            for c in ex:
                key = c + (b, m)
                if key not in cache and key not in errors:
                    cache[key] = None
                    todo_c.append(c)
                    todo_bm.append(ps["bm"])
                    todo_keys.append(key)
        if todo_c:
            o, cn, bmv = packed.encode_keys(todo_c, todo_bm)
            cost, status = eng.eval_batch(o, cn, bmv)
            for key, c, st in zip(todo_keys, cost.tolist(), status.tolist()):
                if st:
                    del cache[key]
                    errors[key] = int(st)
                else:
                    cache[key] = c
        for ps, ex in zip(live, expanded):
            b, m = pairs[ps["bm"]]
            ps["iters"].append(ex)
            bad = next((j for j, c in enumerate(ex) if c + (b, m) in errors), None) if errors else None
            if bad is not None:
                ps["err"] = (len(ps["iters"]) - 1, bad)
                first_err = min(first_err, passes.index(ps))
                continue
            scored = [(cache[c + (b, m)], c) for c in ex]
            scored.sort()
            ps["beam"] = [x[1] for x in scored[:config.beam_width]]
            ps["tops"].append((scored[0][0], scored[0][1]))
    # replay in the reference's sequential order: warnings, trace, best, errors
    best = None
    trace: List[float] = []
    warn = log.isEnabledFor(logging.WARNING)
    for ps in passes:
        b, m = pairs[ps["bm"]]
        seen = set()
        for it, ex in enumerate(ps["iters"]):
            stop = ps["err"][1] if ps["err"] is not None and ps["err"][0] == it else len(ex)
            for c in ex[:stop]:
                key = c + (b, m)
                if key not in seen:
                    seen.add(key)
                    if warn and cache[key] == INFEASIBLE:
                        log.warning("plan %s exceeds device memory; penalized", key)
            if stop < len(ex):
                key = ex[stop] + (b, m)
                abi.raise_for(errors[key], f"candidate {key} failed")
        incumbent = math.inf
        for top_cost, top_key in ps["tops"]:
            incumbent = min(incumbent, top_cost)
            if best is None or (top_cost, top_key) < (best[0], best[1]):
                best = (top_cost, top_key, ps["bm"])
            trace.append(min(incumbent, best[0]))
        if incumbent == math.inf:
            log.warning("no feasible plan for batch=%d micro=%d", b, m)
    if best is None or best[0] == INFEASIBLE:
        raise D.NoFeasiblePlanError("all (batch, micro-batch) pairs infeasible")
    order_ids, counts = best[1]
    order = np.array([packed.fg_pos[f] for f in order_ids], dtype=np.uint8)
    plan, breakdown, feasible = assemble(packed, eng, order,
                                         np.array(counts, dtype=np.uint8), best[2])
    if breakdown is None:
        raise D.NoFeasiblePlanError("all (batch, micro-batch) pairs infeasible")
    return D.SearchResult(plan=plan, breakdown=breakdown, best_cost_trace=trace,
                          evaluated=len(cache))
