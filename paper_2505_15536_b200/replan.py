"""Re-planning over bandwidth-fluctuation snapshots.

The reference has no single entry point for this: the Dynamic Environment
Adapter's re-plan is composed from its APIs - rebuild every
``LinkMeasurement`` with the base alpha/beta/payload/latency and a scaled
``bandwidth_bytes_per_s`` (src/profiling.py:48-78), ``build_topology``
(:167-215), regroup (membership is unchanged because p_t does not depend on
bandwidth; ``min_intra_bandwidth`` is re-derived, src/grouping.py:69-75), then
``exhaustive_plan`` (src/planner.py:374-403).  Here the whole batch of
snapshots is one engine call (gp_replan_snapshots): per-snapshot tables are
patched on the device and one K3 sweep covers every (snapshot, item).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi
from . import domain as D
from .engine import Engine, default_engine
from .layout import PackedInstance, packed_instance
from .planner import assemble


def bandwidth_matrices(packed: PackedInstance,
                       multipliers: Sequence[Dict[Tuple[str, str], float]]) -> np.ndarray:
    """[S, D, D] bandwidths: base link bandwidth x per-pair multiplier
    (keys are (u, v) with u < v), in the packed device order."""
    ids = packed.device_ids
    Dn = len(ids)
    base = packed.bw
    out = np.empty((len(multipliers), Dn, Dn), dtype=np.float64)
    for s, mult in enumerate(multipliers):
        m = np.ones((Dn, Dn))
        for (u, v), f in mult.items():
            i, j = packed.dev_index[u], packed.dev_index[v]
            m[i, j] = m[j, i] = f
        out[s] = base * m
    return out


class SnapshotPlans:
    """Per-snapshot re-plan results as arrays (cost, winner enumeration index,
    status), decoded on access: ``plans[j]`` is the tuple ``(cost, order_ids,
    counts, b, m)`` or the exception the reference's re-plan of snapshot j
    would raise.  Decoding is integer unranking on the host and happens only
    for the snapshots a caller looks at."""

    def __init__(self, packed: PackedInstance, cost: np.ndarray, index: np.ndarray,
                 status: np.ndarray):
        self.packed = packed
        self.cost = np.asarray(cost, dtype=np.float64)
        self.index = np.asarray(index, dtype=np.uint64)
        self.status = np.asarray(status, dtype=np.int32)

    def __len__(self):
        return int(self.status.size)

    def __getitem__(self, j):
        if not -len(self) <= j < len(self):
            raise IndexError(j)
        from .distributed import decode_index
        st = int(self.status[j])
        if st != abi.GP_OK:
            return abi._ERRORS.get(st, D.GeopipeError)(f"snapshot {j}: status {st}")
        p = self.packed
        order, counts, bm = decode_index(int(self.index[j]), p)
        nm = len(p.micros)
        return (float(self.cost[j]), [p.fg_ids[f] for f in order], counts,
                p.batches[bm // nm], p.micros[bm % nm])


def replan_snapshots(model, topology, groups, config, bandwidths: np.ndarray,
                     engine: Optional[Engine] = None, detail: bool = False):
    """Exact re-plan per snapshot.

    Returns, per snapshot, either a SearchResult (``detail=True``: a list of
    plan, splits and CostBreakdown, as ``exhaustive_plan`` on the rebuilt
    topology returns them) or (default) a :class:`SnapshotPlans` whose item j
    is the tuple ``(cost, order_ids, counts, b, m)``; snapshots whose re-plan
    raises carry the exception instance instead.
    """
    from .engine import best_fields
    packed = packed_instance(model, topology, groups, config.bottleneck_factor)
    eng = (engine or default_engine()).load(packed)
    bests, status = eng.replan_snapshots(bandwidths)
    if not detail:
        cost, index = best_fields(bests, bandwidths.shape[0])
        return SnapshotPlans(packed, cost, index, status)
    out: List = []
    k = packed.n_fgs
    nm = len(packed.micros)
    for i in range(bandwidths.shape[0]):
        st = int(status[i])
        if st != abi.GP_OK:
            cls = abi._ERRORS.get(st, D.GeopipeError)
            out.append(cls(f"snapshot {i}: status {st}"))
            continue
        b = bests[i]
        order = [int(x) for x in b.order[:k]]
        counts = [int(x) for x in b.counts[:k]]
        bm = b.batch_index * nm + b.micro_index
        if not detail:
            out.append((b.cost, [packed.fg_ids[f] for f in order], counts,
                        packed.batches[b.batch_index], packed.micros[b.micro_index]))
            continue
        eng.set_bandwidth(bandwidths[i])
        plan, breakdown, feasible = assemble(packed, eng, np.array(order, np.uint8),
                                             np.array(counts, np.uint8), bm)
        if breakdown is None:
            out.append(D.NoFeasiblePlanError(f"snapshot {i}: no feasible plan"))
        else:
            out.append(D.SearchResult(plan=plan, breakdown=breakdown, best_cost_trace=[b.cost],
                                      evaluated=int(b.evaluated)))
    if detail:
        eng.reset_bandwidth()
    return out


def snapshot_topology(topology, p_t: np.ndarray, bandwidth: Optional[np.ndarray] = None):
    """The topology with every link's p_t (and bandwidth) replaced by the
    snapshot's ``[D, D]`` matrices in string-sorted id order; latency kept."""
    ids = sorted(d.id for d in topology.devices)
    pos = {d: i for i, d in enumerate(ids)}
    links = {}
    for key, info in topology.links.items():
        u, v = tuple(key)
        i, j = pos[u], pos[v]
        links[key] = D.LinkInfo(
            metric=D.CommMetric(p_t=float(p_t[i, j])), latency_seconds=info.latency_seconds,
            bandwidth_bytes_per_s=float(bandwidth[i, j]) if bandwidth is not None
            else info.bandwidth_bytes_per_s)
    return D.ClusterTopology(devices=topology.devices, compute=topology.compute, links=links)


def replan_regrouped(model, topology, config, p_t_snapshots, bandwidth_snapshots=None,
                     threshold_net: float = 0.3, threshold_compute: float = 0.3,
                     engine: Optional[Engine] = None):
    """Re-plan per snapshot when p_t changes too:
    every snapshot is regrouped on the GPU (K7, group_first_level +
    group_second_level) and then re-planned exactly (exhaustive_plan through
    the engine).  Returns one SearchResult - or the exception the reference
    would raise - per snapshot, plus the GroupIndex used."""
    from .grouping import regroup_snapshots
    from .planner import exhaustive_plan
    eng = engine or default_engine()
    pts = np.asarray(p_t_snapshots, dtype=np.float64)
    bws = None if bandwidth_snapshots is None else np.asarray(bandwidth_snapshots, np.float64)
    groupings = regroup_snapshots(topology, pts, bws, threshold_net, threshold_compute,
                                  engine=eng)
    out = []
    for s, (_, _, gi) in enumerate(groupings):
        topo_s = snapshot_topology(topology, pts[s], None if bws is None else
                                   np.broadcast_to(bws, pts.shape)[s])
        try:
            out.append((exhaustive_plan(model, topo_s, gi, config, engine=eng), gi))
        except D.GeopipeError as e:
            out.append((e, gi))
    return out


def set_partitions(r: int):
    """Set partitions of r labelled blocks as restricted-growth strings in
    lexicographic order ({abc}, {ab|c}, {ac|b}, {a|bc}, {a|b|c} for r = 3)."""
    out = []

    def rec(prefix, top):
        if len(prefix) == r:
            out.append(list(prefix))
            return
        for v in range(top + 2):
            rec(prefix + [v], max(top, v))
    rec([0], 0)
    return out


def region_grouping_sweep(model, topology, regions: Sequence[Sequence[str]], config,
                          threshold_compute: float = 0.3, engine: Optional[Engine] = None):
    """C2 region-grouping sweep: for every set partition of the
    regions (restricted-growth order), first-level groups = unions of the
    regions of a block (built as group_first_level would), second level by
    group_second_level, then one exact exhaustive_plan.  Returns
    ``(results, best)``: per grouping ``(blocks, SearchResult | exception)``
    and the index of the sweep optimum, the minimum of
    ``(cost, grouping index)`` (ties inside a grouping are already broken by
    exhaustive_plan's key)."""
    from .grouping import fixed_hierarchy
    from .planner import exhaustive_plan
    eng = engine or default_engine()
    results = []
    best = None
    for gi, rgs in enumerate(set_partitions(len(regions))):
        blocks = [sorted(d for r, b in zip(regions, rgs) if b == v for d in r)
                  for v in range(max(rgs) + 1)]
        _, _, groups = fixed_hierarchy(topology, blocks, threshold_compute, engine=eng)
        try:
            res = exhaustive_plan(model, topology, groups, config, engine=eng)
        except D.GeopipeError as e:
            results.append((blocks, e))
            continue
        results.append((blocks, res))
        key = (res.breakdown.plan_cost, gi)
        if best is None or key < best[0]:
            best = (key, gi)
    return results, (best[1] if best is not None else None)
