"""Serialize planner instances and results to JSON fixtures (exact floats).

Instances are stored with every derived value the reference computed (p_c,
p_t, link latency/bandwidth, group capacities and min bandwidths) so the GPU
box can rebuild them as :mod:`paper_2505_15536_b200.domain` mirrors without
the reference.  ``json`` writes floats with ``repr`` - an exact round trip.
"""

from __future__ import annotations

import json
import math
import os

from paper_2505_15536_b200 import domain as D

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _f(x):
    if x is None:
        return None
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return float(x)


def _uf(x):
    if x is None:
        return None
    if isinstance(x, str):
        return float(x)
    return float(x)


def instance_to_dict(model, topo, groups):
    return {
        "layers": [[l.fwd_flops, l.bwd_input_flops, l.bwd_weight_flops,
                    l.activation_out_bytes, l.param_bytes] for l in model.layers],
        "batches": list(model.global_batch_candidates),
        "micros": list(model.microbatch_candidates),
        "devices": [[d.id, d.memory_bytes, topo.p_c(d.id)] for d in topo.devices],
        "links": sorted([sorted(k)[0], sorted(k)[1], v.metric.p_t, v.latency_seconds,
                         v.bandwidth_bytes_per_s] for k, v in topo.links.items()),
        "fgs": [[fg.id, list(fg.member_device_ids), fg.intra_metric,
                 fg.aggregate_capacity, fg.min_intra_bandwidth]
                for fg in groups.fgs.values()],
        "sgs": {f: [[sg.id, list(sg.member_device_ids), sg.aggregate_capacity]
                    for sg in v] for f, v in groups.sgs_by_fg.items()},
    }


def instance_from_dict(doc):
    layers = tuple(D.LayerSpec(*row) for row in doc["layers"])
    model = D.ModelSpec(layers=layers, global_batch_candidates=tuple(doc["batches"]),
                        microbatch_candidates=tuple(doc["micros"]))
    devices = tuple(D.DeviceSpec(id=i, memory_bytes=mem) for i, mem, _ in doc["devices"])
    compute = {i: D.ComputeMetric(p_c=pc) for i, _, pc in doc["devices"]}
    links = {frozenset((u, v)): D.LinkInfo(metric=D.CommMetric(p_t=pt), latency_seconds=lat,
                                           bandwidth_bytes_per_s=bw)
             for u, v, pt, lat, bw in doc["links"]}
    topo = D.ClusterTopology(devices=devices, compute=compute, links=links)
    fgs = [D.FirstLevelGroup(id=i, member_device_ids=tuple(m), intra_metric=im,
                             aggregate_capacity=cap, min_intra_bandwidth=mb)
           for i, m, im, cap, mb in doc["fgs"]]
    sgs = {f: [D.SecondLevelGroup(id=i, parent_fg_id=f, member_device_ids=tuple(m),
                                  aggregate_capacity=cap) for i, m, cap in v]
           for f, v in doc["sgs"].items()}
    return model, topo, D.GroupIndex.build(fgs, sgs)


def plan_to_dict(plan):
    return {
        "batch_b": plan.batch_b, "microbatch_m": plan.microbatch_m,
        "stages": [[s.fg_id, s.layer_start, s.layer_end, s.intra_split.kind.value,
                    [list(p) for p in s.intra_split.parts]] for s in plan.stages],
    }


def breakdown_to_dict(bd):
    return {"plan_cost": _f(bd.plan_cost),
            "per_stage": [[_f(c.fill_seconds), _f(c.run_seconds), _f(c.residual_seconds),
                           _f(c.collective_seconds)] for c in bd.per_stage]}


def result_to_dict(res):
    return {"plan": plan_to_dict(res.plan), "breakdown": breakdown_to_dict(res.breakdown),
            "trace": [_f(x) for x in res.best_cost_trace], "evaluated": res.evaluated}


def normalize_result(res):
    """Comparable form of a SearchResult from either implementation."""
    return json.loads(json.dumps(result_to_dict(res)))


def save(name, doc):
    os.makedirs(GOLDEN, exist_ok=True)
    with open(os.path.join(GOLDEN, name), "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def exists(name):
    return os.path.exists(os.path.join(GOLDEN, name))
