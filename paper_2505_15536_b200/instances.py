"""Synthetic planner instances built without the reference.

An instance is described by a neutral :class:`InstanceSpec` (layer cost table,
regions of device tiers, link parameters).  :func:`build` turns it into the
mirror objects of :mod:`.domain`, deriving every value the way the reference's
constructors do:

* ``p_c = 0.0 + 1.0 / (1.0 / p_c)``  - ``compute_capacity`` with one benchmark
  of time ``1/p_c`` and weight ``1/1`` (``src/profiling.py:100-113,159-164``);
* ``p_t = alpha + beta / m``          - ``comm_capability`` (``:95-97``);
* FG = region, SG = tier; ids ``fg{i}`` / ``fg{i}.sg{j}`` indexed over sorted
  member tuples, ``aggregate_capacity = sum(p_c)`` in member order and
  ``min_intra_bandwidth = min(bw)`` over sorted member pairs, as
  ``group_first_level`` / ``group_second_level`` produce them
  (``src/grouping.py:146-228``).  tests/test_instances.py proves the result
  equal, field by field, to the reference's own grouping of the same cluster.

Bandwidth snapshots (config C3) rescale ``bandwidth_bytes_per_s`` only, so
``p_t``, the grouping and the gateway pairs are unchanged.
"""

from __future__ import annotations

import itertools
import random
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import domain as D

LINK_PAYLOAD_M = 1e8


@dataclass
class InstanceSpec:
    name: str
    layers: List[Tuple[float, float, float, float, float]]
    batches: Tuple[int, ...]
    micros: Tuple[int, ...]
    # regions[r] = list of tiers; tier = list of (p_c, memory_bytes)
    regions: List[List[List[Tuple[float, float]]]]
    intra_bw: List[float]
    intra_lat: List[float]
    cross_bw: float
    cross_lat: float
    jitter_seed: int = 0

    # ---- derived device list (creation order) ----
    def devices(self) -> List[Tuple[str, int, int, float, float]]:
        out = []
        for r, tiers in enumerate(self.regions):
            k = 0
            for t, tier in enumerate(tiers):
                for p_c, mem in tier:
                    out.append((f"r{r}d{k:02d}", r, t, p_c, mem))
                    k += 1
        return out

    def links(self) -> List[Tuple[str, str, float, float]]:
        """(u, v, latency, bandwidth) per unordered pair, creation order."""
        rng = random.Random(self.jitter_seed)
        devs = self.devices()
        out = []
        for a, b in itertools.combinations(devs, 2):
            if a[1] == b[1]:
                bw, lat = self.intra_bw[a[1]], self.intra_lat[a[1]]
            else:
                bw, lat = self.cross_bw, self.cross_lat
            bw = bw * rng.uniform(0.9, 1.1)
            out.append((a[0], b[0], lat, bw))
        return out


# --------------------------------------------------------------------------
# layer tables (App. D)
# --------------------------------------------------------------------------

def transformer_layers(n, d, d_ff, seq, vocab, d_kv=None, gpt2=False,
                       jitter_seed: Optional[int] = None):
    if gpt2:
        P = 4 * d * d + 2 * d * d_ff
    else:
        P = 2 * d * d + 2 * d * d_kv + 3 * d * d_ff
    rows = []
    for i in range(n):
        fwd = float(2 * P * seq + 4 * seq * seq * d)
        param = float(2 * P)
        if i == 0:
            param += float(2 * vocab * d)
        if i == n - 1:
            fwd += float(2 * vocab * d * seq)
            param += float(2 * vocab * d)
        act = float(seq * d * 2)
        rows.append([fwd, fwd, fwd, act, param])
    if jitter_seed is not None:
        rng = random.Random(jitter_seed)
        for row in rows:
            for j in range(5):
                row[j] = row[j] * rng.uniform(0.9, 1.1)
    return [tuple(r) for r in rows]


GB = 1e9


def config(name: str, jitter: bool = False) -> InstanceSpec:
    """App. D configs ``c1``, ``c2``, ``c4`` (``jitter``: fields x U[0.9,1.1], seed 7)."""
    js = 7 if jitter else None
    if name == "c1":
        layers = transformer_layers(24, 1024, 4096, 512, 50257, gpt2=True,
                                    jitter_seed=js)
        regions = [
            [[(1.65e14, 24 * GB)], [(7.1e13, 24 * GB)]],
            [[(3.5e13, 10 * GB), (3.0e13, 10 * GB)]],
        ]
        return InstanceSpec("c1", layers, (128, 256), (8, 16, 32), regions,
                            intra_bw=[1.25e8, 1.25e8], intra_lat=[5e-4, 5e-4],
                            cross_bw=1.25e7, cross_lat=0.03)
    if name == "c2":
        layers = transformer_layers(32, 4096, 11008, 2048, 32000, d_kv=4096,
                                    jitter_seed=js)
        regions = [
            [[(9.89e14, 80 * GB)] * 4, [(3.12e14, 40 * GB)] * 2],
            [[(1.65e14, 24 * GB)] * 3, [(7.1e13, 24 * GB)] * 2],
            [[(3.5e13, 10 * GB)] * 5],
        ]
        return InstanceSpec("c2", layers, (128, 256), (8, 16, 32), regions,
                            intra_bw=[5e10, 1.25e9, 1.25e8],
                            intra_lat=[5e-6, 1e-4, 5e-4],
                            cross_bw=1.25e7, cross_lat=0.03)
    if name == "c4":
        layers = transformer_layers(80, 8192, 28672, 2048, 32000, d_kv=1024,
                                    jitter_seed=js)
        regions = [
            [[(2.25e15, 192 * GB)] * 8, [(9.89e14, 80 * GB)] * 8],
            [[(9.89e14, 80 * GB)] * 12, [(3.12e14, 80 * GB)] * 4],
            [[(1.65e14, 24 * GB)] * 8, [(7.1e13, 24 * GB)] * 8],
            [[(3.5e13, 16 * GB)] * 10, [(2.0e13, 8 * GB)] * 6],
        ]
        return InstanceSpec("c4", layers, (128, 256), (8, 16, 32), regions,
                            intra_bw=[5e10, 5e10, 1.25e9, 1.25e8],
                            intra_lat=[5e-6, 5e-6, 1e-4, 5e-4],
                            cross_bw=1.25e7, cross_lat=0.03)
    raise KeyError(name)


def many_group_config(k: int, n: int, seed: int, batches=(64, 128), micros=(8, 16),
                      jitter: bool = True) -> InstanceSpec:
    """k-region instances (k first-level groups) for the k >= 5 regime where
    the exhaustive space C(n-1, k-1) * k! explodes: each region holds one or
    two tiers of 1-2 devices (random p_c / memory), random intra-region
    bandwidth and latency, 100 Mb/s cross-region links at 30 ms."""
    rng = random.Random(seed)
    regions = []
    for _ in range(k):
        tiers = [[(rng.choice([3.5e13, 7.1e13, 1.65e14, 9.89e14]), rng.choice([8e9, 24e9, 80e9]))]
                 * rng.randint(1, 2)]
        if rng.random() < 0.5:
            tiers.append([(rng.choice([2.0e13, 3.12e14]), 24e9)])
        regions.append(tiers)
    layers = transformer_layers(n, 2048, 5504, 1024, 32000, d_kv=2048,
                                jitter_seed=seed if jitter else None)
    return InstanceSpec(f"k{k}n{n}s{seed}", layers, tuple(batches), tuple(micros), regions,
                        intra_bw=[rng.uniform(1e9, 5e10) for _ in range(k)],
                        intra_lat=[rng.uniform(1e-5, 1e-3) for _ in range(k)],
                        cross_bw=1.25e7, cross_lat=0.03, jitter_seed=seed)


def snapshot_multipliers(spec: InstanceSpec, j: int) -> Dict[Tuple[str, str], float]:
    """C3 snapshot ``j``: bandwidth multiplier per unordered device pair.

    Draw order (App. D): region pairs r1<r2 lexicographically, degraded with
    prob. 0.5 by U[0.4,0.6]; then same-region device pairs over
    ``combinations(sorted ids)`` with prob. 0.2 by U[0.8,1.0].
    """
    rng = random.Random(j)
    devs = spec.devices()
    region = {d[0]: d[1] for d in devs}
    nreg = len(spec.regions)
    cross = {}
    for r1, r2 in itertools.combinations(range(nreg), 2):
        cross[(r1, r2)] = rng.uniform(0.4, 0.6) if rng.random() < 0.5 else 1.0
    mult = {}
    ids = sorted(region)
    for u, v in itertools.combinations(ids, 2):
        ru, rv = region[u], region[v]
        if ru != rv:
            mult[(u, v)] = cross[(min(ru, rv), max(ru, rv))]
    for u, v in itertools.combinations(ids, 2):
        if region[u] == region[v]:
            mult[(u, v)] = rng.uniform(0.8, 1.0) if rng.random() < 0.2 else 1.0
    return mult


# --------------------------------------------------------------------------
# building mirror objects
# --------------------------------------------------------------------------

def build_model(spec: InstanceSpec) -> D.ModelSpec:
    return D.ModelSpec(
        layers=tuple(D.LayerSpec(*row) for row in spec.layers),
        global_batch_candidates=tuple(spec.batches),
        microbatch_candidates=tuple(spec.micros))


def build_topology(spec: InstanceSpec,
                   multipliers: Optional[Dict[Tuple[str, str], float]] = None
                   ) -> D.ClusterTopology:
    devs = spec.devices()
    devices = tuple(sorted(
        (D.DeviceSpec(id=i, memory_bytes=mem,
                      benchmark_times=(("bench", 1.0 / p_c),))
         for i, _, _, p_c, mem in devs), key=lambda d: d.id))
    compute = {}
    for d in devices:
        t = d.benchmark_times[0][1]
        compute[d.id] = D.ComputeMetric(p_c=0.0 + 1.0 / t)
    links = {}
    for u, v, lat, bw in spec.links():
        alpha = LINK_PAYLOAD_M / bw
        eff_bw = bw
        if multipliers is not None:
            eff_bw = bw * multipliers[(min(u, v), max(u, v))]
        links[frozenset((u, v))] = D.LinkInfo(
            metric=D.CommMetric(p_t=alpha + lat / LINK_PAYLOAD_M),
            latency_seconds=lat, bandwidth_bytes_per_s=eff_bw)
    return D.ClusterTopology(devices=devices, compute=compute, links=links)


def build_groups(spec: InstanceSpec, topo: D.ClusterTopology) -> D.GroupIndex:
    devs = spec.devices()
    regions: Dict[int, List[str]] = {}
    tiers: Dict[Tuple[int, int], List[str]] = {}
    for i, r, t, _, _ in devs:
        regions.setdefault(r, []).append(i)
        tiers.setdefault((r, t), []).append(i)
    member_sets = sorted(tuple(sorted(m)) for m in regions.values())
    fgs = []
    sgs_by_fg = {}
    for idx, members in enumerate(member_sets):
        fid = f"fg{idx}"
        pairs = list(itertools.combinations(sorted(members), 2))
        if len(members) < 2:
            intra, min_bw = None, None
        else:
            vals = [topo.p_t(u, v) for u, v in pairs]
            intra = sum(vals) / len(vals)
            min_bw = min(topo.bandwidth(u, v) for u, v in pairs)
        fgs.append(D.FirstLevelGroup(
            id=fid, member_device_ids=members, intra_metric=intra,
            aggregate_capacity=sum(topo.p_c(m) for m in members),
            min_intra_bandwidth=min_bw))
        r = next(rr for rr, mm in regions.items() if tuple(sorted(mm)) == members)
        sg_sets = sorted(tuple(sorted(m)) for (rr, _), m in tiers.items() if rr == r)
        sgs_by_fg[fid] = [
            D.SecondLevelGroup(id=f"{fid}.sg{j}", parent_fg_id=fid,
                               member_device_ids=sm,
                               aggregate_capacity=sum(topo.p_c(x) for x in sm))
            for j, sm in enumerate(sg_sets)]
    return D.GroupIndex.build(fgs, sgs_by_fg)


def build(spec: InstanceSpec, multipliers=None):
    """(model, topology, groups) mirror objects for ``spec``."""
    topo = build_topology(spec, multipliers)
    return build_model(spec), topo, build_groups(spec, topo)


def load(name: str, jitter: bool = False, snapshot: Optional[int] = None):
    spec = config(name, jitter)
    mult = snapshot_multipliers(spec, snapshot) if snapshot is not None else None
    return build(spec, mult)
