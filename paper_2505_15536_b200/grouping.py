"""Two-level device grouping on the GPU (kernel K7) - ``group_first_level`` /
``group_second_level`` of the reference (src/grouping.py:85-228), batched
over topology snapshots.

Devices are ranked in string-sorted id order (``ClusterTopology.device_ids``,
src/profiling.py:191); tuples of sorted ids then compare like arrays of
ranks, which is how the reference's heap breaks key ties.  The device kernel
replays the reference's greedy merge order exactly: a popped pair is the
live pair with the smallest ``(key, a, b)``; a merge creates the pairs of
the new group with every other live group; a failed merge predicate discards
the pair for good.  Keys and merge values are the reference's sums
(CPython 3.12 ``sum``) in the reference's operand order.

Per snapshot the caller supplies ``p_t`` (and optionally the link
bandwidths used for ``min_intra_bandwidth``); ``p_c`` is shared.  This is
the "regroup per snapshot when p_t changes" step of SURVEY.md §8(f) rank 2.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import abi
from . import domain as D


@dataclass(frozen=True)
class Hierarchy:
    """Grouping of one snapshot in rank order (see :func:`topology_arrays`)."""
    fg_of: np.ndarray          # [D] first-level group index (sorted-tuple order)
    sg_of: np.ndarray          # [D] second-level group index within its FG
    fg_intra: np.ndarray       # [n_fg] intra_metric, NaN for singletons
    fg_capacity: np.ndarray    # [n_fg] aggregate_capacity
    fg_min_bw: np.ndarray      # [n_fg] min_intra_bandwidth, NaN for singletons
    sg_capacity: np.ndarray    # [n_sg] aggregate_capacity, FG-major


def topology_arrays(topology):
    """(ids, p_t[D,D], bandwidth[D,D], p_c[D]) in string-sorted id order."""
    ids = sorted(d.id for d in topology.devices)
    n = len(ids)
    pos = {d: i for i, d in enumerate(ids)}
    pt = np.zeros((n, n), dtype=np.float64)
    bw = np.zeros((n, n), dtype=np.float64)
    for key, info in topology.links.items():
        u, v = tuple(key)
        i, j = pos[u], pos[v]
        pt[i, j] = pt[j, i] = info.metric.p_t
        bw[i, j] = bw[j, i] = info.bandwidth_bytes_per_s
    pc = np.array([topology.p_c(d) for d in ids], dtype=np.float64)
    return ids, pt, bw, pc


def to_groups(ids: Sequence[str], h: Hierarchy):
    """Hierarchy -> (FirstLevelGroup list, {fg id: SecondLevelGroup list},
    GroupIndex) mirrors, ids ``fg{i}`` / ``fg{i}.sg{j}`` as the reference
    names them (src/grouping.py:183,222)."""
    n_fg = len(h.fg_capacity)
    fgs, sgs_by_fg = [], {}
    base = 0
    for f in range(n_fg):
        members = tuple(ids[d] for d in np.nonzero(h.fg_of == f)[0])
        fid = f"fg{f}"
        intra = float(h.fg_intra[f])
        mb = float(h.fg_min_bw[f])
        fgs.append(D.FirstLevelGroup(
            id=fid, member_device_ids=members,
            intra_metric=None if len(members) < 2 else intra,
            aggregate_capacity=float(h.fg_capacity[f]),
            min_intra_bandwidth=None if len(members) < 2 else mb))
        idx = np.nonzero(h.fg_of == f)[0]
        n_sg = int(h.sg_of[idx].max()) + 1
        sgs = []
        for j in range(n_sg):
            sm = tuple(ids[d] for d in idx if h.sg_of[d] == j)
            sgs.append(D.SecondLevelGroup(id=f"{fid}.sg{j}", parent_fg_id=fid,
                                          member_device_ids=sm,
                                          aggregate_capacity=float(h.sg_capacity[base + j])))
        base += n_sg
        sgs_by_fg[fid] = sgs
    return fgs, sgs_by_fg, D.GroupIndex.build(fgs, sgs_by_fg)


def group_hierarchies(p_t, bandwidth, p_c, threshold_net=0.3, threshold_compute=0.3,
                      engine=None) -> List[Hierarchy]:
    """K7: grouping of every snapshot ``p_t[s]`` (rank order) on the GPU."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    fg_of, sg_of, nf, ns, fi, fc, fb, sc = eng.group_snapshots(
        p_t, bandwidth, p_c, threshold_net, threshold_compute)
    return [Hierarchy(fg_of[s], sg_of[s], fi[s, :nf[s]], fc[s, :nf[s]], fb[s, :nf[s]],
                      sc[s, :ns[s]]) for s in range(len(nf))]


def group_first_level(topology, threshold: float = 0.3, engine=None):
    """Drop-in for src/grouping.py:146-190 (the second level is computed
    alongside and dropped)."""
    return build_hierarchy(topology, threshold, 0.3, engine)[0]


def build_hierarchy(topology, threshold_net: float = 0.3, threshold_compute: float = 0.3,
                    engine=None):
    """(first-level groups, {fg id: second-level groups}, GroupIndex) of one
    topology (src/grouping.py:231-241 plus GroupIndex.build)."""
    if not topology.devices:
        raise D.EmptyClusterError("topology has no devices")
    if not 0 < threshold_net < 1 or not 0 < threshold_compute < 1:
        raise ValueError("threshold must lie in (0, 1)")
    ids, pt, bw, pc = topology_arrays(topology)
    (h,) = group_hierarchies(pt, bw, pc, threshold_net, threshold_compute, engine)
    return to_groups(ids, h)


def regroup_snapshots(topology, p_t_snapshots, bandwidth_snapshots=None,
                      threshold_net: float = 0.3, threshold_compute: float = 0.3, engine=None):
    """Grouping per snapshot: ``p_t_snapshots[s]`` / ``bandwidth_snapshots[s]``
    ([D, D] in string-sorted id order) replace the topology's link metric and
    bandwidth; returns one ``(fgs, sgs_by_fg, GroupIndex)`` per snapshot."""
    ids, _, bw0, pc = topology_arrays(topology)
    pts = np.asarray(p_t_snapshots, dtype=np.float64)
    bws = bw0 if bandwidth_snapshots is None else np.asarray(bandwidth_snapshots, np.float64)
    hs = group_hierarchies(pts, bws, pc, threshold_net, threshold_compute, engine)
    return [to_groups(ids, h) for h in hs]


def fixed_hierarchy(topology, blocks: Sequence[Sequence[str]], threshold_compute: float = 0.3,
                    engine=None):
    """(fgs, sgs_by_fg, GroupIndex) for a GIVEN partition of the devices into
    first-level groups (``blocks`` of device ids): FirstLevelGroup fields as
    ``group_first_level`` builds them (sorted member tuples, ids over the
    sorted tuples, src/grouping.py:179-189) and ``group_second_level`` per
    group - on the GPU (SURVEY App. D region-grouping sweep)."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    ids, pt, bw, pc = topology_arrays(topology)
    pos = {d: i for i, d in enumerate(ids)}
    tuples = sorted(tuple(sorted(b)) for b in blocks)
    fg_of = np.full(len(ids), 0xffff, np.uint16)
    for f, members in enumerate(tuples):
        for d in members:
            if fg_of[pos[d]] != 0xffff:
                raise D.InputFileError(f"device {d} in two groups")
            fg_of[pos[d]] = f
    if (fg_of == 0xffff).any():
        raise D.InputFileError("partition does not cover every device")
    sg_of, ns, fi, fc, fb, sc = eng.group_fixed(pt, bw, pc, fg_of, len(tuples), threshold_compute)
    h = Hierarchy(fg_of, sg_of, fi, fc, fb, sc)
    return to_groups(ids, h)
