"""Deterministic topologies for the grouping (K7) parity tests.

Each case is rebuilt from its name alone (seeded ``random.Random``), so the
committed golden file ``tests/golden/grouping.json`` holds only the
reference's outputs.  Matrices are in string-sorted id order (rank order).
"""

from __future__ import annotations

import random

import numpy as np


def _rand(seed):
    r = random.Random(seed)
    n = r.randint(2, 40)
    pt = np.zeros((n, n)); bw = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            pt[i, j] = pt[j, i] = r.uniform(0.005, 2.0)
            bw[i, j] = bw[j, i] = r.uniform(1e8, 1e10)
    pc = np.array([r.uniform(0.5, 20.0) for _ in range(n)])
    return pt, bw, pc, r.choice([0.1, 0.3, 0.5, 0.9]), r.choice([0.1, 0.3, 0.6])


def _clustered(seed, n=None):
    r = random.Random(1000 + seed)
    n = n or r.randint(2, 48)
    ncl = r.randint(1, 7)
    cl = [r.randrange(ncl) for _ in range(n)]
    pt = np.zeros((n, n)); bw = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            same = cl[i] == cl[j]
            pt[i, j] = pt[j, i] = r.choice([1.0, 1.0, 1.1]) if same else r.choice([5.0, 6.0, 9.0])
            bw[i, j] = bw[j, i] = r.choice([1e9, 2e9]) if same else r.choice([1e8, 5e7])
    pc = np.array([r.choice([1.0, 2.0, 4.0, 5.0, 10.0]) for _ in range(n)])
    return pt, bw, pc, r.choice([0.1, 0.3, 0.5]), r.choice([0.1, 0.3, 0.6])


def _instance(name, jitter, snap=None):
    from paper_2505_15536_b200 import instances as I
    from paper_2505_15536_b200.grouping import topology_arrays
    _, topo, _ = I.load(name, jitter)
    _, pt, bw, pc = topology_arrays(topo)
    if snap is not None:
        # per-region-pair p_t degradation, and in odd snapshots one region's
        # links to half of its devices degraded (the region splits)
        spec = I.config(name, jitter)
        region = {i: rg for i, rg, _, _, _ in spec.devices()}
        ids = sorted(region)
        r = random.Random(77 + snap)
        regs = sorted(set(region.values()))
        fac = {(a, b): (r.uniform(1.0, 3.0) if r.random() < 0.5 else 1.0)
               for a in regs for b in regs if a <= b}
        hit = r.choice(regs) if snap % 2 else None
        slow = {d for d in ids if region[d] == hit and r.random() < 0.5}
        pt = pt.copy()
        n = len(ids)
        for i in range(n):
            for j in range(i + 1, n):
                a, b = sorted((region[ids[i]], region[ids[j]]))
                f = fac[(a, b)]
                if ids[i] in slow or ids[j] in slow:
                    f *= 2.5
                pt[i, j] = pt[j, i] = pt[i, j] * f
    return pt, bw, pc, 0.3, 0.3


def names():
    out = [f"rand{s}" for s in range(120)] + [f"clus{s}" for s in range(120)]
    out += [f"{c}{'j' if j else ''}" for c in ("c1", "c2", "c4") for j in (0, 1)]
    out += [f"c4snap{s}" for s in range(12)] + [f"c2snap{s}" for s in range(4)]
    out += ["big0", "big1"]
    return out


def build(name):
    """(p_t, bandwidth, p_c, threshold_net, threshold_compute)."""
    if name.startswith("rand"):
        return _rand(int(name[4:]))
    if name.startswith("clus"):
        return _clustered(int(name[4:]))
    if name.startswith("big"):
        return _clustered(500 + int(name[3:]), n=160 if name == "big0" else 256)
    if name[2:6] == "snap":
        return _instance(name[:2], False, int(name[6:]))
    return _instance(name[:2], name.endswith("j"))
