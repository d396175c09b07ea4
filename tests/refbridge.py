"""Bridge to the unmodified reference package (``geopipe``) - test infra only.

The reference is pure-stdlib Python under ``/root/reference/pkg/src``; it is
importable in the build container but absent on the GPU box, so everything
here is guarded by :data:`AVAILABLE`.  Tests that need the live reference skip
without it and fall back to the committed fixtures in ``tests/golden/``.
"""

from __future__ import annotations

import os
import sys

REF_SRC = "/root/reference/pkg/src"
AVAILABLE = os.path.isdir(os.path.join(REF_SRC, "geopipe"))

if AVAILABLE and REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)


def geopipe():
    import geopipe  # noqa: F401  (reference package)
    return geopipe


def build_reference(spec, multipliers=None, threshold=0.3):
    """Build (model, topology, groups) with the reference's own constructors.

    Links are ``LinkMeasurement(alpha=1e8/bw, beta=lat, m=1e8, latency=lat,
    bandwidth=bw*mult)`` and groups come from ``group_first_level`` /
    ``group_second_level`` (src/grouping.py:146-228) - the real thing.
    """
    gp = geopipe()
    from geopipe.timing import GroupIndex
    devs = [gp.DeviceSpec(id=i, memory_bytes=mem,
                          benchmark_times=(("bench", 1.0 / p_c),))
            for i, _, _, p_c, mem in spec.devices()]
    meas = []
    for u, v, lat, bw in spec.links():
        eff = bw
        if multipliers is not None:
            eff = bw * multipliers[(min(u, v), max(u, v))]
        meas.append(gp.LinkMeasurement(
            endpoints=frozenset((u, v)), alpha_seconds=1e8 / bw,
            beta_seconds=lat, payload_bytes_m=1e8, latency_seconds=lat,
            bandwidth_bytes_per_s=eff))
    topo = gp.build_topology(devs, meas)
    fgs = gp.group_first_level(topo, threshold)
    sgs = {fg.id: gp.group_second_level(fg, topo, threshold) for fg in fgs}
    groups = GroupIndex.build(fgs, sgs)
    layers = tuple(gp.LayerSpec(*row) for row in spec.layers)
    model = gp.ModelSpec(layers=layers,
                         global_batch_candidates=tuple(spec.batches),
                         microbatch_candidates=tuple(spec.micros))
    return model, topo, groups
