"""Test helpers: golden cases and reference-order candidate enumeration.

Enumeration follows exhaustive_plan (src/planner.py:389-392, 406-413):
(b, m) major, then itertools.permutations of the sorted group ids, then
compositions in lexicographic order.  Re-implemented here (no reference
needed) so the GPU box can enumerate too.
"""

from __future__ import annotations

import itertools
import os

import numpy as np

import golden_io as G
from paper_2505_15536_b200.layout import PackedInstance

CASES_ALL = sorted(f[:-5] for f in os.listdir(G.GOLDEN)
                   if f.endswith(".json") and os.path.exists(os.path.join(G.GOLDEN, f[:-5] + ".costs.npy")))


def compositions(total, parts):
    if parts == 1:
        yield (total,)
        return
    for first in range(1, total - parts + 2):
        for rest in compositions(total - first, parts - 1):
            yield (first,) + rest


def enumerate_encoded(packed: PackedInstance):
    """(order u8[N,k], counts u8[N,k], bm u8[N]) in enumeration order."""
    k = packed.n_fgs
    n = packed.n_layers
    perms = list(itertools.permutations(range(k)))
    comps = list(compositions(n, k))
    nbm = len(packed.batches) * len(packed.micros)
    N = nbm * len(perms) * len(comps)
    if N == 0:
        z = np.zeros((0, k), np.uint8)
        return z, z.copy(), np.zeros(0, np.uint8)
    P = np.array(perms, dtype=np.uint8)
    Cm = np.array(comps, dtype=np.uint8)
    order = np.tile(np.repeat(P, len(comps), axis=0), (nbm, 1))
    counts = np.tile(Cm, (nbm * len(perms), 1))
    bm = np.repeat(np.arange(nbm, dtype=np.uint8), len(perms) * len(comps))
    return order, counts, bm


def load_case(name):
    doc = G.load(f"{name}.json")
    model, topo, groups = G.instance_from_dict(doc["instance"])
    return doc, model, topo, groups


def golden_costs(name):
    c = np.load(os.path.join(G.GOLDEN, f"{name}.costs.npy"))
    s = np.load(os.path.join(G.GOLDEN, f"{name}.status.npy"))
    return c, s


def same_bits(a, b):
    """Bitwise float equality that treats every NaN alike (error slots)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return (a.view(np.uint64) == b.view(np.uint64)) | both_nan
