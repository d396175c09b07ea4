"""Candidate enumeration helpers (host-side index bookkeeping, no costs).

The exhaustive space is enumerated as exhaustive_plan does
(src/planner.py:389-392, 406-413): (b, m) major, then permutations of the
sorted group ids, then compositions of the layers in lexicographic order.
These tables decode enumeration indices into explicit candidates for the
batch kernels (K2, K5).
"""

from __future__ import annotations

import itertools
import math

import numpy as np


def composition_table(n: int, k: int) -> np.ndarray:
    """All compositions of n into k positive parts, lexicographic, u8[NC, k]."""
    NC = math.comb(n - 1, k - 1)
    out = np.empty((NC, k), dtype=np.uint8)
    for r, cuts in enumerate(itertools.combinations(range(1, n), k - 1)):
        prev = 0
        for j, c in enumerate(cuts):
            out[r, j] = c - prev
            prev = c
        out[r, k - 1] = n - prev
    return out


def permutation_table(k: int) -> np.ndarray:
    return np.array(list(itertools.permutations(range(k))), dtype=np.uint8).reshape(-1, k)


def decode_indices(n: int, k: int, idx: np.ndarray, comps=None, perms=None):
    """Enumeration indices -> (order u8[N,k], counts u8[N,k], bm u8[N])."""
    comps = composition_table(n, k) if comps is None else comps
    perms = permutation_table(k) if perms is None else perms
    NC, NP = comps.shape[0], perms.shape[0]
    idx = np.asarray(idx, dtype=np.int64)
    comp = idx % NC
    r = idx // NC
    return perms[r % NP], comps[comp], (r // NP).astype(np.uint8)
