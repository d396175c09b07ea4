"""Multi-GPU exhaustive re-plan: item sharding + a 16-byte tuple arg-min.

One process per GPU (torch.distributed; NCCL on B200s, gloo for the CPU
tests).  The exhaustive space of `exhaustive_plan` (src/planner.py:389-392)
is partitioned into (micro-batch, stage order) ITEMS, each covering every
batch size and every layer cut; rank r evaluates the contiguous item range
``shard_items(n_items, world, r)`` on its own GPU (K3 sweep) with no
data-path communication.  The only exchange is the final arg-min of one
``(cost bits, tie)`` pair per rank, where ``tie`` orders candidates exactly
as the reference's key ``(cost, (order, cuts))`` with earliest-(b, m)
tie-break does: non-negative doubles and +inf order like
their IEEE bit patterns, so the pair compares as two int64.
"""

from __future__ import annotations

import math
import struct
from typing import Callable, Optional, Tuple

import numpy as np

from . import domain as D

NO_KEY = (math.inf, (1 << 63) - 1)


def shard_items(n_items: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced item range of ``rank``."""
    return n_items * rank // world, n_items * (rank + 1) // world


def space_dims(n_layers: int, k: int, n_batch: int, n_micro: int):
    """(NC, NP, n_items) of the exhaustive space."""
    NC = math.comb(n_layers - 1, k - 1) if k <= n_layers else 0
    NP = math.factorial(k)
    return NC, NP, (n_micro * NP if NC else 0)


def tie_of_index(index: int, NC: int, NP: int, nbm: int) -> int:
    """Global enumeration index -> tie rank ((order rank * NC + cuts rank) * |B||M| + bm)."""
    comp = index % NC
    r = index // NC
    perm = r % NP
    bm = r // NP
    return (perm * NC + comp) * nbm + bm


def index_of_tie(tie: int, NC: int, NP: int, nbm: int) -> int:
    bm = tie % nbm
    pc = tie // nbm
    return (bm * NP + pc // NC) * NC + pc % NC


def _cost_bits(cost: float) -> int:
    return struct.unpack("<q", struct.pack("<d", cost))[0]


def _bits_cost(bits: int) -> float:
    return struct.unpack("<d", struct.pack("<q", bits))[0]


def reduce_key(key: Tuple[float, int], group=None, device=None) -> Tuple[float, int]:
    """All-gather one (cost, tie) per rank and return the global minimum."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return key
    t = torch.tensor([_cost_bits(key[0]), key[1]], dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    keys = [(int(o[0]), int(o[1])) for o in out]
    bits, tie = min(keys)
    return _bits_cost(bits), tie


def sharded_argmin(evaluate_items: Callable[[int, int], Tuple[float, int]], n_items: int,
                   group=None, device=None) -> Tuple[float, int]:
    """Global (cost, tie) arg-min; ``evaluate_items(lo, hi)`` is this rank's
    local arg-min over items [lo, hi) (the engine on a GPU, the oracle in
    CPU tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_items(n_items, world, rank)
    key = evaluate_items(lo, hi) if hi > lo else NO_KEY
    return reduce_key(key, group, device)


def decode_candidate(tie: int, NC: int, NP: int, nbm: int, n_layers: int, k: int):
    """tie -> (order indices, counts, bm) - integer unranking on the host."""
    bm = tie % nbm
    pc = tie // nbm
    perm_rank, comp = pc // NC, pc % NC
    pool = list(range(k))
    order = []
    for i in range(k):
        f = math.factorial(k - 1 - i)
        q, perm_rank = divmod(perm_rank, f)
        order.append(pool.pop(q))
    counts = []
    prev, rem = 0, comp
    for j in range(1, k):
        q = prev + 1
        while True:
            cnt = math.comb(n_layers - q - 1, k - 1 - j)
            if rem < cnt:
                break
            rem -= cnt
            q += 1
        counts.append(q - prev)
        prev = q
    counts.append(n_layers - prev)
    return order, counts, bm


def exhaustive_plan_sharded(model, topology, groups, config, engine=None, group=None):
    """``exhaustive_plan`` over all ranks of ``group``: every rank returns the
    same SearchResult (the reference's, bit for bit)."""
    import torch
    from .engine import default_engine
    from .layout import PackedInstance
    from .planner import assemble
    packed = PackedInstance(model, topology, groups, config.bottleneck_factor)
    eng = (engine or default_engine(torch.cuda.current_device())).load(packed)
    k = packed.n_fgs
    NC, NP, n_items = space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    if n_items == 0:
        raise D.NoFeasiblePlanError("no feasible plan in exhaustive sweep")

    def local(lo, hi):
        b = eng.argmin_items(lo, hi)
        return b.cost, tie_of_index(b.index, NC, NP, nbm)

    cost, tie = sharded_argmin(local, n_items, group, device=torch.device("cuda"))
    order, counts, bm = decode_candidate(tie, NC, NP, nbm, packed.n_layers, k)
    plan, breakdown, feasible = assemble(packed, eng, np.array(order, np.uint8),
                                         np.array(counts, np.uint8), bm)
    if breakdown is None:
        raise D.NoFeasiblePlanError("no feasible plan in exhaustive sweep")
    total = nbm * NP * NC
    return D.SearchResult(plan=plan, breakdown=breakdown, best_cost_trace=[cost],
                          evaluated=total)
