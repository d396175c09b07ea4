"""Multi-GPU re-planning: candidates and snapshots sharded over ranks.

One process per GPU (torch.distributed; NCCL on B200s, gloo for the CPU
tests); the units shard with no data-path communication:

* one exhaustive re-plan (`exhaustive_plan`, src/planner.py:389-392): the
  space is partitioned into (micro-batch, stage order) ITEMS, each covering
  every batch size and every layer cut; rank r sweeps the contiguous item
  range ``shard_items(n_items, world, r)`` on its own GPU (K3).  The only
  exchange is the final arg-min of one ``(first error, cost bits, tie)``
  triple per rank, where ``tie`` orders candidates exactly as the
  reference's key ``(cost, (order, cuts))`` with earliest-(b, m) tie-break
  does: non-negative doubles and +inf order like their
  IEEE bit patterns, so the key compares as int64s.  An erroring candidate
  on any rank makes every rank raise the error with the smallest index;
* a batch of bandwidth snapshots (the adapter's re-planning loop): snapshot
  j goes to the rank whose contiguous shard holds j (K6 per rank); the
  per-snapshot records (cost bits, winner index, status) are all-gathered.
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


NO_ERR = (1 << 63) - 1


def reduce_key(key: Tuple[float, int], group=None, device=None, err=None) -> Tuple[float, int]:
    """All-gather one (cost, tie) per rank - plus its first error, if any -
    and return the global minimum key.  When any rank met an erroring
    candidate, every rank raises the error of the smallest enumeration index
    (the one the reference's sequential loop meets first,
    src/planner.py:389-399), so no rank is left waiting in a collective."""
    import torch
    import torch.distributed as dist
    ek = NO_ERR if err is None else (int(err[0]) << 4) | int(err[1])
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        keys = [(ek, _cost_bits(key[0]), key[1])]
    else:
        t = torch.tensor([ek, _cost_bits(key[0]), key[1]], dtype=torch.int64, device=device)
        out = torch.empty(3 * dist.get_world_size(group), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(out, t, group=group)  # one collective, one D2H
        keys = [tuple(int(x) for x in row) for row in out.cpu().numpy().reshape(-1, 3)]
    e = min(k[0] for k in keys)
    if e != NO_ERR:
        from . import abi
        abi.raise_for(e & 15, f"candidate {e >> 4} raises status {e & 15}")
    bits, tie = min((k[1], k[2]) for k in keys)
    return _bits_cost(bits), tie


def sharded_argmin(evaluate_items: Callable[[int, int], tuple], n_items: int,
                   group=None, device=None) -> Tuple[float, int]:
    """Global (cost, tie) arg-min; ``evaluate_items(lo, hi)`` is this rank's
    local arg-min over items [lo, hi) as ``(cost, tie)`` or ``(cost, tie,
    err)`` with ``err = (first erroring index, status)`` or None (the engine
    on a GPU, the oracle in CPU tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_items(n_items, world, rank)
    r = evaluate_items(lo, hi) if hi > lo else NO_KEY
    key, err = (r[0], r[1]), (r[2] if len(r) > 2 else None)
    return reduce_key(key, group, device, err)


def gather_snapshot_records(local: np.ndarray, n_total: int, group=None, device=None) -> np.ndarray:
    """All-gather the per-snapshot records ``[n_local, 3]`` int64 (cost bits,
    enumeration index, status) of contiguous snapshot shards into the full
    ``[n_total, 3]`` table on every rank."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    width = max(1, -(-n_total // world))
    h = np.zeros((width, 3), dtype=np.int64)
    h[:local.shape[0]] = local
    buf = torch.from_numpy(h).to(device)
    out = torch.empty((world * width, 3), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)  # one collective, one D2H
    allrec = out.cpu().numpy().reshape(world, width, 3)
    rows = []
    for r in range(world):
        lo, hi = shard_items(n_total, world, r)
        rows.append(allrec[r, :hi - lo])
    return np.concatenate(rows) if rows else local


def replan_snapshots_sharded(model, topology, groups, config, bandwidths: np.ndarray,
                             engine=None, group=None):
    """Exact re-plan per bandwidth snapshot (replan.replan_snapshots), the
    snapshots partitioned by index over the ranks of ``group`` (contiguous
    shards); every rank returns the full list, one
    ``(cost, order_ids, counts, b, m)`` tuple or exception per snapshot."""
    import torch
    import torch.distributed as dist
    from . import abi
    from .engine import default_engine
    from .layout import packed_instance
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    packed = packed_instance(model, topology, groups, config.bottleneck_factor)
    eng = (engine or default_engine(torch.cuda.current_device())).load(packed)
    S = bandwidths.shape[0]
    lo, hi = shard_items(S, world, rank)
    if world > 1 and S >= world and packed.n_fgs >= 3:
        allrec = _replan_shard_device(eng, packed, bandwidths, S, lo, hi, world, group)
        if allrec is not None:
            return decode_snapshot_records(packed, allrec)
    rec = np.zeros((hi - lo, 3), dtype=np.int64)
    if hi > lo:
        from .engine import best_fields
        bests, status = eng.replan_snapshots(bandwidths[lo:hi])
        cost, index = best_fields(bests, hi - lo)
        rec[:, 0] = cost.view(np.int64)
        rec[:, 1] = index.view(np.int64)
        rec[:, 2] = status
    allrec = gather_snapshot_records(rec, S, group, torch.device("cuda"))
    return decode_snapshot_records(packed, allrec)


def _replan_shard_device(eng, packed, bandwidths, S, lo, hi, world, group):
    """The device-resident form of the sharded snapshot re-plan: this rank's
    matrices H2D, gp_replan_snapshots_async (K6) into device keys + flags,
    one NCCL all-gather of the [width, 3] records straight from device
    memory and one D2H - no host round trip between the sweep and the
    collective.  Snapshots whose tables raise (flags) are redone by their
    owner through the status-tracking gp_replan_snapshots and shared with a
    second gather (every rank sees the same flags, so the collectives stay
    matched).  None on every rank when any rank's asynchronous re-plan was
    refused (its records carry -1 flags through the same all-gather); the
    caller then takes the host-staged path on all ranks."""
    import torch
    import torch.distributed as dist
    from . import abi
    from .engine import best_fields
    n = hi - lo
    width = -(-S // world)
    Dn = bandwidths.shape[1]
    dev = torch.device("cuda", torch.cuda.current_device())
    key = (width, Dn, world)
    bufs = getattr(eng, "_shard_bufs", None)
    if bufs is None or bufs[0] != key:
        bufs = (key, torch.empty((width, Dn, Dn), dtype=torch.float64, device=dev),
                torch.zeros((width, 2), dtype=torch.int64, device=dev),
                torch.zeros(width, dtype=torch.int32, device=dev),
                torch.zeros((width, 3), dtype=torch.int64, device=dev),
                torch.empty((world * width, 3), dtype=torch.int64, device=dev))
        eng._shard_bufs = bufs
    _, d_bw, d_keys, d_flags, d_rec, d_out = bufs
    cur = torch.cuda.current_stream(dev)
    d_bw[:n].copy_(torch.from_numpy(np.ascontiguousarray(bandwidths[lo:hi], dtype=np.float64)),
                   non_blocking=True)
    est = torch.cuda.ExternalStream(eng.stream, device=dev)
    est.wait_stream(cur)
    ok = True
    try:
        eng.replan_snapshots_async(d_bw.data_ptr(), n, d_keys.data_ptr(), d_flags.data_ptr())
    except D.GeopipeError:
        ok = False  # e.g. an instance that needs the status path for every snapshot
    cur.wait_stream(est)
    if ok:
        d_rec[:n, :2].copy_(d_keys[:n])
        d_rec[:n, 2].copy_(d_flags[:n])
    else:
        d_rec[:, 2].fill_(-1)  # tells every rank: all take the host-staged path
    dist.all_gather_into_tensor(d_out, d_rec, group=group)
    allrec = d_out.cpu().numpy().reshape(world, width, 3)
    if (allrec[:, 0, 2] == -1).any():
        return None
    NC, NP, _ = space_dims(packed.n_layers, packed.n_fgs, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    rows = []
    for r in range(world):
        rlo, rhi = shard_items(S, world, r)
        rows.append(allrec[r, :rhi - rlo])
    recs = np.concatenate(rows)
    flags = recs[:, 2] != 0
    tie = recs[:, 1].view(np.uint64)
    empty = tie == np.uint64(0xFFFFFFFFFFFFFFFF)
    t = np.where(empty, np.uint64(0), tie)
    bm, pc = t % np.uint64(nbm), t // np.uint64(nbm)
    index = (bm * np.uint64(NP) + pc // np.uint64(NC)) * np.uint64(NC) + pc % np.uint64(NC)
    out = np.zeros((S, 3), dtype=np.int64)
    out[:, 0] = np.where(empty, 0, recs[:, 0])
    out[:, 1] = index.view(np.int64)
    out[:, 2] = np.where(empty, abi.GP_ERR_NO_FEASIBLE, abi.GP_OK)
    if flags.any():  # the owners redo their flagged snapshots with status tracking
        mine = [j for j in range(lo, hi) if flags[j]]
        loc = out[lo:hi].copy()
        for j in mine:
            bests, status = eng.replan_snapshots(bandwidths[j:j + 1])
            cost, idx = best_fields(bests, 1)
            loc[j - lo] = (cost.view(np.int64)[0], idx.view(np.int64)[0], status[0])
        out = gather_snapshot_records(loc, S, group, dev)
    return out


def decode_snapshot_records(packed, rec: np.ndarray):
    """Per-snapshot records -> replan.SnapshotPlans (item j = ``(cost,
    order_ids, counts, b, m)`` or the exception the reference would raise)."""
    from .replan import SnapshotPlans
    rec = np.ascontiguousarray(rec, dtype=np.int64)
    return SnapshotPlans(packed, rec[:, 0].view(np.float64), rec[:, 1].view(np.uint64),
                         rec[:, 2].astype(np.int32))


def decode_index(index: int, packed):
    """Enumeration index -> (order indices, counts, bm) of ``packed``'s space."""
    k, n = packed.n_fgs, packed.n_layers
    NC, NP, _ = space_dims(n, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    return decode_candidate(tie_of_index(index, NC, NP, nbm), NC, NP, nbm, n, k)


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
    from .layout import packed_instance
    from .planner import assemble
    packed = packed_instance(model, topology, groups, config.bottleneck_factor)
    eng = (engine or default_engine(torch.cuda.current_device())).load(packed)
    k = packed.n_fgs
    NC, NP, n_items = space_dims(packed.n_layers, k, len(packed.batches), len(packed.micros))
    nbm = len(packed.batches) * len(packed.micros)
    if n_items == 0:
        raise D.NoFeasiblePlanError("no feasible plan in exhaustive sweep")

    def local(lo, hi):
        from . import abi
        st, b, msg = eng.argmin_items_status(lo, hi)
        if st == abi.GP_OK:
            return b.cost, tie_of_index(b.index, NC, NP, nbm), None
        if st == abi.GP_ERR_NO_FEASIBLE:  # empty item range
            return NO_KEY[0], NO_KEY[1], None
        return NO_KEY[0], NO_KEY[1], (int(b.index), st)

    cost, tie = sharded_argmin(local, n_items, group, device=torch.device("cuda"))
    order, counts, bm = decode_candidate(tie, NC, NP, nbm, packed.n_layers, k)
    plan, breakdown, feasible = assemble(packed, eng, np.array(order, np.uint8),
                                         np.array(counts, np.uint8), bm)
    if breakdown is None:
        raise D.NoFeasiblePlanError("no feasible plan in exhaustive sweep")
    total = nbm * NP * NC
    return D.SearchResult(plan=plan, breakdown=breakdown, best_cost_trace=[cost],
                          evaluated=total)


class PeerGather:
    """All-gather of fixed-size per-rank device records through peer memory
    (C-ABI gp_peer_*): every rank's slot is stored into every rank's buffer
    over NVLink by one kernel, with a system-scope arrival counter the
    receiving GPU waits on - no NCCL call in the data path.  Used for the K6
    winners (16 B per snapshot) of a sharded snapshot batch.  ``ok`` is False
    on every rank when any rank could not set it up (callers fall back to
    NCCL's all-gather)."""

    def __init__(self, engine, slot_bytes: int, group=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from .engine import lib
        self.eng = engine
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.slot = (int(slot_bytes) + 15) // 16 * 16
        self.epoch = 0
        self._owned = C.c_void_p()
        self._opened = []
        handle = (C.c_char * 64)()
        ok = lib().gp_peer_alloc(engine.handle, 256 + 2 * self.world * self.slot, C.byref(self._owned),
                                 handle) == 0
        handles = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, bytes(handle) if ok else None, group=group)
        else:
            handles = [bytes(handle) if ok else None]
        ok = ok and all(h is not None for h in handles)
        bases = []
        for r, h in enumerate(handles):
            if not ok:
                break
            if r == self.rank:
                bases.append(self._owned.value)
                continue
            p = C.c_void_p()
            hb = (C.c_char * 64).from_buffer_copy(h)
            if lib().gp_peer_open(engine.handle, hb, C.byref(p)) != 0:
                ok = False
                break
            self._opened.append(p)
            bases.append(p.value)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
        if self.world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.ok = bool(flag.item())
        self._bases = (C.c_void_p * self.world)(*(bases if self.ok else [None] * self.world))

    @property
    def records(self) -> int:
        """Device address of the latest gather's slots (rank r's at + r *
        slot).  Epochs alternate between two tables, so the table stays valid
        until this rank's next-but-one gather; consume it (in stream order)
        before the next gather."""
        return self._owned.value + 256 + (self.epoch & 1) * self.world * self.slot

    def gather(self, d_src: int) -> None:
        """Asynchronous on the engine stream: slot_bytes from device address
        d_src into every rank's buffer, then wait for every rank's slot."""
        from .engine import _check, lib
        self.epoch += 1
        _check(lib().gp_peer_allgather(self.eng.handle, d_src, self.slot, self.rank, self.world,
                                        self._bases, self.epoch))

    def read(self) -> bytes:
        """The gathered slots (synchronises the engine stream); raises when a
        wait timed out (a rank's slot never arrived)."""
        import ctypes as C
        from . import domain as D
        from .engine import _check, lib
        head = (C.c_uint64 * 2)()
        _check(lib().gp_peer_read(self.eng.handle, self._owned.value, head, 16))
        if head[1]:
            raise D.DeviceError(f"peer all-gather: {head[1]} arrival(s) missing after the timeout")
        buf = (C.c_char * (self.world * self.slot))()
        _check(lib().gp_peer_read(self.eng.handle, self.records, buf, self.world * self.slot))
        return bytes(buf)

    def close(self, barrier=None) -> None:
        """Unmap the peers' buffers, wait for every rank to have done so
        (``barrier``, e.g. torch.distributed.barrier), free this one."""
        from .engine import lib
        for p in self._opened:
            lib().gp_peer_close(self.eng.handle, p, 0)
        self._opened = []
        if barrier is not None:
            barrier()
        if self._owned.value:
            lib().gp_peer_close(self.eng.handle, self._owned, 1)
            self._owned = type(self._owned)()
