"""Batched input layout: reference objects -> structure-of-arrays tables.

:class:`PackedInstance` reads a ``(model, topology, groups, config)`` quadruple
(the reference's own objects or the mirrors in :mod:`.domain`) once and lays
it out as the flat fp64/u32 arrays of ``gp_instance`` (include/geopipe_b200.h):

* layers    : five fp64 columns ``[n]``                 (src/plans.py:12-30)
* devices   : ``p_c``, ``memory_bytes`` ``[D]`` in topology order, plus the
              rank of each id in string order           (src/profiling.py:125-156)
* links     : dense ``[D, D]`` p_t / latency / bandwidth (symmetric)
* groups    : first-level groups in sorted-id order (``sorted(groups.fgs)``,
              src/planner.py:384) as CSR over member device indices, with
              ``aggregate_capacity`` and ``min_intra_bandwidth``; second-level
              groups per first-level group in ``sgs_by_fg`` order as CSR
* (b, m)    : ``global_batch_candidates`` x ``microbatch_candidates``

No arithmetic on plan costs happens here - only gathering of the numbers the
reference objects already hold.  The packed arrays are what gp_ctx_load copies
to HBM (and what the test-only oracle consumes).
"""

from __future__ import annotations

import ctypes as C
from collections import OrderedDict
from typing import Dict, List

import numpy as np

from . import abi
from . import domain as D


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


_CACHE: "OrderedDict[tuple, PackedInstance]" = OrderedDict()
_CACHE_SIZE = 16


def packed_instance(model, topology, groups, bottleneck_factor: float = 1.25) -> "PackedInstance":
    """PackedInstance of a (model, topology, groups) triple, cached by object
    identity.  The reference's inputs are frozen and shareable
    (SURVEY.md §8(b)), so a triple seen before packs to the same arrays; the
    cache holds strong references, so an id is never reused while cached.
    This is what makes repeated drop-in calls on the same objects (the
    planner's and the adapter's re-plan loop) cost microseconds on the host."""
    key = (id(model), id(topology), id(groups), float(bottleneck_factor))
    hit = _CACHE.get(key)
    if hit is not None and hit.model is model and hit.topology is topology and hit.groups is groups:
        _CACHE.move_to_end(key)
        return hit
    p = PackedInstance(model, topology, groups, bottleneck_factor)
    _CACHE[key] = p
    while len(_CACHE) > _CACHE_SIZE:
        _CACHE.popitem(last=False)
    return p


class PackedInstance:
    def __init__(self, model, topology, groups, bottleneck_factor: float = 1.25):
        layers = model.layers
        n = len(layers)
        if n == 0:
            raise D.InputFileError("model has no layers")
        if n > abi.GP_MAX_LAYERS:
            raise D.InputFileError(f"{n} layers exceed the engine limit "
                                   f"{abi.GP_MAX_LAYERS}")
        self.model = model
        self.topology = topology
        self.groups = groups
        self.n_layers = n
        cols = np.array([[l.fwd_flops, l.bwd_input_flops, l.bwd_weight_flops,
                          l.activation_out_bytes, l.param_bytes] for l in layers],
                        dtype=np.float64)
        self.fwd = np.ascontiguousarray(cols[:, 0])
        self.bwd_in = np.ascontiguousarray(cols[:, 1])
        self.bwd_w = np.ascontiguousarray(cols[:, 2])
        self.act = np.ascontiguousarray(cols[:, 3])
        self.param = np.ascontiguousarray(cols[:, 4])
        self.batches = tuple(int(b) for b in model.global_batch_candidates)
        self.micros = tuple(int(m) for m in model.microbatch_candidates)
        self.batch = np.array(self.batches, dtype=np.int64)
        self.micro = np.array(self.micros, dtype=np.int64)
        if len(self.batches) * len(self.micros) > 255:
            raise D.InputFileError("at most 255 (batch, micro-batch) pairs")

        # devices in topology order
        self.device_ids: List[str] = [d.id for d in topology.devices]
        dev_index: Dict[str, int] = {d: i for i, d in enumerate(self.device_ids)}
        self.dev_index = dev_index
        Dn = len(self.device_ids)
        self.n_devices = Dn
        self.p_c = np.array([topology.p_c(d) for d in self.device_ids], dtype=np.float64)
        self.memory = np.array([d.memory_bytes for d in topology.devices], dtype=np.float64)
        order = sorted(range(Dn), key=lambda i: self.device_ids[i])
        self.id_rank = np.empty(Dn, dtype=np.uint32)
        for r, i in enumerate(order):
            self.id_rank[i] = r
        self.p_t = np.zeros((Dn, Dn), dtype=np.float64)
        self.lat = np.zeros((Dn, Dn), dtype=np.float64)
        self.bw = np.zeros((Dn, Dn), dtype=np.float64)
        links = topology.links
        nl = len(links)
        if nl:
            ends = [tuple(k) for k in links]
            infos = list(links.values())
            ii = np.fromiter((dev_index[e[0]] for e in ends), np.intp, nl)
            jj = np.fromiter((dev_index[e[-1]] for e in ends), np.intp, nl)
            for mat, vals in ((self.p_t, (x.metric.p_t for x in infos)),
                              (self.lat, (x.latency_seconds for x in infos)),
                              (self.bw, (x.bandwidth_bytes_per_s for x in infos))):
                v = np.fromiter(vals, np.float64, nl)
                mat[ii, jj] = v
                mat[jj, ii] = v

        # groups in sorted-id (string) order
        self.fg_ids: List[str] = sorted(groups.fgs)
        if len(self.fg_ids) > abi.GP_MAX_STAGES:
            raise D.InputFileError(f"{len(self.fg_ids)} first-level groups exceed "
                                   f"the engine limit {abi.GP_MAX_STAGES}")
        self.fg_pos = {f: i for i, f in enumerate(self.fg_ids)}
        fg_off, fg_mem, fg_cap, fg_bw, fg_has = [0], [], [], [], []
        sg_off_fg, sg_off, sg_mem, sg_cap = [0], [0], [], []
        self.sg_ids: List[List[str]] = []
        for f in self.fg_ids:
            fg = groups.fgs[f]
            members = list(fg.member_device_ids)
            if len(members) > abi.GP_MAX_MEMBERS:
                raise D.InputFileError(f"group {f} exceeds {abi.GP_MAX_MEMBERS} devices")
            fg_mem.extend(dev_index[d] for d in members)
            fg_off.append(len(fg_mem))
            fg_cap.append(float(fg.aggregate_capacity))
            mb = fg.min_intra_bandwidth
            fg_bw.append(float(mb) if mb is not None else 0.0)
            fg_has.append(0 if mb is None else 1)
            sgs = list(groups.sgs_by_fg[f])
            if len(sgs) > abi.GP_MAX_SGS:
                raise D.InputFileError(f"group {f} has more than {abi.GP_MAX_SGS} subgroups")
            self.sg_ids.append([sg.id for sg in sgs])
            for sg in sgs:
                sg_mem.extend(dev_index[d] for d in sg.member_device_ids)
                sg_off.append(len(sg_mem))
                sg_cap.append(float(sg.aggregate_capacity))
            sg_off_fg.append(len(sg_off) - 1)
        u32 = lambda x: np.array(x, dtype=np.uint32)
        self.fg_member_offset = u32(fg_off)
        self.fg_members = u32(fg_mem) if fg_mem else np.zeros(1, np.uint32)
        self.fg_capacity = np.array(fg_cap, dtype=np.float64)
        self.fg_min_bw = np.array(fg_bw, dtype=np.float64)
        self.fg_has_min_bw = np.array(fg_has, dtype=np.uint8)
        self.fg_sg_offset = u32(sg_off_fg)
        self.sg_member_offset = u32(sg_off)
        self.sg_members = u32(sg_mem) if sg_mem else np.zeros(1, np.uint32)
        self.sg_capacity = np.array(sg_cap if sg_cap else [0.0], dtype=np.float64)
        self.bottleneck_factor = float(bottleneck_factor)
        self.struct = self._make_struct()

    @property
    def n_fgs(self) -> int:
        return len(self.fg_ids)

    def bm_pairs(self):
        """(b, m) in exhaustive_plan / search_plan loop order."""
        return [(b, m) for b in self.batches for m in self.micros]

    def _make_struct(self) -> abi.GpInstance:
        d, u, i = C.c_double, C.c_uint32, C.c_int64
        s = abi.GpInstance()
        s.n_layers = self.n_layers
        s.fwd_flops = _ptr(self.fwd, d)
        s.bwd_input_flops = _ptr(self.bwd_in, d)
        s.bwd_weight_flops = _ptr(self.bwd_w, d)
        s.activation_out_bytes = _ptr(self.act, d)
        s.param_bytes = _ptr(self.param, d)
        s.n_batch = len(self.batches)
        s.batch = _ptr(self.batch, i)
        s.n_micro = len(self.micros)
        s.micro = _ptr(self.micro, i)
        s.n_devices = self.n_devices
        s.p_c = _ptr(self.p_c, d)
        s.memory_bytes = _ptr(self.memory, d)
        s.id_rank = _ptr(self.id_rank, u)
        s.p_t = _ptr(self.p_t, d)
        s.latency = _ptr(self.lat, d)
        s.bandwidth = _ptr(self.bw, d)
        s.n_fgs = self.n_fgs
        s.fg_member_offset = _ptr(self.fg_member_offset, u)
        s.fg_members = _ptr(self.fg_members, u)
        s.fg_capacity = _ptr(self.fg_capacity, d)
        s.fg_min_bw = _ptr(self.fg_min_bw, d)
        s.fg_has_min_bw = _ptr(self.fg_has_min_bw, C.c_uint8)
        s.fg_sg_offset = _ptr(self.fg_sg_offset, u)
        s.sg_member_offset = _ptr(self.sg_member_offset, u)
        s.sg_members = _ptr(self.sg_members, u)
        s.sg_capacity = _ptr(self.sg_capacity, d)
        s.bottleneck_factor = self.bottleneck_factor
        return s

    # ---- candidate encoding ----
    def encode_keys(self, keys, bm_index):
        """``(order ids, counts)`` tuples -> (order u8[n,k], counts u8[n,k], bm u8[n])."""
        n = len(keys)
        k = len(keys[0][0]) if n else self.n_fgs
        pos = self.fg_pos
        order = np.array([[pos[f] for f in o] for o, _ in keys], dtype=np.uint8).reshape(n, k)
        counts = np.array([c for _, c in keys], dtype=np.uint8).reshape(n, k)
        if np.isscalar(bm_index):
            bm = np.full(n, bm_index, dtype=np.uint8)
        else:
            bm = np.asarray(bm_index, dtype=np.uint8)
        return order, counts, bm

    def encode(self, cands, bm_index):
        """Candidates -> (order u8[n,k], counts u8[n,k], bm u8[n])."""
        n = len(cands)
        k = len(cands[0].order) if n else self.n_fgs
        order = np.empty((n, k), dtype=np.uint8)
        counts = np.empty((n, k), dtype=np.uint8)
        pos = self.fg_pos
        for i, c in enumerate(cands):
            order[i] = [pos[f] for f in c.order]
            counts[i] = c.counts
        if np.isscalar(bm_index):
            bm = np.full(n, bm_index, dtype=np.uint8)
        else:
            bm = np.asarray(bm_index, dtype=np.uint8)
        return order, counts, bm
