"""ctypes binding of ``oracle/liboracle.so`` - TEST INFRASTRUCTURE ONLY.

The oracle is the CPU restatement of the reference planner path (see
``oracle/oracle.c``).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
CPU-baseline legs of ``bench.py`` may import this module: it is the checker
and the timed CPU baseline, never part of the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2505_15536_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P = C.POINTER
        L.or_psum.restype = C.c_double
        L.or_psum.argtypes = [P(C.c_double), C.c_size_t]
        L.or_proportional_split.argtypes = [C.c_int64, P(C.c_double), C.c_int, C.c_int,
                                            P(C.c_int64)]
        L.or_tp_grid.argtypes = [P(C.c_double), C.c_int, P(C.c_double), P(C.c_double)]
        L.or_dp_fractions.argtypes = [P(C.c_double), C.c_int, P(C.c_double)]
        L.or_evaluate.argtypes = [P(abi.GpInstance), C.c_uint32, P(C.c_uint8),
                                  P(C.c_uint8), C.c_uint32, P(C.c_double),
                                  P(abi.GpPlanInfo)]
        L.or_space_size.restype = C.c_uint64
        L.or_space_size.argtypes = [P(abi.GpInstance)]
        L.or_decode.argtypes = [P(abi.GpInstance), C.c_uint64, P(C.c_uint8),
                                P(C.c_uint8), P(C.c_uint32)]
        L.or_argmin_range.argtypes = [P(abi.GpInstance), C.c_uint64, C.c_uint64,
                                      C.c_int, P(abi.GpBest)]
        L.or_eval_batch.argtypes = [P(abi.GpInstance), C.c_uint32, C.c_uint64,
                                    P(C.c_uint8), P(C.c_uint8), P(C.c_uint8),
                                    P(C.c_double), P(C.c_uint8), C.c_int]
        L.or_eval_range.argtypes = [P(abi.GpInstance), C.c_uint64, C.c_uint64, P(C.c_double),
                                    P(C.c_uint8), C.c_int]
        L.or_group_detail.argtypes = [P(abi.GpInstance), C.c_uint32, P(abi.GpGroupInfo)]
        L.or_sim_1f1b.argtypes = [P(abi.GpTiming), C.c_int, P(C.c_double)]
        L.or_sim_batch.argtypes = [P(abi.GpTiming), C.c_uint64, C.c_int, P(C.c_double),
                                   P(C.c_uint8)]
        L.or_sim_policy_batch.argtypes = [P(abi.GpTiming), C.c_uint64, C.c_int, C.c_int,
                                          P(abi.GpTrace), P(C.c_uint32), P(C.c_double),
                                          P(C.c_uint8)]
        L.or_sim_report_batch.argtypes = [P(abi.GpTiming), C.c_uint64, C.c_int, C.c_int,
                                          P(abi.GpTrace), P(C.c_uint32), P(abi.GpSimOptions),
                                          P(abi.GpSimReport), P(C.c_double), P(C.c_uint8)]
        L.or_sim_schedule_batch.argtypes = [P(abi.GpTiming), C.c_uint64, C.c_int, C.c_int,
                                            P(abi.GpTrace), P(C.c_uint32), P(abi.GpSimOptions),
                                            P(C.c_uint64), P(abi.GpOp), P(C.c_uint64),
                                            P(abi.GpTransfer), P(C.c_uint64), P(abi.GpAction),
                                            P(C.c_uint8)]
        L.or_validate_schedule.argtypes = [P(abi.GpTiming), P(abi.GpOp), C.c_uint64, C.c_double,
                                           C.c_double, C.c_uint32, P(abi.GpViolation),
                                           P(C.c_uint32), P(C.c_double)]
        L.or_group_hierarchy.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                                         C.c_double, C.c_double, P(C.c_uint16), P(C.c_uint16),
                                         P(C.c_uint32), P(C.c_uint32), P(C.c_double),
                                         P(C.c_double), P(C.c_double), P(C.c_double)]
        L.or_group_fixed.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(C.c_double),
                                     P(C.c_uint16), C.c_int, C.c_double, P(C.c_uint16),
                                     P(C.c_uint32), P(C.c_double), P(C.c_double), P(C.c_double),
                                     P(C.c_double)]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def psum(xs) -> float:
    a = np.ascontiguousarray(xs, dtype=np.float64)
    return lib().or_psum(_dp(a), a.size)


def proportional_split(total, weights, minimum=0):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(len(w), dtype=np.int64)
    st = lib().or_proportional_split(int(total), _dp(w), len(w), int(minimum),
                                     out.ctypes.data_as(C.POINTER(C.c_int64)))
    abi.raise_for(st, "cannot honor the minimum share")
    return [int(x) for x in out]


def tp_grid(caps):
    c = np.ascontiguousarray(caps, dtype=np.float64)
    rf = np.zeros(len(c)); cf = np.zeros(len(c))
    ok = lib().or_tp_grid(_dp(c), len(c), _dp(rf), _dp(cf))
    return [(float(a), float(b)) for a, b in zip(rf, cf)] if ok else None


def dp_fractions(caps):
    c = np.ascontiguousarray(caps, dtype=np.float64)
    fr = np.zeros(len(c))
    lib().or_dp_fractions(_dp(c), len(c), _dp(fr))
    return [float(x) for x in fr]


def evaluate(packed, order, counts, bm, detail=False):
    """(status, cost[, GpPlanInfo]) for one encoded candidate."""
    o = np.ascontiguousarray(order, dtype=np.uint8)
    n = np.ascontiguousarray(counts, dtype=np.uint8)
    cost = C.c_double(0.0)
    info = abi.GpPlanInfo() if detail else None
    st = lib().or_evaluate(C.byref(packed.struct), len(o), _u8(o), _u8(n), int(bm),
                           C.byref(cost), C.byref(info) if detail else None)
    return (st, cost.value, info) if detail else (st, cost.value)


def eval_batch(packed, order, counts, bm, threads=1):
    order = np.ascontiguousarray(order, dtype=np.uint8)
    counts = np.ascontiguousarray(counts, dtype=np.uint8)
    bm = np.ascontiguousarray(bm, dtype=np.uint8)
    n, k = order.shape
    cost = np.empty(n, dtype=np.float64)
    status = np.empty(n, dtype=np.uint8)
    lib().or_eval_batch(C.byref(packed.struct), k, n, _u8(order), _u8(counts),
                        _u8(bm), _dp(cost), _u8(status), int(threads))
    return cost, status


def eval_range(packed, lo, hi, threads=1):
    """(cost, status) of every candidate with enumeration index in [lo, hi)."""
    n = max(0, int(hi) - int(lo))
    cost = np.empty(n, dtype=np.float64)
    status = np.empty(n, dtype=np.uint8)
    if n:
        st = lib().or_eval_range(C.byref(packed.struct), int(lo), int(hi), _dp(cost), _u8(status),
                                 int(threads))
        abi.raise_for(st, "bad instance")
    return cost, status


def space_size(packed) -> int:
    return int(lib().or_space_size(C.byref(packed.struct)))


def decode(packed, idx):
    k = packed.n_fgs
    o = np.zeros(k, dtype=np.uint8); c = np.zeros(k, dtype=np.uint8)
    bm = C.c_uint32(0)
    lib().or_decode(C.byref(packed.struct), int(idx), _u8(o), _u8(c), C.byref(bm))
    return o, c, bm.value


def argmin_range(packed, lo, hi, threads=1):
    best = abi.GpBest()
    st = lib().or_argmin_range(C.byref(packed.struct), int(lo), int(hi),
                               int(threads), C.byref(best))
    return st, best


def group_detail(packed, f):
    g = abi.GpGroupInfo()
    lib().or_group_detail(C.byref(packed.struct), int(f), C.byref(g))
    return g


def sim_batch(packed_timings, n, iterations=1):
    """(makespans, status) of gp_timing records (simulate.pack_timings)."""
    ms = np.empty(n, dtype=np.float64)
    st = np.empty(n, dtype=np.uint8)
    lib().or_sim_batch(packed_timings, n, int(iterations), _dp(ms), _u8(st))
    return ms, st


def sim_policy_batch(packed_timings, n, policy, iterations=1, traces=None, trace_index=None):
    """(makespans, status) under ``policy`` (abi.POLICY_CODE) and traces."""
    ms = np.empty(n, dtype=np.float64)
    st = np.empty(n, dtype=np.uint8)
    ti = None
    if trace_index is not None:
        ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
    lib().or_sim_policy_batch(packed_timings, n, int(policy), int(iterations), traces,
                              ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                              _dp(ms), _u8(st))
    return ms, st


def sim_reports(packed_timings, n, policy, iterations=1, traces=None, trace_index=None,
                adapter=False, async_iterations=False, degrade=1.2, recover=1.05):
    """(GpSimReport array, iteration_ends[n, iterations], status) of
    simulate_timing with every SimConfig option."""
    opts = abi.GpSimOptions(int(bool(adapter)), int(bool(async_iterations)),
                            float(degrade), float(recover))
    reps = (abi.GpSimReport * max(1, n))()
    ends = np.zeros((n, iterations), dtype=np.float64)
    st = np.empty(n, dtype=np.uint8)
    ti = None
    if trace_index is not None:
        ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
    lib().or_sim_report_batch(packed_timings, n, int(policy), int(iterations), traces,
                              ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                              C.byref(opts), reps, _dp(ends), _u8(st))
    return reps, ends, st


def group_hierarchy(pt, bw, pc, thr_net=0.3, thr_comp=0.3):
    """(status, grouping.Hierarchy) of group_first_level + group_second_level
    for one topology in rank order (grouping.topology_arrays)."""
    from paper_2505_15536_b200.grouping import Hierarchy
    pt = np.ascontiguousarray(pt, dtype=np.float64)
    bw = np.ascontiguousarray(bw, dtype=np.float64)
    pc = np.ascontiguousarray(pc, dtype=np.float64)
    n = len(pc)
    fg_of = np.zeros(n, np.uint16); sg_of = np.zeros(n, np.uint16)
    nf = C.c_uint32(0); ns = C.c_uint32(0)
    fi = np.zeros(max(n, 1)); fc = np.zeros(max(n, 1)); fb = np.zeros(max(n, 1))
    sc = np.zeros(max(n, 1))
    u16 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint16))
    st = lib().or_group_hierarchy(n, _dp(pt), _dp(bw), _dp(pc), float(thr_net), float(thr_comp),
                                  u16(fg_of), u16(sg_of), C.byref(nf), C.byref(ns), _dp(fi),
                                  _dp(fc), _dp(fb), _dp(sc))
    if st:
        return st, None
    return st, Hierarchy(fg_of, sg_of, fi[:nf.value].copy(), fc[:nf.value].copy(),
                         fb[:nf.value].copy(), sc[:ns.value].copy())


def sim_schedules(packed_timings, n, policy, iterations=1, traces=None, trace_index=None,
                  adapter=False, async_iterations=False, degrade=1.2, recover=1.05):
    """(reports, op_offset, ops, xfer_offset, transfers, status, action_offset,
    actions): the full schedules (PipeOp / TransferRecord / AdapterAction
    records) of a batch of timings."""
    reps, _, st = sim_reports(packed_timings, n, policy, iterations, traces, trace_index,
                              adapter, async_iterations, degrade, recover)
    nops = np.array([reps[i].n_ops for i in range(n)], dtype=np.uint64)
    nxf = np.array([reps[i].n_transfers for i in range(n)], dtype=np.uint64)
    ooff = np.zeros(n + 1, np.uint64); ooff[1:] = np.cumsum(nops)
    xoff = np.zeros(n + 1, np.uint64); xoff[1:] = np.cumsum(nxf)
    ops = (abi.GpOp * max(1, int(ooff[-1])))()
    xfs = (abi.GpTransfer * max(1, int(xoff[-1])))()
    aoff = np.zeros(n + 1, np.uint64)
    aoff[1:] = np.cumsum([reps[i].adapter_actions for i in range(n)])
    acts = (abi.GpAction * max(1, int(aoff[-1])))()
    opts = abi.GpSimOptions(int(bool(adapter)), int(bool(async_iterations)),
                            float(degrade), float(recover))
    ti = None
    if trace_index is not None:
        ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
    st2 = np.empty(n, dtype=np.uint8)
    u64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
    lib().or_sim_schedule_batch(packed_timings, n, int(policy), int(iterations), traces,
                                ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                                C.byref(opts), u64(ooff), ops, u64(xoff), xfs, u64(aoff), acts,
                                _u8(st2))
    return reps, ooff, ops, xoff, xfs, st2, aoff, acts


def validate_schedule(timing_struct, ops, n, makespan, tol=1e-9, max_violations=4096, first=0):
    """(violation records, count, busy[16]) of one schedule: gp_op records
    ops[first : first + n]."""
    ops = C.cast(C.addressof(ops) + int(first) * C.sizeof(abi.GpOp), C.POINTER(abi.GpOp))
    out = (abi.GpViolation * max_violations)()
    nv = C.c_uint32(0)
    busy = np.zeros(abi.GP_MAX_STAGES)
    lib().or_validate_schedule(C.byref(timing_struct), ops, int(n), float(makespan), float(tol),
                               max_violations, out, C.byref(nv), _dp(busy))
    return [out[i] for i in range(min(nv.value, max_violations))], nv.value, busy


def group_fixed(pt, bw, pc, fg_of, n_fg, thr_comp=0.3):
    """(status, grouping.Hierarchy) for a given first-level partition
    (fg_of in sorted-member-tuple order): group statistics + second level."""
    from paper_2505_15536_b200.grouping import Hierarchy
    pt = np.ascontiguousarray(pt, dtype=np.float64)
    bw = np.ascontiguousarray(bw, dtype=np.float64)
    pc = np.ascontiguousarray(pc, dtype=np.float64)
    fg = np.ascontiguousarray(fg_of, dtype=np.uint16)
    n = len(pc)
    sg_of = np.zeros(n, np.uint16)
    ns = C.c_uint32(0)
    fi = np.zeros(max(n, 1)); fc = np.zeros(max(n, 1)); fb = np.zeros(max(n, 1))
    sc = np.zeros(max(n, 1))
    u16 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint16))
    st = lib().or_group_fixed(n, _dp(pt), _dp(bw), _dp(pc), u16(fg), int(n_fg), float(thr_comp),
                              u16(sg_of), C.byref(ns), _dp(fi), _dp(fc), _dp(fb), _dp(sc))
    if st:
        return st, None
    return st, Hierarchy(fg.copy(), sg_of, fi[:n_fg].copy(), fc[:n_fg].copy(), fb[:n_fg].copy(),
                         sc[:ns.value].copy())
