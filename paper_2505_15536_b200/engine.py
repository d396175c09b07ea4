"""ctypes binding of the CUDA engine ``libgeopipe_b200.so`` (include/geopipe_b200.h).

This is the only way the package computes plan costs.  There is no CPU
fallback: if the shared library is missing, or no sm_100 device is visible,
every call raises :class:`~.domain.DeviceError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import abi
from . import domain as D

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GP_ENGINE_LIB") or os.path.join(HERE, "libgeopipe_b200.so")

_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load the engine library (raises DeviceError when it is not built)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise D.DeviceError(
                f"CUDA engine not built: {LIB_PATH} is missing "
                "(run __graft_entry__.build() or make -C paper_2505_15536_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
        L.gp_version.restype = C.c_char_p
        L.gp_last_error.restype = C.c_char_p
        L.gp_ctx_create.argtypes = [C.c_int, P(vp)]
        L.gp_ctx_load.argtypes = [vp, P(abi.GpInstance)]
        L.gp_ctx_destroy.argtypes = [vp]
        L.gp_ctx_destroy.restype = None
        L.gp_ctx_stream.argtypes = [vp]
        L.gp_ctx_stream.restype = vp
        u8p = P(C.c_uint8)
        L.gp_eval_batch.argtypes = [vp, C.c_uint32, C.c_uint64, u8p, u8p, u8p,
                                    P(C.c_double), u8p]
        L.gp_eval_batch_device.argtypes = [vp, C.c_uint32, C.c_uint64, vp, vp, vp, vp, vp]
        L.gp_argmin_batch_device.argtypes = [vp, C.c_uint64, vp, vp, vp, vp]
        L.gp_space_size.argtypes = [vp, P(C.c_uint64)]
        L.gp_argmin_range.argtypes = [vp, C.c_uint64, C.c_uint64, P(abi.GpBest)]
        L.gp_argmin_range_async.argtypes = [vp, C.c_uint64, C.c_uint64]
        L.gp_argmin_fetch.argtypes = [vp, P(abi.GpBest)]
        L.gp_argmin_items_async.argtypes = [vp, C.c_uint64, C.c_uint64]
        L.gp_argmin_bnb_async.argtypes = [vp]
        L.gp_plan_detail.argtypes = [vp, C.c_uint32, u8p, u8p, C.c_uint32,
                                     P(abi.GpPlanInfo)]
        L.gp_solve.argtypes = [vp, C.c_uint64, C.c_uint64, P(abi.GpBest), P(abi.GpPlanInfo)]
        L.gp_replan.argtypes = [vp, P(abi.GpInstance), P(abi.GpBest), P(abi.GpPlanInfo)]
        L.gp_group_splits.argtypes = [vp, C.c_uint32, P(abi.GpGroupInfo)]
        L.gp_set_bandwidth.argtypes = [vp, P(C.c_double)]
        L.gp_reset_bandwidth.argtypes = [vp]
        L.gp_diag_verify_begin.argtypes = [vp, C.c_uint64, C.c_uint64]
        L.gp_diag_verify_end.argtypes = [vp, P(C.c_double)]
        L.gp_diag_fp64_peak.argtypes = [C.c_int, P(C.c_double)]
        L.gp_sim_1f1b.argtypes = [vp, vp, C.c_uint64, C.c_uint32, P(C.c_double), u8p]
        L.gp_sim_1f1b_device.argtypes = [vp, vp, C.c_uint64, C.c_uint32, vp, vp]
        L.gp_simulate.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, vp, C.c_uint32,
                                  P(C.c_uint32), P(C.c_double), u8p]
        L.gp_simulate_report.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, vp,
                                         C.c_uint32, P(C.c_uint32), P(abi.GpSimOptions),
                                         P(abi.GpSimReport), P(C.c_double), u8p]
        u64p = P(C.c_uint64)
        L.gp_simulate_schedule.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, vp,
                                           C.c_uint32, P(C.c_uint32), P(abi.GpSimOptions),
                                           u64p, P(abi.GpOp), u64p, P(abi.GpTransfer), u64p,
                                           P(abi.GpAction), u8p]
        L.gp_validate_schedules.argtypes = [vp, vp, C.c_uint64, u64p, P(abi.GpOp),
                                            P(C.c_double), C.c_uint32, C.c_double, C.c_uint32,
                                            P(abi.GpViolation), P(C.c_uint32), P(C.c_double), u8p]
        u16p = P(C.c_uint16)
        L.gp_group_snapshots.argtypes = [vp, C.c_uint32, C.c_uint32, P(C.c_double),
                                         P(C.c_double), P(C.c_double), C.c_double, C.c_double,
                                         u16p, u16p, P(C.c_uint32), P(C.c_uint32), P(C.c_double),
                                         P(C.c_double), P(C.c_double), P(C.c_double)]
        L.gp_group_fixed.argtypes = [vp, C.c_uint32, P(C.c_double), P(C.c_double), P(C.c_double),
                                     u16p, C.c_uint32, C.c_double, u16p, P(C.c_uint32),
                                     P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double)]
        L.gp_replan_snapshots.argtypes = [vp, P(C.c_double), C.c_uint32, P(abi.GpBest),
                                          P(C.c_int32)]
        L.gp_replan_snapshots_async.argtypes = [vp, vp, C.c_uint32, vp, vp]
        L.gp_peer_alloc.argtypes = [vp, C.c_uint64, P(vp), vp]
        L.gp_peer_open.argtypes = [vp, vp, P(vp)]
        L.gp_peer_close.argtypes = [vp, vp, C.c_int]
        L.gp_peer_read.argtypes = [vp, vp, vp, C.c_uint64]
        L.gp_peer_allgather.argtypes = [vp, vp, C.c_uint64, C.c_uint32, C.c_uint32, P(vp), C.c_uint64]
        L.gp_sim_candidates.argtypes = [vp, C.c_uint32, C.c_uint64, u8p, u8p, u8p, C.c_uint32,
                                        C.c_double, P(C.c_double), u8p]
        L.gp_ctx_set_k3_mode.argtypes = [vp, C.c_int]
        L.gp_diag_checks.argtypes = [vp, P(C.c_uint32)]
        L.gp_diag_kernel_timing.argtypes = [vp, C.c_int, P(C.c_double), P(C.c_uint64)]
        L.gp_diag_replan_timing.argtypes = [vp, C.c_int, P(C.c_double)]
        L.gp_diag_replan_host.argtypes = [vp, P(C.c_double)]
        L.gp_plan_cost.argtypes = [vp, C.c_uint32, P(abi.GpPlanStage), C.c_int64, C.c_int64,
                                   C.c_double, P(abi.GpPlanInfo), P(abi.GpTiming)]
        L.gp_plan_timing.argtypes = [vp, C.c_uint32, C.c_uint64, u8p, u8p, u8p, C.c_double,
                                     P(abi.GpTiming), u8p]
        _lib = L
        return L


def _check(status: int) -> None:
    if status != abi.GP_OK:
        msg = lib().gp_last_error().decode(errors="replace")
        abi.raise_for(status, msg)


def _u8(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


class Engine:
    """One engine context on one CUDA device (one stream)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.gp_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device
        self.packed = None
        # the instance whose tables the context holds unmodified (None after a
        # bandwidth snapshot or a failed load): load() of it again is a no-op
        self._clean = None

    def close(self):
        if self._h:
            lib().gp_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib().gp_ctx_stream(self._h) or 0

    def load(self, packed) -> "Engine":
        """Stage ``packed`` (gp_ctx_load); a no-op when the context already
        holds exactly this instance's tables."""
        if packed is self._clean:
            return self
        self._clean = None
        _check(lib().gp_ctx_load(self._h, C.byref(packed.struct)))
        self.packed = packed
        self._clean = packed
        return self

    def space_size(self) -> int:
        out = C.c_uint64(0)
        _check(lib().gp_space_size(self._h, C.byref(out)))
        return out.value

    def eval_batch(self, order, counts, bm):
        order = np.ascontiguousarray(order, dtype=np.uint8)
        counts = np.ascontiguousarray(counts, dtype=np.uint8)
        bm = np.ascontiguousarray(bm, dtype=np.uint8)
        n, k = order.shape
        cost = np.empty(n, dtype=np.float64)
        status = np.empty(n, dtype=np.uint8)
        if n:
            _check(lib().gp_eval_batch(self._h, k, n, _u8(order), _u8(counts), _u8(bm),
                                       cost.ctypes.data_as(C.POINTER(C.c_double)),
                                       _u8(status)))
        return cost, status

    def eval_batch_device(self, k, n, d_order, d_counts, d_bm, d_cost, d_status):
        """Device-pointer variant (ints), asynchronous on :attr:`stream`."""
        _check(lib().gp_eval_batch_device(self._h, k, n, d_order, d_counts, d_bm,
                                          d_cost, d_status))

    def argmin_batch_device(self, n, d_cost, d_status, d_keys, d_out):
        """Device-pointer arg-min of an evaluated batch (ints; d_keys may be
        0), asynchronous on :attr:`stream`: d_out[0:2] (u64) = (cost bits,
        key) of the least (cost, key) with status 0 (gp_argmin_batch_device)."""
        _check(lib().gp_argmin_batch_device(self._h, int(n), d_cost, d_status, d_keys or None, d_out))

    def argmin_range(self, lo: int, hi: int) -> abi.GpBest:
        best = abi.GpBest()
        _check(lib().gp_argmin_range(self._h, int(lo), int(hi), C.byref(best)))
        return best

    def solve(self, lo: int, hi: int):
        """Arg-min over [lo, hi) plus the winner's plan detail, one sync."""
        best = abi.GpBest()
        info = abi.GpPlanInfo()
        _check(lib().gp_solve(self._h, int(lo), int(hi), C.byref(best), C.byref(info)))
        return best, info

    def replan(self, packed):
        """Load + exhaustive arg-min + winner detail in one call (CUDA graph
        replayed for every instance of the same shape)."""
        best = abi.GpBest()
        info = abi.GpPlanInfo()
        self._clean = None
        st = lib().gp_replan(self._h, C.byref(packed.struct), C.byref(best), C.byref(info))
        self.packed = packed
        if st in (abi.GP_OK, abi.GP_ERR_INFEASIBLE_SPLIT, abi.GP_ERR_NO_FEASIBLE,
                  abi.GP_ERR_DEGENERATE, abi.GP_ERR_TOPOLOGY):
            self._clean = packed  # the tables were built (a candidate raised, or not)
        _check(st)
        return best, info

    def argmin_range_async(self, lo: int, hi: int) -> None:
        _check(lib().gp_argmin_range_async(self._h, int(lo), int(hi)))

    def argmin_items(self, item_lo: int, item_hi: int) -> abi.GpBest:
        """Arg-min over (micro-batch, order) items [item_lo, item_hi)."""
        _check(lib().gp_argmin_items_async(self._h, int(item_lo), int(item_hi)))
        return self.argmin_fetch()

    def argmin_bnb(self) -> abi.GpBest:
        """Exhaustive arg-min by exact branch-and-bound (K4)."""
        _check(lib().gp_argmin_bnb_async(self._h))
        return self.argmin_fetch()

    def argmin_fetch(self) -> abi.GpBest:
        best = abi.GpBest()
        _check(lib().gp_argmin_fetch(self._h, C.byref(best)))
        return best

    def argmin_fetch_status(self):
        """(status, GpBest, message) without raising: on a per-candidate
        error, GpBest.index is the first erroring candidate's index."""
        best = abi.GpBest()
        st = lib().gp_argmin_fetch(self._h, C.byref(best))
        msg = lib().gp_last_error().decode(errors="replace") if st else ""
        return st, best, msg

    def argmin_items_status(self, item_lo: int, item_hi: int):
        """argmin_items without raising (multi-GPU shards): (status, GpBest, message)."""
        _check(lib().gp_argmin_items_async(self._h, int(item_lo), int(item_hi)))
        return self.argmin_fetch_status()

    def plan_detail(self, order, counts, bm: int) -> abi.GpPlanInfo:
        o = np.ascontiguousarray(order, dtype=np.uint8)
        c = np.ascontiguousarray(counts, dtype=np.uint8)
        info = abi.GpPlanInfo()
        _check(lib().gp_plan_detail(self._h, len(o), _u8(o), _u8(c), int(bm),
                                    C.byref(info)))
        return info

    def group_splits(self, f: int) -> abi.GpGroupInfo:
        """TP grid tiles / DP fractions of group f of the loaded instance (a
        function of the instance's capacities and membership only: cached on
        the PackedInstance, which is immutable)."""
        cache = getattr(self.packed, "_group_splits", None) if self.packed is not None else None
        if cache is not None and f in cache:
            return cache[f]
        g = abi.GpGroupInfo()
        _check(lib().gp_group_splits(self._h, int(f), C.byref(g)))
        if self.packed is not None:
            if cache is None:
                try:
                    cache = self.packed._group_splits = {}
                except AttributeError:  # slotted instance: no cache
                    return g
            cache[f] = g
        return g

    def sim_1f1b(self, packed_timings, n: int, iterations: int = 1):
        """(makespans, status) for gp_timing records (simulate.pack_timings)."""
        ms = np.empty(n, dtype=np.float64)
        st = np.empty(n, dtype=np.uint8)
        if n:
            _check(lib().gp_sim_1f1b(self._h, C.cast(packed_timings, C.c_void_p), n,
                                     int(iterations),
                                     ms.ctypes.data_as(C.POINTER(C.c_double)), _u8(st)))
        return ms, st

    def simulate(self, packed_timings, n: int, policy: int, iterations: int = 1,
                 packed_traces=None, n_traces: int = 0, trace_index=None):
        """(makespans, status) under a schedule policy and network traces."""
        ms = np.empty(n, dtype=np.float64)
        st = np.empty(n, dtype=np.uint8)
        ti = None
        if trace_index is not None:
            ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
        if n:
            _check(lib().gp_simulate(
                self._h, C.cast(packed_timings, C.c_void_p), n, int(policy), int(iterations),
                C.cast(packed_traces, C.c_void_p) if packed_traces is not None else None,
                int(n_traces), ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                ms.ctypes.data_as(C.POINTER(C.c_double)), _u8(st)))
        return ms, st

    def simulate_report(self, packed_timings, n: int, policy: int, iterations: int = 1,
                        packed_traces=None, n_traces: int = 0, trace_index=None,
                        adapter: bool = False, async_iterations: bool = False,
                        degrade: float = 1.2, recover: float = 1.05):
        """(GpSimReport array, iteration_ends[n, iterations], status): the
        full simulate_timing event engine with every SimConfig option."""
        opts = abi.GpSimOptions(int(bool(adapter)), int(bool(async_iterations)),
                                float(degrade), float(recover))
        reps = (abi.GpSimReport * max(1, n))()
        ends = np.zeros((n, iterations), dtype=np.float64)
        st = np.empty(n, dtype=np.uint8)
        ti = None
        if trace_index is not None:
            ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
        if n:
            _check(lib().gp_simulate_report(
                self._h, C.cast(packed_timings, C.c_void_p), n, int(policy), int(iterations),
                C.cast(packed_traces, C.c_void_p) if packed_traces is not None else None,
                int(n_traces), ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                C.byref(opts), reps, ends.ctypes.data_as(C.POINTER(C.c_double)), _u8(st)))
        return reps, ends, st

    def simulate_schedule(self, packed_timings, n: int, policy: int, iterations: int,
                          packed_traces, n_traces: int, trace_index, opts, op_offset, xfer_offset,
                          action_offset=None):
        """(ops, transfers, actions, status) for timings whose op / transfer /
        action counts (a previous simulate_report) set the offsets."""
        op_offset = np.ascontiguousarray(op_offset, dtype=np.uint64)
        ops = (abi.GpOp * max(1, int(op_offset[-1])))()
        xfs = None
        if xfer_offset is not None:
            xfer_offset = np.ascontiguousarray(xfer_offset, dtype=np.uint64)
            xfs = (abi.GpTransfer * max(1, int(xfer_offset[-1])))()
        acts = None
        if action_offset is not None:
            action_offset = np.ascontiguousarray(action_offset, dtype=np.uint64)
            acts = (abi.GpAction * max(1, int(action_offset[-1])))()
        st = np.empty(n, dtype=np.uint8)
        ti = None
        if trace_index is not None:
            ti = np.ascontiguousarray(trace_index, dtype=np.uint32)
        u64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
        if n:
            _check(lib().gp_simulate_schedule(
                self._h, C.cast(packed_timings, C.c_void_p), n, int(policy), int(iterations),
                C.cast(packed_traces, C.c_void_p) if packed_traces is not None else None,
                int(n_traces), ti.ctypes.data_as(C.POINTER(C.c_uint32)) if ti is not None else None,
                C.byref(opts), u64(op_offset), ops,
                u64(xfer_offset) if xfs is not None else None, xfs,
                u64(action_offset) if acts is not None else None, acts, _u8(st)))
        return ops, xfs, acts, st

    def validate_schedules(self, packed_timings, n: int, op_offset, ops, makespans,
                           iterations: int, tol: float = 1e-9, max_violations: int = 64):
        """(violations[n, max], counts, busy[n, 16], status) - K8."""
        op_offset = np.ascontiguousarray(op_offset, dtype=np.uint64)
        ms = np.ascontiguousarray(makespans, dtype=np.float64)
        viol = (abi.GpViolation * max(1, n * max_violations))()
        nv = np.zeros(n, np.uint32)
        busy = np.zeros((n, abi.GP_MAX_STAGES))
        st = np.empty(n, dtype=np.uint8)
        if n:
            _check(lib().gp_validate_schedules(
                self._h, C.cast(packed_timings, C.c_void_p), n,
                op_offset.ctypes.data_as(C.POINTER(C.c_uint64)), ops,
                ms.ctypes.data_as(C.POINTER(C.c_double)), int(iterations), float(tol),
                int(max_violations), viol, nv.ctypes.data_as(C.POINTER(C.c_uint32)),
                busy.ctypes.data_as(C.POINTER(C.c_double)), _u8(st)))
        return viol, nv, busy, st

    def group_snapshots(self, p_t, bandwidth, p_c, threshold_net=0.3, threshold_compute=0.3):
        """K7 grouping of ``p_t[n_snap, D, D]`` (rank order); returns the raw
        arrays (fg_of, sg_of, n_fg, n_sg, fg_intra, fg_cap, fg_min_bw, sg_cap)."""
        p_t = np.ascontiguousarray(p_t, dtype=np.float64)
        if p_t.ndim == 2:
            p_t = p_t[None]
        ns, D = p_t.shape[0], p_t.shape[1]
        bw = None
        if bandwidth is not None:
            bw = np.ascontiguousarray(np.broadcast_to(bandwidth, p_t.shape), dtype=np.float64)
        pc = np.ascontiguousarray(p_c, dtype=np.float64)
        fg_of = np.zeros((ns, D), np.uint16); sg_of = np.zeros((ns, D), np.uint16)
        nf = np.zeros(ns, np.uint32); nsg = np.zeros(ns, np.uint32)
        fi, fc, fb, sc = (np.zeros((ns, D)) for _ in range(4))
        P = C.POINTER
        dp = lambda a: a.ctypes.data_as(P(C.c_double))
        u16 = lambda a: a.ctypes.data_as(P(C.c_uint16))
        u32 = lambda a: a.ctypes.data_as(P(C.c_uint32))
        _check(lib().gp_group_snapshots(self._h, D, ns, dp(p_t), dp(bw) if bw is not None else None,
                                        dp(pc), float(threshold_net), float(threshold_compute),
                                        u16(fg_of), u16(sg_of), u32(nf), u32(nsg), dp(fi), dp(fc),
                                        dp(fb), dp(sc)))
        return fg_of, sg_of, nf, nsg, fi, fc, fb, sc

    def plan_cost(self, stages, batch: int, micro: int, opt_seconds: float = 0.0,
                  timing: bool = False):
        """(GpPlanInfo, GpTiming | None) of an explicit plan (gp_plan_stage array)."""
        info = abi.GpPlanInfo()
        tim = abi.GpTiming() if timing else None
        _check(lib().gp_plan_cost(self._h, len(stages), stages, int(batch), int(micro),
                                  float(opt_seconds), C.byref(info),
                                  C.byref(tim) if tim is not None else None))
        return info, tim

    def plan_timing(self, order, counts, bm, opt_seconds: float = 0.0):
        """(gp_timing array, status) of explicit candidates of the loaded instance."""
        order = np.ascontiguousarray(order, dtype=np.uint8)
        counts = np.ascontiguousarray(counts, dtype=np.uint8)
        bm = np.ascontiguousarray(bm, dtype=np.uint8)
        n, k = order.shape
        out = (abi.GpTiming * max(1, n))()
        st = np.empty(n, dtype=np.uint8)
        if n:
            _check(lib().gp_plan_timing(self._h, k, n, _u8(order), _u8(counts), _u8(bm),
                                        float(opt_seconds), out, _u8(st)))
        return out, st

    def group_fixed(self, p_t, bandwidth, p_c, fg_of, n_fg: int, threshold_compute=0.3):
        """Statistics + second level of a given first-level partition (rank order)."""
        p_t = np.ascontiguousarray(p_t, dtype=np.float64)
        D = p_t.shape[0]
        bw = np.ascontiguousarray(bandwidth, dtype=np.float64) if bandwidth is not None else None
        pc = np.ascontiguousarray(p_c, dtype=np.float64)
        fg = np.ascontiguousarray(fg_of, dtype=np.uint16)
        sg_of = np.zeros(D, np.uint16)
        ns = C.c_uint32(0)
        fi, fc, fb, sc = (np.zeros(D) for _ in range(4))
        P = C.POINTER
        dp = lambda a: a.ctypes.data_as(P(C.c_double))
        u16 = lambda a: a.ctypes.data_as(P(C.c_uint16))
        _check(lib().gp_group_fixed(self._h, D, dp(p_t), dp(bw) if bw is not None else None, dp(pc),
                                    u16(fg), int(n_fg), float(threshold_compute), u16(sg_of),
                                    C.byref(ns), dp(fi), dp(fc), dp(fb), dp(sc)))
        return sg_of, ns.value, fi[:n_fg], fc[:n_fg], fb[:n_fg], sc[:ns.value]

    def sim_candidates(self, order, counts, bm, iterations: int = 1, opt_seconds: float = 0.0):
        """1F1B makespans of explicit candidates of the loaded instance."""
        order = np.ascontiguousarray(order, dtype=np.uint8)
        counts = np.ascontiguousarray(counts, dtype=np.uint8)
        bm = np.ascontiguousarray(bm, dtype=np.uint8)
        n, k = order.shape
        ms = np.empty(n, dtype=np.float64)
        st = np.empty(n, dtype=np.uint8)
        if n:
            _check(lib().gp_sim_candidates(self._h, k, n, _u8(order), _u8(counts), _u8(bm),
                                           int(iterations), float(opt_seconds),
                                           ms.ctypes.data_as(C.POINTER(C.c_double)), _u8(st)))
        return ms, st

    def replan_snapshots(self, bandwidths: np.ndarray):
        """Exhaustive arg-min per bandwidth snapshot (bandwidths [S, D, D]).

        Returns (bests, status): a ctypes array of GpBest and int32 codes."""
        bw = np.ascontiguousarray(bandwidths, dtype=np.float64)
        n = bw.shape[0]
        out = (abi.GpBest * max(1, n))()
        st = np.zeros(n, dtype=np.int32)
        if n:
            _check(lib().gp_replan_snapshots(self._h, bw.ctypes.data_as(C.POINTER(C.c_double)), n,
                                             out, st.ctypes.data_as(C.POINTER(C.c_int32))))
        return out, st


    def replan_snapshots_async(self, d_bandwidth: int, n_snap: int, d_keys: int,
                               d_flags: int) -> None:
        """Device pointers (ints), asynchronous on :attr:`stream`: per snapshot
        the arg-min key (cost bits, tie) -> d_keys[2i:2i+2] (int64) and the
        table flags -> d_flags[i] (gp_replan_snapshots_async)."""
        _check(lib().gp_replan_snapshots_async(self._h, d_bandwidth, int(n_snap), d_keys, d_flags))

    def device_checks(self) -> int:
        """Checked builds: first failing device check line since the last
        call (0 none); 0xFFFFFFFF when the checks are compiled out."""
        v = C.c_uint32(0)
        _check(lib().gp_diag_checks(self._h, C.byref(v)))
        return v.value

    def kernel_timing(self, enable: bool):
        """Start (True) / end (False) a window of CUDA-event timing around
        every sweep launch; ending returns (total device ms, launches)."""
        ms, n = C.c_double(0.0), C.c_uint64(0)
        _check(lib().gp_diag_kernel_timing(self._h, int(bool(enable)), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def set_k3_mode(self, mode: int) -> None:
        """Force the exhaustive-kernel variant (-1 auto, 0/1/2, 3 generic)."""
        _check(lib().gp_ctx_set_k3_mode(self._h, int(mode)))

    def replan_timing(self, enable: bool = True) -> float:
        """Turn on/off CUDA-event timing of the gp_replan graph; returns the
        device milliseconds of the last timed graph (-1 before the first)."""
        out = C.c_double(-1.0)
        _check(lib().gp_diag_replan_timing(self._h, int(bool(enable)), C.byref(out)))
        return out.value

    def replan_host_us(self):
        """Host phases of the last timed gp_replan (us): arena fill, graph
        launch call, wait, result decode."""
        out = (C.c_double * 4)()
        _check(lib().gp_diag_replan_host(self._h, out))
        return list(out)

    def set_bandwidth(self, bw: np.ndarray) -> None:
        a = np.ascontiguousarray(bw, dtype=np.float64)
        self._clean = None
        _check(lib().gp_set_bandwidth(self._h, a.ctypes.data_as(C.POINTER(C.c_double))))

    def reset_bandwidth(self) -> None:
        """Back to the loaded instance's bandwidths and min_intra_bandwidth values."""
        _check(lib().gp_reset_bandwidth(self._h))
        self._clean = self.packed

    def verify_begin(self, lo: int, n: int) -> None:
        """Parity tests: record every evaluated candidate's cost at global
        position g - lo (g = snapshot * space_size + index, lo <= g < lo + n)
        until :meth:`verify_end` (gp_diag_verify_begin)."""
        self._verify_n = int(n)
        _check(lib().gp_diag_verify_begin(self._h, int(lo), int(n)))

    def verify_end(self) -> np.ndarray:
        out = np.empty(self._verify_n, dtype=np.float64)
        _check(lib().gp_diag_verify_end(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out


def best_fields(bests, n: int):
    """(cost f64[n], index u64[n]) views of a ctypes GpBest array (no per-item
    Python work)."""
    dt = np.dtype({"names": ["cost", "index"], "formats": ["<f8", "<u8"], "offsets": [0, 8],
                   "itemsize": C.sizeof(abi.GpBest)})
    a = np.frombuffer(bests, dtype=dt, count=n)
    return a["cost"].copy(), a["index"].copy()


def fp64_peak(device: int = 0) -> float:
    """Measured FP64 add issue rate (ops/s) of ``device``."""
    out = C.c_double(0.0)
    _check(lib().gp_diag_fp64_peak(int(device), C.byref(out)))
    return out.value


_tls = threading.local()


def default_engine(device: int = 0) -> Engine:
    """Per-thread engine context (contexts are not shared across threads)."""
    engines = getattr(_tls, "engines", None)
    if engines is None:
        engines = _tls.engines = {}
    eng = engines.get(device)
    if eng is None:
        eng = engines[device] = Engine(device)
    return eng
