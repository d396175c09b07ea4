"""Pipeline schedules on the GPU: generation (K5 full with op / transfer
records), validation and bubble fractions (K8) - the reference's
``generate_schedule`` / ``SimReport.schedule`` / ``validate_schedule`` /
``bubble_fraction`` (src/schedule.py:77-182, src/engine.py:230-431).

Schedules are returned as the mirror types below, field for field the
reference's ``PipeOp`` / ``TransferRecord`` / ``Schedule``; ``OpKind`` values
are the reference's letters.  Validation messages are formatted here from
the device's violation records with the reference's f-strings.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi
from . import domain as D
from .simulate import SimConfig, pack_timings, pack_traces


class OpKind(enum.Enum):
    FORWARD = "F"
    BACKWARD = "B"
    WEIGHT_UPDATE = "W"
    WEIGHT_SYNC = "S"
    OPTIMIZER_STEP = "O"


_KINDS = (OpKind.FORWARD, OpKind.BACKWARD, OpKind.WEIGHT_UPDATE, OpKind.WEIGHT_SYNC,
          OpKind.OPTIMIZER_STEP)
_KIND_CODE = {k.value: i for i, k in enumerate(_KINDS)}


@dataclass(frozen=True)
class PipeOp:
    kind: OpKind
    stage: int
    start: float
    end: float
    size: int
    iteration: int
    microbatch_id: Optional[int] = None


@dataclass(frozen=True)
class TransferRecord:
    link_id: str
    direction: str
    boundary: int
    start: float
    end: float
    size: int
    iteration: int
    microbatch_id: int


@dataclass(frozen=True)
class AdapterAction:
    t: float
    stage: int
    old_size: int
    new_size: int
    signal: str


@dataclass(frozen=True)
class Schedule:
    ops: Tuple[Tuple[PipeOp, ...], ...]
    makespan: float
    policy: str
    num_stages: int
    micro_count: int

    def stage_ops(self, s: int) -> Tuple[PipeOp, ...]:
        return self.ops[s]


def generate_schedules(timings: Sequence, policy="1f1b", traces: Sequence = (), trace_index=None,
                       adapter_enabled: bool = False, config=None, engine=None,
                       with_actions: bool = False):
    """(Schedule, transfers[, adapter actions]) per timing:
    ``simulate_timing(...).schedule`` / ``.transfers`` / ``.adapter_actions``
    of the reference, computed on the GPU."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    config = config if config is not None else SimConfig()
    pol = getattr(policy, "value", policy)
    code = abi.POLICY_CODE[pol]
    arr = pack_timings(timings)
    tr = pack_traces(traces) if traces else None
    its = int(config.iterations)
    ad = getattr(config, "adapter", None)
    asy = bool(getattr(config, "async_iterations", False))
    deg, rec = getattr(ad, "degrade_factor", 1.2), getattr(ad, "recover_factor", 1.05)
    n = len(timings)
    reps, _, st = eng.simulate_report(arr, n, code, its, tr, len(traces), trace_index,
                                      adapter=adapter_enabled, async_iterations=asy,
                                      degrade=deg, recover=rec)
    _raise(st)
    ooff = np.zeros(n + 1, np.uint64)
    ooff[1:] = np.cumsum([reps[i].n_ops for i in range(n)])
    xoff = np.zeros(n + 1, np.uint64)
    xoff[1:] = np.cumsum([reps[i].n_transfers for i in range(n)])
    aoff = np.zeros(n + 1, np.uint64)
    aoff[1:] = np.cumsum([reps[i].adapter_actions for i in range(n)])
    opts = abi.GpSimOptions(int(bool(adapter_enabled)), int(asy), float(deg), float(rec))
    ops, xfs, acts, st = eng.simulate_schedule(arr, n, code, its, tr, len(traces), trace_index,
                                               opts, ooff, xoff, aoff)
    _raise(st)
    out = []
    for i, t in enumerate(timings):
        sched, xf = records_to_schedule(t, ops, int(ooff[i]), int(ooff[i + 1]), xfs, int(xoff[i]),
                                        int(xoff[i + 1]), float(reps[i].makespan), pol)
        actions = tuple(AdapterAction(a.t, a.stage, a.old_size, a.new_size,
                                      abi.ACTION_SIGNALS[a.signal])
                        for a in (acts[j] for j in range(int(aoff[i]), int(aoff[i + 1]))))
        out.append((sched, xf) if not with_actions else (sched, xf, actions))
    return out


def records_to_schedule(timing, ops, o0, o1, xfs, x0, x1, makespan, policy):
    """(Schedule, transfers) mirrors from gp_op / gp_transfer records."""
    S = len(timing.stages)
    per = [[] for _ in range(S)]
    for j in range(o0, o1):
        o = ops[j]
        per[o.stage].append(PipeOp(_KINDS[o.kind], o.stage, o.start, o.end, o.size, o.iteration,
                                   None if o.microbatch_id < 0 else o.microbatch_id))
    links = [b.link_id for b in timing.boundaries]
    xf = tuple(TransferRecord(links[x.boundary], "fwd" if x.direction == 0 else "bwd",
                              x.boundary, x.start, x.end, x.size, x.iteration, x.microbatch_id)
               for x in (xfs[j] for j in range(x0, x1)))
    sched = Schedule(ops=tuple(tuple(p) for p in per), makespan=makespan, policy=policy,
                     num_stages=S, micro_count=int(timing.batch) // int(timing.microbatch))
    return sched, xf


def _raise(st):
    bad = np.nonzero(st)[0]
    if bad.size:
        i = int(bad[0])
        if int(st[i]) == abi.GP_ERR_CUDA:
            raise D.DeviceError(f"timing {i}: simulator queue capacity exceeded")
        abi.raise_for(int(st[i]), f"timing {i}: event loop stalled with work remaining"
                      if int(st[i]) == abi.GP_ERR_SCHEDULING else f"timing {i} failed")


def pack_schedules(schedules: Sequence):
    """Schedules (reference or mirror objects) -> (op offsets, gp_op array,
    iterations bound)."""
    n_ops = [sum(len(x) for x in sc.ops) for sc in schedules]
    off = np.zeros(len(schedules) + 1, np.uint64)
    off[1:] = np.cumsum(n_ops)
    arr = (abi.GpOp * max(1, int(off[-1])))()
    j = 0
    its = 0
    for sc in schedules:
        for s, stage_ops in enumerate(sc.ops):
            for o in stage_ops:
                r = arr[j]
                r.start, r.end, r.size = o.start, o.end, int(o.size)
                r.microbatch_id = -1 if o.microbatch_id is None else int(o.microbatch_id)
                r.iteration = int(o.iteration)
                r.kind = _KIND_CODE[getattr(o.kind, "value", o.kind)]
                r.stage = s
                its = max(its, int(o.iteration) + 1)
                j += 1
    return off, arr, max(its, 1)


def format_violation(v) -> str:
    """The reference's message for one device violation record."""
    s, it, k = v.stage, v.iteration, v.microbatch_id
    return [
        lambda: f"stage {s}: op {_KINDS[v.kind].value} ends before it starts",
        lambda: f"stage {s}: ops overlap at t={v.t:.6g}",
        lambda: f"F(stage {s}, mb {k}, iter {it}) starts before its activation arrives",
        lambda: f"B(stage {s}, mb {k}, iter {it}) starts before F ends",
        lambda: f"B(stage {s}, mb {k}, iter {it}) starts before its gradient arrives",
        lambda: f"W(stage {s}, mb {k}, iter {it}) starts before B ends",
        lambda: f"stage {s} iter {it}: expected one sync and one optimizer",
        lambda: f"stage {s} iter {it}: sync starts before last weight update",
        lambda: f"stage {s} iter {it}: optimizer starts before sync ends",
    ][v.code]()


def validate_schedules(schedules: Sequence, timings: Sequence, tol: float = 1e-9,
                       engine=None, max_violations: int = 64) -> List[List[str]]:
    """``validate_schedule(schedule_i, timing_i, tol)`` for every schedule,
    on the GPU (K8, one thread per schedule)."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    n = len(schedules)
    off, arr, its = pack_schedules(schedules)
    tarr = pack_timings(timings)
    ms = [sc.makespan for sc in schedules]
    viol, nv, _, st = eng.validate_schedules(tarr, n, off, arr, ms, its, tol, max_violations)
    if st.any():
        i = int(np.nonzero(st)[0][0])
        abi.raise_for(int(st[i]), f"schedule {i}: micro-batch ids must be dense per "
                                  f"(stage, iteration, kind)")
    if (nv > max_violations).any():  # rerun with room for every violation
        return validate_schedules(schedules, timings, tol, eng, int(nv.max()))
    return [[format_violation(viol[i * max_violations + q]) for q in range(int(nv[i]))]
            for i in range(n)]


def bubble_fractions(schedules: Sequence, timings: Sequence, engine=None) -> List[List[float]]:
    """``bubble_fraction(schedule)`` per schedule (src/schedule.py:174-182),
    busy sums on the GPU."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    for sc in schedules:
        if sc.makespan <= 0:
            raise ValueError("makespan must be positive")
    n = len(schedules)
    off, arr, its = pack_schedules(schedules)
    _, _, busy, st = eng.validate_schedules(pack_timings(timings), n, off, arr,
                                            [sc.makespan for sc in schedules], its, 1e-9, 0)
    if st.any():
        i = int(np.nonzero(st)[0][0])
        abi.raise_for(int(st[i]), f"schedule {i}: unsupported op structure")
    return [[(sc.makespan - float(busy[i, s])) / sc.makespan for s in range(sc.num_stages)]
            for i, sc in enumerate(schedules)]
