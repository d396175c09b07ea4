"""Batched pipeline-time simulation (K5) - the makespan of the reference's
discrete-event engine.

``simulate_makespans(timings, iterations)`` returns, for every timing,
``simulate_timing(timing, Policy.ONE_F_ONE_B, CONSTANT_TRACE,
adapter_enabled=False, config=SimConfig(iterations=...)).makespan``
(src/simulator.py:71-113 -> PipelineEngine.run, src/engine.py:230-431), bit
for bit, computed by one GPU thread per timing;
``simulate_makespans_policy`` does the same for GPIPE / 1F1B / ZB_ORIGINAL /
ZB_COMPACT under per-timing NetworkTrace breakpoints (src/nettrace.py:12-76),
e.g. to rank candidate plans by simulated makespan under bandwidth drops.  Timings are the reference's
``PlanTiming`` objects (or the mirrors below); ``make_timing`` mirrors the
reference fixture builder (src/schedule.py:27-74).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence, Tuple

import numpy as np

from . import abi
from . import domain as D


@dataclass(frozen=True)
class StageTiming:
    fwd_per_sample: float
    bwd_per_sample: float
    wgt_per_sample: float
    al_seconds: float
    sync_seconds: float
    opt_seconds: float
    effective_capacity: float


@dataclass(frozen=True)
class BoundaryTiming:
    link_id: str
    latency_seconds: float
    bandwidth_bytes_per_s: float
    act_bytes_per_sample: float
    grad_bytes_per_sample: float


@dataclass(frozen=True)
class PlanTiming:
    stages: Tuple[StageTiming, ...]
    boundaries: Tuple[BoundaryTiming, ...]
    batch: int
    microbatch: int

    @property
    def num_stages(self) -> int:
        return len(self.stages)


def make_timing(fwd, bwd, wgt, transfer, microbatch=1, micro_count=1, sync=None, opt=None,
                latency=0.0) -> PlanTiming:
    """Mirror of the reference fixture builder (src/schedule.py:27-74)."""
    S = len(fwd)
    if not (len(bwd) == len(wgt) == S) or len(transfer) != S - 1:
        raise D.InvalidTimingError("timing vectors have inconsistent lengths")
    sync = sync or [0.0] * S
    opt = opt or [0.0] * S
    stages = tuple(StageTiming(fwd[s] / microbatch, bwd[s] / microbatch, wgt[s] / microbatch,
                               sync[s], sync[s], opt[s], 1.0) for s in range(S))
    bounds = tuple(BoundaryTiming(f"{i}-{i + 1}", latency, 1.0,
                                  max(transfer[i] - latency, 0.0) / microbatch,
                                  max(transfer[i] - latency, 0.0) / microbatch)
                   for i in range(S - 1))
    return PlanTiming(stages, bounds, microbatch * micro_count, microbatch)


def pack_timings(timings: Sequence) -> "C.Array":
    """PlanTiming objects -> contiguous gp_timing records (include/geopipe_b200.h)."""
    arr = (abi.GpTiming * max(1, len(timings)))()
    for i, t in enumerate(timings):
        S = len(t.stages)
        if S < 1 or S > abi.GP_MAX_STAGES:
            raise D.InvalidTimingError(f"{S} stages outside [1, {abi.GP_MAX_STAGES}]")
        if len(t.boundaries) != S - 1:
            raise D.InvalidTimingError(f"expected {S - 1} boundaries, got {len(t.boundaries)}")
        r = arr[i]
        r.n_stages = S
        r.batch = int(t.batch)
        r.microbatch = int(t.microbatch)
        for s, st in enumerate(t.stages):
            r.fwd[s] = st.fwd_per_sample
            r.bwd[s] = st.bwd_per_sample
            r.wgt[s] = st.wgt_per_sample
            r.sync[s] = st.sync_seconds
            r.opt[s] = st.opt_seconds
        for b, bt in enumerate(t.boundaries):
            r.lat[b] = bt.latency_seconds
            r.bw[b] = bt.bandwidth_bytes_per_s
            r.act[b] = bt.act_bytes_per_sample
            r.grad[b] = bt.grad_bytes_per_sample
    return arr


def pack_traces(traces: Sequence, n_boundaries: int = abi.GP_MAX_STAGES) -> "C.Array":
    """NetworkTrace objects (``breakpoints: {link_id: ((t, mult), ...)}``) ->
    gp_trace records; link "b-(b+1)" of boundary b (src/timing.py:219)."""
    arr = (abi.GpTrace * max(1, len(traces)))()
    for i, tr in enumerate(traces):
        bps = getattr(tr, "breakpoints", tr) or {}
        for link, points in bps.items():
            try:
                a, b = (int(x) for x in str(link).split("-"))
            except ValueError:
                continue  # links that are not stage boundaries never apply
            if b != a + 1 or not 0 <= a < abi.GP_MAX_STAGES:
                continue
            if len(points) > abi.GP_MAX_BREAKPOINTS:
                raise D.InputFileError(f"trace link {link}: more than "
                                       f"{abi.GP_MAX_BREAKPOINTS} breakpoints")
            arr[i].n_points[a] = len(points)
            for j, (t, mult) in enumerate(points):
                arr[i].t[a][j] = float(t)
                arr[i].mult[a][j] = float(mult)
    return arr


def simulate_makespans_policy(timings: Sequence, policy: str = "1f1b", iterations: int = 1,
                              traces: Sequence = (), trace_index=None, engine=None) -> np.ndarray:
    """Makespans of ``simulate_timing(t, policy, trace, adapter_enabled=False,
    SimConfig(iterations))`` for every timing (traces[trace_index[i]], or the
    constant trace when ``traces`` is empty)."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    code = abi.POLICY_CODE[getattr(policy, "value", policy)]
    arr = pack_timings(timings)
    tr = pack_traces(traces) if traces else None
    ms, st = eng.simulate(arr, len(timings), code, iterations, tr, len(traces), trace_index)
    bad = np.nonzero(st)[0]
    if bad.size:
        abi.raise_for(int(st[bad[0]]), f"timing {int(bad[0])} failed to simulate")
    return ms


def simulate_makespans(timings: Sequence, iterations: int = 1, engine=None) -> np.ndarray:
    """1F1B makespans of ``timings`` on the GPU (raises like the reference)."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    arr = pack_timings(timings)
    ms, st = eng.sim_1f1b(arr, len(timings), iterations)
    bad = np.nonzero(st)[0]
    if bad.size:
        abi.raise_for(int(st[bad[0]]), f"timing {int(bad[0])} failed to simulate")
    return ms


def simulate_timing_makespan(timing, iterations: int = 1, engine=None) -> float:
    return float(simulate_makespans([timing], iterations, engine)[0])
