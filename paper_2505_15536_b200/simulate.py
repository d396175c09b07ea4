"""Batched 1F1B pipeline-time simulation (K5) - the makespan of the reference's
discrete-event engine.

``simulate_makespans(timings, iterations)`` returns, for every timing,
``simulate_timing(timing, Policy.ONE_F_ONE_B, CONSTANT_TRACE,
adapter_enabled=False, config=SimConfig(iterations=...)).makespan``
(src/simulator.py:71-113 -> PipelineEngine.run, src/engine.py:230-431), bit
for bit, computed by one GPU thread per timing.  Timings are the reference's
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
