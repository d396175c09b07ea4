"""Batched pipeline-time simulation (K5) - the makespan of the reference's
discrete-event engine.

``simulate_makespans(timings, iterations)`` returns, for every timing,
``simulate_timing(timing, Policy.ONE_F_ONE_B, CONSTANT_TRACE,
adapter_enabled=False, config=SimConfig(iterations=...)).makespan``
(src/simulator.py:71-113 -> PipelineEngine.run, src/engine.py:230-431), bit
for bit, computed by one GPU thread per timing;
``simulate_makespans_policy`` does the same for GPIPE / 1F1B / ZB_ORIGINAL /
ZB_COMPACT under per-timing NetworkTrace breakpoints (src/nettrace.py:12-76),
e.g. to rank candidate plans by simulated makespan under bandwidth drops;
``simulate_timings`` / ``simulate_timing`` run the full engine (adapter,
asynchronous iterations) and return the scalar fields of ``SimReport``
(src/simulator.py:31-113).  Timings are the reference's
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


@dataclass(frozen=True)
class AdapterConfig:
    """Mirror of src/adapter.py:127-130."""
    degrade_factor: float = 1.2
    recover_factor: float = 1.05


@dataclass(frozen=True)
class SimConfig:
    """Mirror of src/simulator.py:21-28 (the reference's object works too)."""
    iterations: int = 3
    warmup_iterations: int = 1
    opt_seconds: float = 0.0
    async_iterations: bool = False
    adapter: AdapterConfig = AdapterConfig()
    seed: int = 0


@dataclass(frozen=True)
class SimSummary:
    """The scalar fields of SimReport (src/simulator.py:31-43), computed as
    simulate_timing does; per-op / per-transfer lists are not materialised,
    only their counts."""
    makespan: float
    throughput: float
    steady_throughput: float
    bubble_fractions: Tuple[float, ...]
    iteration_ends: Tuple[float, ...]
    adapter_action_count: int
    transfer_count: int
    op_count: int
    policy: str
    adapter_enabled: bool
    total_samples: int


def simulate_timings(timings: Sequence, policy="1f1b", traces: Sequence = (), trace_index=None,
                     adapter_enabled: bool = False, config=None, engine=None):
    """``simulate_timing(t, policy, traces[trace_index[i]], adapter_enabled,
    config)`` for every timing, batched on the GPU (one thread per timing).
    Raises the reference's exceptions (SchedulingBugError for a stalled
    engine, InvalidTimingError for malformed timings)."""
    from .engine import default_engine
    eng = engine if engine is not None else default_engine()
    config = config if config is not None else SimConfig()
    pol = getattr(policy, "value", policy)
    code = abi.POLICY_CODE[pol]
    arr = pack_timings(timings)
    tr = pack_traces(traces) if traces else None
    its = int(config.iterations)
    ad = getattr(config, "adapter", None)
    reps, ends, st = eng.simulate_report(
        arr, len(timings), code, its, tr, len(traces), trace_index, adapter=adapter_enabled,
        async_iterations=bool(getattr(config, "async_iterations", False)),
        degrade=getattr(ad, "degrade_factor", 1.2), recover=getattr(ad, "recover_factor", 1.05))
    bad = np.nonzero(st)[0]
    if bad.size:
        i = int(bad[0])
        if int(st[i]) == abi.GP_ERR_CUDA:
            raise D.DeviceError(f"timing {i}: simulator queue capacity exceeded")
        abi.raise_for(int(st[i]), f"timing {i}: event loop stalled with work remaining"
                      if int(st[i]) == abi.GP_ERR_SCHEDULING else f"timing {i} failed to simulate")
    out = []
    warm = min(int(config.warmup_iterations), its - 1)
    for i, t in enumerate(timings):
        r = reps[i]
        makespan = float(r.makespan)
        it_ends = tuple(float(x) for x in ends[i])
        total = int(t.batch) * its
        steady_samples = int(t.batch) * (its - warm)
        steady_start = it_ends[warm - 1] if warm > 0 else 0.0
        busy = [float(r.busy[s]) for s in range(len(t.stages))]
        out.append(SimSummary(
            makespan=makespan,
            throughput=total / makespan,
            steady_throughput=steady_samples / (makespan - steady_start),
            bubble_fractions=tuple((makespan - b) / makespan for b in busy),
            iteration_ends=it_ends,
            adapter_action_count=int(r.adapter_actions),
            transfer_count=int(r.n_transfers),
            op_count=int(r.n_ops),
            policy=pol,
            adapter_enabled=bool(adapter_enabled),
            total_samples=total,
        ))
    return out


def simulate_timing(timing, policy="1f1b", trace=None, adapter_enabled: bool = False,
                    config=None, engine=None) -> SimSummary:
    """Single-timing form of :func:`simulate_timings` (src/simulator.py:71-77)."""
    traces = (trace,) if trace is not None else ()
    return simulate_timings([timing], policy, traces, None, adapter_enabled, config, engine)[0]
