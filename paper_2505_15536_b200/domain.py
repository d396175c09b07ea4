"""Value types of the plan-evaluation boundary, mirroring the reference API.

The drop-in functions in :mod:`paper_2505_15536_b200.planner` accept the
reference's own objects (``geopipe.ModelSpec``, ``geopipe.ClusterTopology``,
``geopipe.timing.GroupIndex``) or these mirrors interchangeably: only the
attribute names below are read (duck typing).  Results are returned as these
mirrors, whose fields and field order equal the reference's:

* ``LayerSpec`` / ``ModelSpec``            -> ``src/plans.py:12-57``
* ``SplitKind`` / ``IntraSplit`` / ``StageAssignment`` / ``ParallelPlan``
                                          -> ``src/plans.py:60-134``
* ``DeviceSpec`` / ``LinkInfo`` / ``ClusterTopology``
                                          -> ``src/profiling.py:23-45,116-156``
* ``FirstLevelGroup`` / ``SecondLevelGroup`` -> ``src/grouping.py:21-39``
* ``GroupIndex``                          -> ``src/timing.py:28-44``
* ``StageCost`` / ``CostBreakdown``       -> ``src/costmodel.py:27-43``
* ``Candidate`` / ``SearchConfig`` / ``SearchResult``
                                          -> ``src/planner.py:36-62``
* exception classes                       -> ``src/errors.py:4-66``

(``src/`` = ``/root/reference/pkg/src/geopipe/``.)  Nothing in this module
computes a plan cost; it only holds data.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, FrozenSet, List, Optional, Tuple


# --------------------------------------------------------------------------
# errors (src/errors.py:4-66); the C-ABI status codes map onto these
# --------------------------------------------------------------------------

class GeopipeError(Exception):
    """Root of every error raised by the planner boundary."""


class InputFileError(GeopipeError):
    """Invalid input value (C-ABI status 1)."""


class InfeasibleSplitError(GeopipeError):
    """More pipeline stages than layers (C-ABI status 2)."""


class NoFeasiblePlanError(GeopipeError):
    """Every candidate violated device memory (C-ABI status 3)."""


class DegenerateGroupError(GeopipeError):
    """A stage's group has no usable compute capacity (C-ABI status 4)."""


class InvalidTopologyError(GeopipeError):
    """A link with zero bandwidth is on the plan's path (C-ABI status 5)."""


class DeviceError(GeopipeError):
    """The CUDA engine failed or is unavailable (C-ABI status 6)."""


class InvalidTimingError(GeopipeError):
    """Timing vectors inconsistent with the stage count (src/errors.py:53)."""


class EmptyClusterError(GeopipeError):
    """Grouping was asked to run on a topology with no devices."""


class InvalidMeasurementError(GeopipeError):
    """A link measurement violates its invariants (src/errors.py:8-9)."""


class InvalidBenchmarkError(GeopipeError):
    """A compute benchmark list is empty or has non-positive times."""


class IncompleteTopologyError(GeopipeError):
    """The link matrix is missing pairs or contains duplicates."""

    def __init__(self, message, missing=(), duplicates=()):
        super().__init__(message)
        self.missing = list(missing)
        self.duplicates = list(duplicates)


class SchedulingBugError(GeopipeError):
    """The 1F1B event loop stalled (src/errors.py:57-62)."""

    def __init__(self, message, state_dump=None):
        super().__init__(message)
        self.state_dump = state_dump or {}


# --------------------------------------------------------------------------
# model and plan (src/plans.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class LayerSpec:
    fwd_flops: float
    bwd_input_flops: float
    bwd_weight_flops: float
    activation_out_bytes: float
    param_bytes: float

    def __post_init__(self):  # src/plans.py:22-26
        for name in ("fwd_flops", "bwd_input_flops", "bwd_weight_flops",
                     "activation_out_bytes", "param_bytes"):
            if getattr(self, name) <= 0:
                raise InputFileError(f"layer field {name} must be positive")

    @property
    def total_flops(self) -> float:
        # association as in src/plans.py:28-30
        return (self.fwd_flops + self.bwd_input_flops) + self.bwd_weight_flops


@dataclass(frozen=True)
class ModelSpec:
    layers: Tuple[LayerSpec, ...]
    global_batch_candidates: Tuple[int, ...] = (128, 256)
    microbatch_candidates: Tuple[int, ...] = (8, 16, 32)

    def __post_init__(self):  # src/plans.py:41-53
        if not self.layers:
            raise InputFileError("model has no layers")
        for b in self.global_batch_candidates:
            if b <= 0:
                raise InputFileError("batch candidates must be positive")
            for m in self.microbatch_candidates:
                if m <= 0:
                    raise InputFileError("micro-batch candidates must be positive")
                if b % m != 0:
                    raise InputFileError(f"micro-batch {m} does not divide batch {b}")

    @property
    def num_layers(self) -> int:
        return len(self.layers)


class SplitKind(enum.Enum):
    UNIFORM = "uniform"
    ASYMMETRIC_PP = "asymmetric_pp"
    ASYMMETRIC_DP = "asymmetric_dp"
    ASYMMETRIC_TP_DP = "asymmetric_tp_dp"


@dataclass(frozen=True)
class IntraSplit:
    kind: SplitKind
    parts: Tuple[tuple, ...] = ()


@dataclass(frozen=True)
class StageAssignment:
    fg_id: str
    layer_start: int
    layer_end: int
    intra_split: IntraSplit = IntraSplit(SplitKind.UNIFORM)

    @property
    def layer_range(self) -> range:
        return range(self.layer_start, self.layer_end)


@dataclass(frozen=True)
class ParallelPlan:
    stages: Tuple[StageAssignment, ...]
    batch_b: int
    microbatch_m: int

    def __post_init__(self):  # src/plans.py:106-122
        if self.batch_b <= 0 or self.microbatch_m <= 0:
            raise InputFileError("batch and micro-batch must be positive")
        if self.batch_b % self.microbatch_m != 0:
            raise InputFileError(
                f"micro-batch {self.microbatch_m} does not divide batch {self.batch_b}")
        fgs = [s.fg_id for s in self.stages]
        if len(set(fgs)) != len(fgs):
            raise InputFileError("stage order must use distinct first-level groups")
        pos = 0
        for s in self.stages:
            if s.layer_start != pos or s.layer_end <= s.layer_start:
                raise InputFileError("stage layer ranges must tile the layer list without gaps")
            pos = s.layer_end

    @property
    def micro_count(self) -> int:
        return self.batch_b // self.microbatch_m

    @property
    def num_layers(self) -> int:
        return self.stages[-1].layer_end

    @property
    def num_stages(self) -> int:
        return len(self.stages)


# --------------------------------------------------------------------------
# topology and groups (src/profiling.py, src/grouping.py, src/timing.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class DeviceSpec:
    id: str
    memory_bytes: float
    benchmark_times: Tuple[Tuple[str, float], ...] = ()
    region_tag: str = ""


@dataclass(frozen=True)
class CommMetric:
    p_t: float


@dataclass(frozen=True)
class ComputeMetric:
    p_c: float


@dataclass(frozen=True)
class LinkInfo:
    metric: CommMetric
    latency_seconds: float
    bandwidth_bytes_per_s: float


@dataclass(frozen=True)
class ClusterTopology:
    """Devices (sorted by id) with p_c and a complete symmetric link matrix."""

    devices: Tuple[DeviceSpec, ...]
    compute: Dict[str, ComputeMetric] = field(compare=False)
    links: Dict[FrozenSet[str], LinkInfo] = field(compare=False)

    @property
    def device_ids(self) -> List[str]:
        return [d.id for d in self.devices]

    def device(self, device_id: str) -> DeviceSpec:
        for d in self.devices:
            if d.id == device_id:
                return d
        raise KeyError(device_id)

    def p_c(self, device_id: str) -> float:
        return self.compute[device_id].p_c

    def p_t(self, a: str, b: str) -> float:
        return self.links[frozenset((a, b))].metric.p_t

    def link(self, a: str, b: str) -> LinkInfo:
        return self.links[frozenset((a, b))]

    def bandwidth(self, a: str, b: str) -> float:
        return self.links[frozenset((a, b))].bandwidth_bytes_per_s

    def latency(self, a: str, b: str) -> float:
        return self.links[frozenset((a, b))].latency_seconds


@dataclass(frozen=True)
class FirstLevelGroup:
    id: str
    member_device_ids: Tuple[str, ...]
    intra_metric: Optional[float]
    aggregate_capacity: float
    min_intra_bandwidth: Optional[float]


@dataclass(frozen=True)
class SecondLevelGroup:
    id: str
    parent_fg_id: str
    member_device_ids: Tuple[str, ...]
    aggregate_capacity: float


@dataclass(frozen=True)
class GroupIndex:
    fgs: Dict[str, FirstLevelGroup]
    sgs: Dict[str, SecondLevelGroup]
    sgs_by_fg: Dict[str, Tuple[SecondLevelGroup, ...]]

    @staticmethod
    def build(fgs, sgs_by_fg) -> "GroupIndex":
        return GroupIndex(
            fgs={fg.id: fg for fg in fgs},
            sgs={sg.id: sg for v in sgs_by_fg.values() for sg in v},
            sgs_by_fg={k: tuple(v) for k, v in sgs_by_fg.items()},
        )


# --------------------------------------------------------------------------
# cost and search results (src/costmodel.py, src/planner.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class StageCost:
    fill_seconds: float
    run_seconds: float
    residual_seconds: float
    collective_seconds: float

    @property
    def total(self) -> float:
        return (((self.fill_seconds + self.run_seconds)
                 + self.residual_seconds) + self.collective_seconds)


@dataclass(frozen=True)
class CostBreakdown:
    per_stage: Tuple[StageCost, ...]
    plan_cost: float


@dataclass(frozen=True)
class Candidate:
    order: Tuple[str, ...]
    counts: Tuple[int, ...]


@dataclass(frozen=True)
class SearchConfig:
    seed: int
    beam_width: int = 8
    max_iter: int = 20
    bottleneck_factor: float = 1.25
    opt_seconds: float = 0.0

    def __post_init__(self):
        if self.beam_width < 1 or self.max_iter < 1:
            raise ValueError("beam_width and max_iter must be >= 1")


@dataclass
class SearchResult:
    plan: ParallelPlan
    breakdown: CostBreakdown
    best_cost_trace: List[float]
    evaluated: int
