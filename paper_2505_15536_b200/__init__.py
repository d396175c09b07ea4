"""paper_2505_15536_b200 - B200-native batched plan evaluation for DeepCEE.

Drop-in for the reference planner's hot path (``geopipe.search_plan`` /
``geopipe.exhaustive_plan`` and the batched ``_evaluate`` beneath them):
the same call signatures and result types, with every candidate evaluated by
hand-written sm_100a CUDA kernels behind the C-ABI in
``include/geopipe_b200.h``.  See DESIGN.md.
"""

from .domain import (
    Candidate,
    ClusterTopology,
    CostBreakdown,
    DegenerateGroupError,
    DeviceError,
    DeviceSpec,
    FirstLevelGroup,
    GeopipeError,
    GroupIndex,
    InfeasibleSplitError,
    InputFileError,
    IntraSplit,
    InvalidTopologyError,
    LayerSpec,
    ModelSpec,
    NoFeasiblePlanError,
    ParallelPlan,
    SearchConfig,
    SearchResult,
    SecondLevelGroup,
    SplitKind,
    StageAssignment,
    StageCost,
)
from .engine import Engine, default_engine
from .layout import PackedInstance
from .planner import exhaustive_plan, search_plan

__version__ = "0.1.0"

__all__ = [
    "Candidate", "ClusterTopology", "CostBreakdown", "DegenerateGroupError",
    "DeviceError", "DeviceSpec", "FirstLevelGroup", "GeopipeError", "GroupIndex",
    "InfeasibleSplitError", "InputFileError", "IntraSplit", "InvalidTopologyError",
    "LayerSpec", "ModelSpec", "NoFeasiblePlanError", "ParallelPlan", "SearchConfig",
    "SearchResult", "SecondLevelGroup", "SplitKind", "StageAssignment", "StageCost",
    "Engine", "default_engine", "PackedInstance", "exhaustive_plan", "search_plan",
]
