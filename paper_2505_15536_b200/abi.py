"""ctypes mirror of ``include/geopipe_b200.h`` (structs, status codes).

Kept in one place so the product binding (:mod:`.engine`) and the test-only
oracle binding (``oracle/oracle.py``) agree on the layout byte for byte.
"""

from __future__ import annotations

import ctypes as C

from . import domain as D

GP_OK = 0
GP_ERR_INPUT = 1
GP_ERR_INFEASIBLE_SPLIT = 2
GP_ERR_NO_FEASIBLE = 3
GP_ERR_DEGENERATE = 4
GP_ERR_TOPOLOGY = 5
GP_ERR_CUDA = 6
GP_ERR_TIMING = 7
GP_ERR_SCHEDULING = 8

GP_UNIFORM, GP_ASYM_PP, GP_ASYM_DP, GP_ASYM_TP_DP = 0, 1, 2, 3
KIND_OF = {
    GP_UNIFORM: D.SplitKind.UNIFORM,
    GP_ASYM_PP: D.SplitKind.ASYMMETRIC_PP,
    GP_ASYM_DP: D.SplitKind.ASYMMETRIC_DP,
    GP_ASYM_TP_DP: D.SplitKind.ASYMMETRIC_TP_DP,
}

GP_MAX_STAGES = 16
GP_MAX_SGS = 16
GP_MAX_LAYERS = 255
GP_MAX_MEMBERS = 1024

_ERRORS = {
    GP_ERR_INPUT: D.InputFileError,
    GP_ERR_INFEASIBLE_SPLIT: D.InfeasibleSplitError,
    GP_ERR_NO_FEASIBLE: D.NoFeasiblePlanError,
    GP_ERR_DEGENERATE: D.DegenerateGroupError,
    GP_ERR_TOPOLOGY: D.InvalidTopologyError,
    GP_ERR_CUDA: D.DeviceError,
    GP_ERR_TIMING: D.InvalidTimingError,
    GP_ERR_SCHEDULING: D.SchedulingBugError,
}


def raise_for(status: int, message: str = "") -> None:
    if status == GP_OK:
        return
    cls = _ERRORS.get(status, D.GeopipeError)
    raise cls(message or f"status {status}")


_dp = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)


class GpInstance(C.Structure):
    _fields_ = [
        ("n_layers", C.c_uint32),
        ("fwd_flops", _dp), ("bwd_input_flops", _dp), ("bwd_weight_flops", _dp),
        ("activation_out_bytes", _dp), ("param_bytes", _dp),
        ("n_batch", C.c_uint32), ("batch", _i64p),
        ("n_micro", C.c_uint32), ("micro", _i64p),
        ("n_devices", C.c_uint32),
        ("p_c", _dp), ("memory_bytes", _dp), ("id_rank", _u32p),
        ("p_t", _dp), ("latency", _dp), ("bandwidth", _dp),
        ("n_fgs", C.c_uint32),
        ("fg_member_offset", _u32p), ("fg_members", _u32p),
        ("fg_capacity", _dp), ("fg_min_bw", _dp), ("fg_has_min_bw", _u8p),
        ("fg_sg_offset", _u32p), ("sg_member_offset", _u32p),
        ("sg_members", _u32p), ("sg_capacity", _dp),
        ("bottleneck_factor", C.c_double),
    ]


class GpBest(C.Structure):
    _fields_ = [
        ("cost", C.c_double), ("index", C.c_uint64),
        ("batch_index", C.c_uint32), ("micro_index", C.c_uint32),
        ("k", C.c_uint32),
        ("order", C.c_uint8 * GP_MAX_STAGES), ("counts", C.c_uint8 * GP_MAX_STAGES),
        ("evaluated", C.c_uint64),
    ]


class GpStageInfo(C.Structure):
    _fields_ = [
        ("kind", C.c_uint32), ("n_parts", C.c_uint32),
        ("pp_sg", C.c_uint32 * GP_MAX_SGS),
        ("pp_start", C.c_uint32 * GP_MAX_SGS),
        ("pp_end", C.c_uint32 * GP_MAX_SGS),
        ("fill_seconds", C.c_double), ("run_seconds", C.c_double),
        ("residual_seconds", C.c_double), ("collective_seconds", C.c_double),
    ]


class GpPlanInfo(C.Structure):
    _fields_ = [
        ("feasible", C.c_int32), ("k", C.c_uint32), ("plan_cost", C.c_double),
        ("stage", GpStageInfo * GP_MAX_STAGES),
    ]


class GpGroupInfo(C.Structure):
    _fields_ = [
        ("tp_ok", C.c_int32), ("n_members", C.c_uint32), ("n_sgs", C.c_uint32),
        ("tp_row", C.c_double * GP_MAX_MEMBERS),
        ("tp_col", C.c_double * GP_MAX_MEMBERS),
        ("dp_fraction", C.c_double * GP_MAX_SGS),
    ]


class GpTiming(C.Structure):
    _fields_ = [
        ("n_stages", C.c_uint32), ("pad", C.c_uint32),
        ("batch", C.c_int64), ("microbatch", C.c_int64),
        ("fwd", C.c_double * GP_MAX_STAGES), ("bwd", C.c_double * GP_MAX_STAGES),
        ("wgt", C.c_double * GP_MAX_STAGES), ("sync", C.c_double * GP_MAX_STAGES),
        ("opt", C.c_double * GP_MAX_STAGES), ("lat", C.c_double * GP_MAX_STAGES),
        ("bw", C.c_double * GP_MAX_STAGES), ("act", C.c_double * GP_MAX_STAGES),
        ("grad", C.c_double * GP_MAX_STAGES),
    ]


GP_POLICY_GPIPE, GP_POLICY_1F1B, GP_POLICY_ZB_ORIGINAL, GP_POLICY_ZB_COMPACT = 0, 1, 2, 3
POLICY_CODE = {"gpipe": 0, "1f1b": 1, "zb_original": 2, "zb_compact": 3}
GP_MAX_BREAKPOINTS = 256


class GpTrace(C.Structure):
    _fields_ = [
        ("n_points", C.c_uint32 * GP_MAX_STAGES),
        ("t", (C.c_double * GP_MAX_BREAKPOINTS) * GP_MAX_STAGES),
        ("mult", (C.c_double * GP_MAX_BREAKPOINTS) * GP_MAX_STAGES),
    ]


class GpSimOptions(C.Structure):
    _fields_ = [
        ("adapter", C.c_uint32), ("async_iterations", C.c_uint32),
        ("degrade_factor", C.c_double), ("recover_factor", C.c_double),
    ]


class GpSimReport(C.Structure):
    _fields_ = [
        ("makespan", C.c_double), ("busy", C.c_double * GP_MAX_STAGES),
        ("adapter_actions", C.c_uint32), ("n_ops", C.c_uint32),
        ("n_transfers", C.c_uint32), ("pad", C.c_uint32),
    ]


class GpOp(C.Structure):
    _fields_ = [
        ("start", C.c_double), ("end", C.c_double), ("size", C.c_int32),
        ("microbatch_id", C.c_int32), ("iteration", C.c_uint32),
        ("kind", C.c_uint8), ("stage", C.c_uint8), ("pad", C.c_uint16),
    ]


class GpTransfer(C.Structure):
    _fields_ = [
        ("start", C.c_double), ("end", C.c_double), ("size", C.c_int32),
        ("microbatch_id", C.c_int32), ("iteration", C.c_uint32),
        ("boundary", C.c_uint8), ("direction", C.c_uint8), ("pad", C.c_uint16),
    ]


class GpAction(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("stage", C.c_int32), ("old_size", C.c_int32),
        ("new_size", C.c_int32), ("signal", C.c_uint32),
    ]


ACTION_SIGNALS = ("fill", "drain", "degraded", "recovered")


class GpViolation(C.Structure):
    _fields_ = [
        ("t", C.c_double), ("iteration", C.c_uint32), ("microbatch_id", C.c_int32),
        ("code", C.c_uint8), ("stage", C.c_uint8), ("kind", C.c_uint8), ("pad", C.c_uint8),
        ("pad2", C.c_uint32),
    ]


OP_KINDS = ("F", "B", "W", "S", "O")


class GpPlanStage(C.Structure):
    _fields_ = [
        ("fg", C.c_uint32), ("layer_start", C.c_uint32), ("layer_end", C.c_uint32),
        ("kind", C.c_uint32), ("n_parts", C.c_uint32),
        ("pp_sg", C.c_uint32 * GP_MAX_SGS), ("pp_start", C.c_uint32 * GP_MAX_SGS),
        ("pp_end", C.c_uint32 * GP_MAX_SGS),
    ]


KIND_CODE = {v: k for k, v in KIND_OF.items()}
