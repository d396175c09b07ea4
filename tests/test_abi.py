"""The C-ABI library: built for sm_100a, exports every symbol the header
declares, ctypes layouts equal the C compiler's, and it refuses to run
without a B200 (no CPU fallback)."""

import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2505_15536_b200 import abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "geopipe_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(gp_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def built_lib():
    if not os.path.exists(engine.LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2505_15536_b200", "csrc")],
                       check=True)
    return engine.LIB_PATH


def test_header_declares_entry_points():
    names = _declared()
    for n in ["gp_ctx_create", "gp_ctx_load", "gp_eval_batch", "gp_argmin_range",
              "gp_plan_detail", "gp_set_bandwidth", "gp_ctx_destroy", "gp_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol(built_lib):
    out = subprocess.run(["nm", "-D", "--defined-only", built_lib], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gp_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_library_is_sm100a(built_lib):
    out = subprocess.run(["cuobjdump", "--list-elf", built_lib], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_ctypes_layout_matches_c(oracle_lib):
    L = oracle_lib.lib()
    L.or_abi_sizeof.restype = C.c_size_t
    for i, t in enumerate([abi.GpInstance, abi.GpBest, abi.GpPlanInfo, abi.GpGroupInfo,
                           abi.GpStageInfo]):
        assert L.or_abi_sizeof(i) == C.sizeof(t)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(built_lib):
    from paper_2505_15536_b200 import DeviceError, exhaustive_plan, SearchConfig
    from paper_2505_15536_b200 import instances as I
    with pytest.raises(DeviceError):
        engine.Engine(0)
    m, t, g = I.load("c1")
    with pytest.raises(DeviceError):
        exhaustive_plan(m, t, g, SearchConfig(seed=0), engine=None)
