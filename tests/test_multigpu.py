"""Sharded product paths on >= 2 GPUs of one box (torchrun, NCCL): every
rank's answer equals the single-GPU reference answer (golden fixtures).

Skipped when fewer than two GPUs are visible (the single-GPU gate); run with
``gpurun --gpus 2`` / ``--gpus 4``.
"""

import json
import os
import subprocess
import sys

import pytest

import golden_io as G

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module")
def sharded(tmp_path_factory):
    n = _ngpu()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    path = str(tmp_path_factory.mktemp("mgpu") / "out.json")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29641", os.path.join(HERE, "mgpu_worker.py"),
           path]
    subprocess.run(cmd, check=True, timeout=600)
    with open(path) as f:
        return json.load(f)


def test_all_ranks_agree(sharded):
    assert sharded["world"] >= 2
    assert sharded["all_ranks_equal"]


@pytest.mark.parametrize("name", ["c1j", "c2", "c2j", "rand10", "k5n9", "k6n8", "k8n9"])
def test_sharded_exhaustive_matches_reference(sharded, name):
    assert sharded["exhaustive"][name] == G.load(f"{name}.json")["exhaustive"]["result"]


@pytest.mark.parametrize("name", ["c4", "c4j"])
def test_sharded_exhaustive_c4_matches_oracle(sharded, name):
    exp = G.load(f"{name}.json")["oracle_argmin"]
    res = sharded["exhaustive"][name]
    assert res["breakdown"]["plan_cost"] == exp["cost"]
    assert res["evaluated"] == exp["evaluated"]


@pytest.mark.parametrize("name", ["err_gateway", "err_intra_bw"])
def test_sharded_errors_match_reference(sharded, name):
    assert sharded["errors"][name] == G.load(f"{name}.json")["exhaustive"]["error"]


def test_sharded_snapshots_match_golden(sharded):
    snap = G.load("c3_snapshots.json")["snapshots"]
    got = sharded["snapshots"]
    assert len(got) == 37
    for j, r in enumerate(got):
        assert r[0] == snap[j]["cost"], j


def test_sharded_snapshots_with_raising_tables(sharded):
    assert sharded["flagged_equal"]
    assert sharded["flagged_errors"] >= 1
    assert sharded["refused_equal"], sharded["refused_kinds"]
    assert sharded["pinned_equal"]


def test_peer_memory_allgather_matches_nccl(sharded):
    assert sharded["peer_ok"], "peer-memory set-up failed (no P2P between the GPUs?)"
    assert sharded["peer_equal"] == [True, True, True]
    assert sharded["peer_pipelined_equal"] == [True] * 6
