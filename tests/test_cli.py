"""CLI routed through the engine vs the reference CLI (src/cli.py).

Golden: tests/golden/cli_outputs.json = return code, stdout, stderr and
written files of the reference's ``geopipe`` CLI on the input files under
tests/golden/cli/ (scripts/make_golden.py dump_cli).
"""

import os

import pytest

import golden_io as G
from paper_2505_15536_b200 import domain as D
from paper_2505_15536_b200 import fileio
from paper_2505_15536_b200.cli import main

from cli_cases import cli_commands, run_cli

GOLD = G.load("cli_outputs.json")
INPUTS = os.path.join(G.GOLDEN, "cli")
CMDS = cli_commands()


def _run(case, argv, tmp):
    args = [a.replace("{d}", INPUTS).replace("{o}", str(tmp)) for a in argv]
    rc, so, se = run_cli(main, args)
    return rc, so.replace(INPUTS, "{d}").replace(str(tmp), "{o}"), \
        se.replace(INPUTS, "{d}").replace(str(tmp), "{o}"), args


def test_fileio_reads_instances_like_the_instance_builder():
    from paper_2505_15536_b200 import instances as I
    for name in ("c1", "c2"):
        topo = fileio.read_cluster(os.path.join(INPUTS, f"{name}_cluster.json"))
        model = fileio.read_model(os.path.join(INPUTS, f"{name}_model.json"))
        m2, t2, _ = I.load(name, True)
        assert model == m2
        assert topo.devices == tuple(D.DeviceSpec(d.id, d.memory_bytes, d.benchmark_times,
                                                  d.region_tag) for d in topo.devices)
        assert {d: topo.p_c(d) for d in topo.device_ids} == {d: t2.p_c(d) for d in t2.device_ids}
        assert topo.links == t2.links


def test_bad_file_diagnostic_matches_reference(tmp_path):
    rc, so, se, _ = _run("bad:group", dict(CMDS)["bad:group"], tmp_path)
    exp = GOLD["bad:group"]
    assert (rc, so, se) == (exp["rc"], exp["stdout"], exp["stderr"])


def test_fileio_errors_name_the_field(tmp_path):
    p = tmp_path / "m.json"
    p.write_text('{"schema": "model/v1", "layers": [{"fwd_flops": 1.0}]}')
    with pytest.raises(D.InputFileError, match="activation_out_bytes"):
        fileio.read_model(p)
    p.write_text('{"schema": "plan/v2"}')
    with pytest.raises(D.InputFileError, match="schema"):
        fileio.read_plan(p)


@pytest.mark.gpu
def test_cli_matches_reference(tmp_path):
    """Every golden command, in order (later commands read the plan files
    the earlier ``plan`` commands wrote)."""
    for case, argv in CMDS:
        rc, so, se, args = _run(case, argv, tmp_path)
        exp = GOLD[case]
        assert rc == exp["rc"], (case, se)
        assert so == exp["stdout"], case
        assert se == exp["stderr"], case
        for name, text in exp["files"].items():
            assert (tmp_path / name).read_text() == text, (case, name)
