"""Commands of the CLI goldens (shared by scripts/make_golden.py and
tests/test_cli.py)."""

from __future__ import annotations


def cli_commands():
    """(case, argv) of the CLI goldens; {d} is the inputs directory, {o} an
    output directory the command may write to."""
    cmds = []
    for base in ("small", "hetero", "c1", "c2"):
        c, m = f"{{d}}/{base}_cluster.json", f"{{d}}/{base}_model.json"
        cmds.append((f"{base}:group", ["group", c]))
        cmds.append((f"{base}:group-dot", ["group", c, "--dot"]))
        cmds.append((f"{base}:plan", ["plan", c, m, "--seed", "0", "--out", f"{{o}}/{base}_plan.json"]))
        cmds.append((f"{base}:plan-exhaustive", ["plan", c, m, "--exhaustive"]))
        p = f"{{o}}/{base}_plan.json"
        cmds.append((f"{base}:cost", ["cost", c, m, p]))
        cmds.append((f"{base}:simulate", ["simulate", c, m, p]))
        cmds.append((f"{base}:simulate-zb-adapter-trace",
                     ["simulate", c, m, p, "--policy", "zb_compact", "--adapter", "--trace",
                      "{d}/trace.json", "--iterations", "4"]))
        cmds.append((f"{base}:compare", ["compare", c, m, p, "--adapter", "--trace",
                                         "{d}/trace.json"]))
    hc, hm, he = "{d}/hetero_cluster.json", "{d}/hetero_model.json", "{d}/hetero_plan_edited.json"
    cmds.append(("hetero:cost-edited", ["cost", hc, hm, he]))
    cmds.append(("hetero:simulate-edited", ["simulate", hc, hm, he, "--policy", "gpipe"]))
    cmds.append(("hetero:compare-edited", ["compare", hc, hm, he]))
    cmds.append(("small:plan-seed3", ["plan", "{d}/small_cluster.json", "{d}/small_model.json",
                                      "--seed", "3", "--beam-width", "2", "--max-iter", "5"]))
    cmds.append(("bad:group", ["group", "{d}/bad_cluster.json"]))
    return cmds


def run_cli(main_fn, argv):
    import contextlib
    import io
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        try:
            rc = main_fn(argv)
        except SystemExit as e:
            rc = e.code
    return rc, out.getvalue(), err.getvalue()
