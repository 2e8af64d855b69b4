"""The command line mirror (paper_1304_5966_b200/cli.py) against golden runs
of the reference's cli.run_cli (tests/golden/make_golden_cli.py): identical
exit codes everywhere and byte-identical stdout for the alignments.  Error
runs stop before the device and run on CPU; alignments need the GPU."""
import contextlib
import io

import pytest

from conftest import load_golden
from paper_1304_5966_b200 import cli

GOLDEN = load_golden("golden_cli.json.gz")


def _run(tmp_path, args):
    for name, text in GOLDEN["files"].items():
        (tmp_path / name).write_text(text)
    argv = [str(tmp_path / a) if a in GOLDEN["files"] or a.endswith(".fa") else a for a in args]
    so, se = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
        rc = cli.run_cli(argv)
    return rc, so.getvalue(), se.getvalue()


ERRORS = [r for r in GOLDEN["runs"] if r["rc"] != 0]
RUNS = [r for r in GOLDEN["runs"] if r["rc"] == 0]


@pytest.mark.parametrize("case", ERRORS, ids=[" ".join(r["args"]) for r in ERRORS])
def test_cli_errors(tmp_path, case):
    rc, out, err = _run(tmp_path, case["args"])
    assert rc == case["rc"]
    assert out == case["stdout"] == ""
    assert err  # a message on standard error


@pytest.mark.gpu
@pytest.mark.parametrize("case", RUNS, ids=[" ".join(r["args"]) for r in RUNS])
def test_cli_outputs(tmp_path, case):
    rc, out, _ = _run(tmp_path, case["args"])
    assert rc == 0
    assert out == case["stdout"]


@pytest.mark.gpu
def test_cli_output_file(tmp_path):
    case = next(r for r in RUNS if r["args"][-1] == "pair")
    rc, out, _ = _run(tmp_path, case["args"] + ["--output", str(tmp_path / "o.txt")])
    assert rc == 0 and out == ""
    assert (tmp_path / "o.txt").read_text() == case["stdout"]
