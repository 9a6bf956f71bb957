"""The command-line entry point (cli.py), shaped like the reference's
(cli.py:221-271): same flags, defaults, streams and exit codes; the record
stream of the default search is byte-identical to the one the reference
wrote (tests/golden/cli_default_records.*, make_cli_format.py)."""
import io
import json
import os
from contextlib import redirect_stderr, redirect_stdout

import pytest

from paper_1211_3056_b200.cli import main

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _run(argv):
    out, err = io.StringIO(), io.StringIO()
    with redirect_stdout(out), redirect_stderr(err):
        rc = main(argv)
    return rc, out.getvalue(), err.getvalue()


@pytest.mark.parametrize("argv", [["search", "--range", "17"], ["search", "--range", "0:99999999"],
                                  ["search", "--phase2-split", "3"], ["search", "--p", "1"]])
def test_configuration_errors_exit_2(argv):
    rc, out, err = _run(argv)
    assert rc == 2 and "configuration error" in err and out == ""


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["jsonl", "csv"])
def test_default_search_is_byte_identical_to_the_reference(fmt):
    rc, out, err = _run(["search", "--format", fmt])
    assert rc == 0
    with open(os.path.join(GOLDEN, f"cli_default_records.{fmt}")) as fh:
        assert out == fh.read()
    assert err.splitlines()[0] == "phase,domains_in,domains_out,arguments_covered,wall_ms"


@pytest.mark.gpu
def test_range_and_degree_flags_give_the_exhaustive_records():
    """search --range over a 2^20-argument binary64 slice, at the reference's
    degree 2 and at degree 4 (the high-degree path): the records equal the
    reference's exhaustive enumeration (tests/golden/exhaustive.json)."""
    with open(os.path.join(GOLDEN, "exhaustive.json")) as fh:
        c = next(x for x in json.load(fh) if x["name"] == "exp_p53_2p20_e16")
    for degree in ("2", "4"):
        rc, out, err = _run(["search", "--p", "53", "--eps-bits", "16", "--domain-bits", "15",
                             "--range", f"{c['start']}:{c['count']}", "--degree", degree, "--interval", "20"])
        assert rc == 0, err
        got = [json.loads(line) for line in out.splitlines()]
        assert [[r["arg_bits"], r["distance_num"], bool(r.get("undecided", False))] for r in got] == c["records"]
