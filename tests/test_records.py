"""Record / stats streams in the reference CLI's formats (cli.py:116-149),
byte-compared with streams the reference itself wrote
(tests/golden/make_cli_format.py: the default `search` invocation, whose
first record and count test_cli.py:12-18 pins)."""
import csv
import io
import json
import os

import pytest

from golden_io import case, config_of

from paper_1211_3056_b200.arith import UFrac
from paper_1211_3056_b200.fpformat import HrCaseRecord
from paper_1211_3056_b200.funnel import PhaseRow, PhaseStats
from paper_1211_3056_b200.records import emit_records, emit_stats, record_dict, write_records

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden_text(name):
    with open(os.path.join(GOLDEN, name), newline="") as fh:
        return fh.read()


def golden_records():
    c = case("p13_cli_default")
    return [HrCaseRecord(int(a, 16), UFrac(raw, 64), dom, und) for a, raw, dom, und in c["records"]]


def render(records, kind):
    buf = io.StringIO()
    emit_records(records, kind, buf)
    return buf.getvalue()


def normalised_stats(text):
    rows = list(csv.reader(io.StringIO(text)))
    for r in rows[1:]:
        if r[0] != "choice":
            assert float(r[4]) >= 0.0
            r[4] = "-"
    buf = io.StringIO()
    csv.writer(buf, lineterminator="\n").writerows(rows)
    return buf.getvalue()


@pytest.mark.parametrize("kind", ["jsonl", "csv"])
def test_records_byte_identical_to_reference(kind):
    assert render(golden_records(), kind) == golden_text(f"cli_default_records.{kind}")


def test_first_record_and_count():
    """test_cli.py:12-18, 28-39."""
    lines = render(golden_records(), "jsonl").splitlines()
    assert len(lines) == 42
    first = json.loads(lines[0])
    assert first == {"arg_bits": "0x8001046", "distance_num": 24674833356615680, "distance_den_log2": 64, "domain": 4}
    assert list(first) == ["arg_bits", "distance_num", "distance_den_log2", "domain"]


def test_undecided_flag_and_bad_kind(tmp_path):
    rec = HrCaseRecord(0x10, UFrac(5, 64), 3, True)
    assert record_dict(rec)["undecided"] is True
    assert render([rec], "csv").splitlines()[1] == "0x10,5,64,3"   # the CSV form has no undecided column
    with pytest.raises(ValueError):
        render([rec], "xml")
    path = tmp_path / "r.jsonl"
    write_records(str(path), golden_records())
    assert path.read_bytes() == golden_text("cli_default_records.jsonl").encode()


def test_stats_format():
    c = case("p13_cli_default")
    st = c["stats"]
    rows = [PhaseRow("phase1", st["phase1"][0], st["phase1"][1], st["phase1"][2], 1.5),
            PhaseRow("phase2", st["phase2"][0], st["phase2"][1], st["phase2"][2], 0.25),
            PhaseRow("phase3", st["phase3"][0], st["phase3"][1], st["phase3"][2], 0.0),
            PhaseRow("confirm", st["confirm"][0], st["confirm"][1], st["confirm"][0], 12.0)]
    buf = io.StringIO()
    emit_stats(PhaseStats(rows, [(0, "regular")]), buf)
    assert buf.getvalue().splitlines()[1].endswith(",1.500")
    assert normalised_stats(buf.getvalue()) == golden_text("cli_default_stats.csv")


@pytest.mark.gpu
def test_run_pipeline_streams_match_reference():
    """The device pipeline's records and stats, written in the reference's
    formats, equal the reference CLI's default output."""
    from paper_1211_3056_b200 import run_pipeline

    records, stats = run_pipeline(0, config_of(case("p13_cli_default")))
    for kind in ("jsonl", "csv"):
        assert render(records, kind) == golden_text(f"cli_default_records.{kind}")
    buf = io.StringIO()
    emit_stats(stats, buf)
    assert normalised_stats(buf.getvalue()) == golden_text("cli_default_stats.csv")
