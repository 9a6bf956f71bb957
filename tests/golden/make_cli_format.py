"""Golden record/stats streams of the reference CLI's default search
(cli.py:116-149 formats; test_cli.py:12-18 default invocation: exp, p=13,
eps=2^-8, binade 0, N=16, regular).  Runs the reference in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_format.py

Writes cli_default_records.jsonl / .csv and cli_default_stats.csv (the
stats' wall_ms column replaced by "-", being a timing).
"""
import csv
import io
import os

from hardround.cli import _emit_records, _emit_stats, _pipeline_config, build_parser
from hardround.pipeline import run_pipeline

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    args = build_parser().parse_args(["search"])
    cfg = _pipeline_config(args)
    records, stats = run_pipeline(args.binade, cfg)
    for kind in ("jsonl", "csv"):
        buf = io.StringIO()
        _emit_records(records, kind, buf)
        with open(os.path.join(HERE, f"cli_default_records.{kind}"), "w", newline="") as fh:
            fh.write(buf.getvalue())
    buf = io.StringIO()
    _emit_stats(stats, buf)
    rows = list(csv.reader(io.StringIO(buf.getvalue())))
    for r in rows[1:]:
        if r[0] != "choice":
            r[4] = "-"
    with open(os.path.join(HERE, "cli_default_stats.csv"), "w", newline="") as fh:
        csv.writer(fh, lineterminator="\n").writerows(rows)
    print(len(records), "records")


if __name__ == "__main__":
    main()
