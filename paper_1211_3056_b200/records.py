"""Record and stats streams in the reference's formats.

Restates the reference CLI's writers (cli.py:116-149) so that output from
`run_pipeline`, `run_slice`, `run_range` or the multi-GPU merge
(`shard.run_sharded`) can be written as the reference writes it:
- records as JSON lines or CSV, in argument order;
- phase stats as CSV.

For equal records the output is byte-identical to the reference's
(tests/test_records.py checks it against streams the reference wrote,
tests/golden/make_cli_format.py).
"""
from __future__ import annotations

import csv
import json
from typing import IO, Iterable

from .fpformat import HrCaseRecord

RECORD_FIELDS = ("arg_bits", "distance_num", "distance_den_log2", "domain")
STATS_FIELDS = ("phase", "domains_in", "domains_out", "arguments_covered", "wall_ms")
FORMATS = ("jsonl", "csv")


def record_dict(rec: HrCaseRecord) -> dict:
    """cli.py:116-125: the key order is part of the format."""
    out = {
        "arg_bits": hex(rec.argument),
        "distance_num": rec.distance.raw,
        "distance_den_log2": rec.distance.width,
        "domain": rec.domain_id,
    }
    if rec.undecided:
        out["undecided"] = True
    return out


def emit_records(records: Iterable[HrCaseRecord], kind: str, sink: IO[str]) -> None:
    """cli.py:128-138.  `kind` is "jsonl" or "csv"; the CSV form has a header
    row and no `undecided` column, as in the reference."""
    if kind not in FORMATS:
        raise ValueError(f"unknown record format {kind!r}; expected one of {FORMATS}")
    if kind == "jsonl":
        for rec in records:
            sink.write(json.dumps(record_dict(rec), sort_keys=False) + "\n")
        return
    writer = csv.writer(sink, lineterminator="\n")
    writer.writerow(RECORD_FIELDS)
    for rec in records:
        d = record_dict(rec)
        writer.writerow([d[k] for k in RECORD_FIELDS])


def emit_stats(stats, sink: IO[str]) -> None:
    """cli.py:141-149: one row per phase, then one `choice` row per
    algorithm choice."""
    writer = csv.writer(sink, lineterminator="\n")
    writer.writerow(STATS_FIELDS)
    for row in stats.rows:
        writer.writerow([row.phase, row.domains_in, row.domains_out, row.arguments_covered, f"{row.wall_ms:.3f}"])
    for piece, choice in stats.algorithm_choices:
        writer.writerow(["choice", piece, choice, "", ""])


def write_records(path: str, records: Iterable[HrCaseRecord], kind: str = "jsonl") -> None:
    """The reference's `--out` file: UTF-8, newline translation off
    (cli.py:156-157)."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        emit_records(records, kind, fh)
