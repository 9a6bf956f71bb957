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
from collections.abc import Sequence
from typing import IO, Iterable

import numpy as np

from .arith import UFrac
from .fpformat import EXP_BIAS, HrCaseRecord

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
        if isinstance(records, RecordSet) and not records.undecided.any():
            # same bytes as json.dumps(record_dict(rec)), without the objects
            h = records._high
            sink.writelines(f'{{"arg_bits": "{hex(h | i)}", "distance_num": {d}, "distance_den_log2": 64, '
                            f'"domain": {m}}}\n' for i, d, m in zip(records.index.tolist(), records.dist.tolist(),
                                                                     records.dom.tolist()))
            return
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


class RecordSet(Sequence):
    """HR records (or candidates) of one binade as numpy columns: argument
    index within the binade, distance raw (2^-64 units), domain id,
    undecided flag.  A Sequence of HrCaseRecord (built on access), so it
    compares, iterates and indexes like the reference's lists while a
    2^36-argument range at a loose eps (millions of records) stays arrays.
    float_bits of an argument = ((binade + 1 + 2^15) << (p - 1)) | index
    (fpmodel.py:126-137)."""

    def __init__(self, precision: int, binade: int, index, dist, dom, undecided=None):
        self.precision, self.binade = precision, binade
        self.index = np.asarray(index, dtype=np.uint64)
        self.dist = np.asarray(dist, dtype=np.uint64)
        self.dom = np.asarray(dom, dtype=np.uint64)
        self.undecided = (np.zeros(len(self.index), dtype=bool) if undecided is None
                          else np.asarray(undecided, dtype=bool))

    @property
    def _high(self) -> int:
        return (self.binade + 1 + EXP_BIAS) << (self.precision - 1)

    def __len__(self) -> int:
        return len(self.index)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return RecordSet(self.precision, self.binade, self.index[k], self.dist[k], self.dom[k], self.undecided[k])
        return HrCaseRecord(self._high | int(self.index[k]), UFrac(int(self.dist[k]), 64), int(self.dom[k]),
                            bool(self.undecided[k]))

    def __iter__(self):
        h = self._high
        for i, d, m, u in zip(self.index.tolist(), self.dist.tolist(), self.dom.tolist(), self.undecided.tolist()):
            yield HrCaseRecord(h | i, UFrac(d, 64), m, u)

    def __eq__(self, other) -> bool:
        if isinstance(other, RecordSet):
            if len(self) != len(other):
                return False
            if (self.precision, self.binade) == (other.precision, other.binade):
                return bool(np.array_equal(self.index, other.index) and np.array_equal(self.dist, other.dist)
                            and np.array_equal(self.dom, other.dom)
                            and np.array_equal(self.undecided, other.undecided))
        try:
            return list(self) == list(other)
        except TypeError:
            return NotImplemented

    __hash__ = None

    def __repr__(self) -> str:
        return f"RecordSet({len(self)} records, p={self.precision}, binade={self.binade})"

    @staticmethod
    def of(records, precision: int, binade: int) -> "RecordSet":
        """Columns of HrCaseRecord objects of one binade."""
        recs = list(records)
        mask = (1 << (precision - 1)) - 1
        return RecordSet(precision, binade, [r.argument & mask for r in recs], [r.distance.raw for r in recs],
                         [r.domain_id for r in recs], [r.undecided for r in recs])

    @staticmethod
    def concat(sets, precision: int, binade: int) -> "RecordSet":
        sets = [s if isinstance(s, RecordSet) else RecordSet.of(s, precision, binade) for s in sets]
        if not sets:
            return RecordSet(precision, binade, [], [], [])
        return RecordSet(precision, binade, np.concatenate([s.index for s in sets]),
                         np.concatenate([s.dist for s in sets]), np.concatenate([s.dom for s in sets]),
                         np.concatenate([s.undecided for s in sets]))

    def merged(self, other: "RecordSet") -> "RecordSet":
        """The union of two argument-sorted sets with distinct arguments, in
        argument order: the few records another path decided are inserted
        by position instead of re-sorting millions."""
        if not len(other):
            return self
        pos = np.searchsorted(self.index, other.index)
        ins = lambda a, b: np.insert(a, pos, b)  # noqa: E731
        return RecordSet(self.precision, self.binade, ins(self.index, other.index), ins(self.dist, other.dist),
                         ins(self.dom, other.dom), ins(self.undecided, other.undecided))

    def sorted(self) -> "RecordSet":
        """Ascending by argument (then distance, domain: HrCaseRecord order)."""
        if len(self.index) < 2 or bool(np.all(self.index[1:] > self.index[:-1])):
            return self  # already strictly ascending by argument (the usual case)
        order = np.lexsort((self.undecided, self.dom, self.dist, self.index))
        return RecordSet(self.precision, self.binade, self.index[order], self.dist[order], self.dom[order],
                         self.undecided[order])
