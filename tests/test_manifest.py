"""Resumable range manifest (funnel.run_range(manifest=...)): the line
format round-trips, a manifest of another run is refused, a torn last line
is ignored; on the GPU a resumed run equals an uninterrupted one."""
import json

import pytest

from golden_io import case, config_of

from paper_1211_3056_b200.arith import UFrac
from paper_1211_3056_b200.fpformat import HrCaseRecord
from paper_1211_3056_b200.funnel import PhaseRow, PhaseStats, interval_line, manifest_key, read_manifest


def _stats():
    return PhaseStats([PhaseRow("phase1", 10, 3, 320, 1.5), PhaseRow("confirm", 2, 1, 2, 0.25)], [(0, "regular")])


def test_lines_round_trip(tmp_path):
    cfg = config_of(case("p13_cli_default"))
    key = manifest_key("exp", 0, 0, 4096, cfg, 1024)
    recs = [HrCaseRecord(0x8001046, UFrac(24674833356615680, 64), 4), HrCaseRecord(0x10, UFrac(5, 64), 1, True)]
    p = tmp_path / "m.jsonl"
    p.write_text(json.dumps({"kind": "header", "key": key}) + "\n" + interval_line(0, 0, "regular", recs, _stats())
                 + "\n" + interval_line(1, 1024, "lefevre", [], _stats())[:40] + "\n")  # torn last line
    done = read_manifest(str(p), key)
    assert list(done) == [0]
    bstart, algo, r, st = done[0]
    assert (bstart, algo) == (0, "regular") and r == recs
    assert st.rows == _stats().rows and st.algorithm_choices == [(0, "regular")]
    with pytest.raises(ValueError):
        read_manifest(str(p), manifest_key("exp", 0, 0, 8192, cfg, 1024))
    assert read_manifest(str(tmp_path / "absent.jsonl"), key) == {}


@pytest.mark.gpu
def test_resumed_range_equals_uninterrupted(tmp_path):
    from paper_1211_3056_b200.funnel import run_range

    c = case("p13_cli_default")
    cfg = config_of(c)
    whole = run_range("exp", 0, 0, 1 << 12, cfg, interval_args=1 << 10, workers=1)
    p = tmp_path / "m.jsonl"
    first = run_range("exp", 0, 0, 1 << 12, cfg, interval_args=1 << 10, workers=1, manifest=str(p))
    lines = p.read_text().splitlines()
    assert len(lines) == 1 + len(whole.interval_stats) > 2
    p.write_text("\n".join(lines[:2]) + "\n" + lines[2][:25])  # crash after interval 0, mid-line
    resumed = run_range("exp", 0, 0, 1 << 12, cfg, interval_args=1 << 10, workers=1, manifest=str(p))
    for out in (first, resumed):
        assert out.records == whole.records
        assert out.choices == whole.choices
        assert [[(r.phase, r.domains_in, r.domains_out, r.arguments_covered) for r in st.rows]
                for st in out.interval_stats] == [[(r.phase, r.domains_in, r.domains_out, r.arguments_covered)
                                                   for r in st.rows] for st in whole.interval_stats]


def test_torn_header_starts_over(tmp_path):
    """A crash that tore the header line leaves no finished interval, and
    the key ignores the host worker count but not the results' config."""
    import dataclasses

    from paper_1211_3056_b200.funnel import _manifest_has_header

    cfg = config_of(case("p13_cli_default"))
    key = manifest_key("exp", 0, 0, 4096, cfg, 1024)
    p = tmp_path / "m.jsonl"
    p.write_text(json.dumps({"kind": "header", "key": key})[:17])
    assert not _manifest_has_header(str(p))
    assert read_manifest(str(p), key) == {}
    wide = dataclasses.replace(cfg, phase=dataclasses.replace(cfg.phase, parallel_width=7))
    assert manifest_key("exp", 0, 0, 4096, wide, 1024) == key
    other = dataclasses.replace(cfg, phase=dataclasses.replace(cfg.phase, phase2_split=16))
    assert manifest_key("exp", 0, 0, 4096, other, 1024) != key


def test_enclose_is_thread_safe():
    """mpmath's interval precision is process-global: enclosures computed
    from two threads at different precisions equal single-threaded ones."""
    import threading
    from fractions import Fraction

    from paper_1211_3056_b200 import enclosure

    xs = [Fraction((1 << 52) + 7919 * k, 1 << 52) for k in range(1, 400)]
    want = {}
    for prec in (160, 400):
        for x in xs:
            want[(x, prec)] = enclosure._enclose_locked("exp", x, max(prec, 53) + 8)
    enclosure.enclose.cache_clear()
    got, errs = {}, []

    def work(prec):
        try:
            for x in xs:
                got[(x, prec)] = enclosure.enclose("exp", x, prec)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    import sys

    old = sys.getswitchinterval()
    sys.setswitchinterval(1e-6)
    try:
        ts = [threading.Thread(target=work, args=(p,)) for p in (160, 400)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        sys.setswitchinterval(old)
        enclosure.enclose.cache_clear()
    assert not errs and got == want


@pytest.mark.gpu
def test_run_range_threads_equal_run_slice():
    """run_range builds interval i+1 in a thread while interval i confirms
    (both call enclose): the records must equal one run_slice's."""
    from paper_1211_3056_b200.funnel import run_range, run_slice

    c = case("p13_cli_default")
    cfg = config_of(c)
    whole = run_slice("exp", 0, 0, 1 << 12, cfg, workers=1)
    ranged = run_range("exp", 0, 0, 1 << 12, cfg, interval_args=1 << 9, workers=1)
    assert ranged.records == whole.records
    # the host-buffer call's device-side statistics equal the per-phase path's
    for phase in ("phase1", "phase2", "phase3", "confirm"):
        want = whole.stats.row(phase)
        got = [st.row(phase) for st in ranged.interval_stats]
        assert sum(r.domains_in for r in got) == want.domains_in, phase
        assert sum(r.domains_out for r in got) == want.domains_out, phase
        assert sum(r.arguments_covered for r in got) == want.arguments_covered, phase
