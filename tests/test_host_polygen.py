"""Host polynomial generation (this package's restatement, mpmath) gives the
reference's super-domain schedule, Taylor coefficients, hierarchical split
and eps' budgets exactly (tests/golden fixtures).  CPU-only."""

from fractions import Fraction

import pytest

from golden_io import case, config_of
from paper_1211_3056_b200.arith import as_int
from paper_1211_3056_b200.slices import build_super_domains


@pytest.mark.parametrize("name", ["p13_exp_b0", "p13_log_b0", "p13_exp2_b1", "p13_exp_b-1",
                                  "p53_exp_2p20_e16_N15", "p53_exp_ragged", "p53_log_sqrt2_e16", "p53_exp_delta1",
                                  "p53_exp_F128", "p53_exp_F64", "p53_exp2_e16"])
def test_super_domains_match_reference(name):
    c = case(name)
    cfg = config_of(c)
    lo, cnt = c["slice"]
    supers = build_super_domains(c["fn"], c["binade"], cfg.fmt, cfg.polygen, lo, cnt)
    assert len(supers) == len(c["supers"])
    for got, want in zip(supers, c["supers"]):
        assert (got.index_start, got.count, got.n_p, got.tau, got.mu, got.nu, got.e_out, got.dom_id0) == (
            want["index_start"], want["count"], want["n_p"], want["tau"], want["mu"], want["nu"], want["e_out"],
            want["dom_id0"])
        assert [[hex(as_int(x)) for x in rp.coeffs] for rp in got.r_polys] == want["r_polys"]
        assert got.eps_prime == Fraction(int(want["eps_prime"][0]), int(want["eps_prime"][1]))


def test_parallel_generation_is_identical():
    c = case("p53_exp_2p20_e16_N12")
    cfg = config_of(c)
    lo, cnt = c["slice"]
    a = build_super_domains(c["fn"], c["binade"], cfg.fmt, cfg.polygen, lo, cnt, workers=1)
    b = build_super_domains(c["fn"], c["binade"], cfg.fmt, cfg.polygen, lo, cnt, workers=4)
    assert a == b


@pytest.mark.parametrize("workers", [1, 3])
def test_confirmation_matches_reference_records(workers, monkeypatch):
    """Host confirmation (decide_hr per phase-3 candidate, pipeline.py:447-462),
    serial and spread over processes, gives the reference's records."""
    from golden_io import essence
    from paper_1211_3056_b200 import funnel
    from paper_1211_3056_b200.arith import UFrac
    from paper_1211_3056_b200.fpformat import HrCaseRecord

    monkeypatch.setattr(funnel, "CONFIRM_CHUNK", 4)
    for name in ("p53_exp_2p20_e16_N12", "p53_log_sqrt2_e16", "p13_exp_b0"):
        c = case(name)
        cfg = config_of(c)
        cand = [HrCaseRecord(int(h, 16), UFrac(d, 64), i) for h, d, i in c["phase3"]]
        recs = funnel.confirm_candidates(c["fn"], cand, cfg.fmt, workers)
        assert essence(recs) == c["records"], name


def test_parallel_packing_is_identical(monkeypatch):
    """pack_slice over forked workers equals the sequential packing, column
    for column, and a failing host check still raises."""
    import numpy as np

    from paper_1211_3056_b200 import slices
    from paper_1211_3056_b200.slices import pack_slice

    monkeypatch.setattr(slices, "PACK_PARALLEL_MIN", 0)

    c = case("p16_exp_b1")  # 131 super-domains
    cfg = config_of(c)
    sup = build_super_domains(c["fn"], c["binade"], cfg.fmt, cfg.polygen, *c["slice"])
    a = pack_slice(sup, cfg.fmt, cfg.polygen, cfg.word_bits, c["binade"])
    b = pack_slice(sup, cfg.fmt, cfg.polygen, cfg.word_bits, c["binade"], workers=4)
    for k in ("coef", "G", "s2abs", "n_dom", "dom_n", "last_n", "dom_base", "m0", "shift_bound_ok"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k
    with pytest.raises(ValueError):
        pack_slice(sup, cfg.fmt, cfg.polygen, cfg.word_bits, c["binade"], budget_ceiling=Fraction(0), workers=4)
