"""Host polynomial generation (this package's restatement, mpmath) gives the
reference's super-domain schedule, Taylor coefficients, hierarchical split
and eps' budgets exactly (tests/golden fixtures).  CPU-only."""

from fractions import Fraction

import pytest

from golden_io import case, config_of
from paper_1211_3056_b200.arith import as_int
from paper_1211_3056_b200.slices import build_super_domains


@pytest.mark.parametrize("name", ["p13_exp_b0", "p13_log_b0", "p13_exp2_b1", "p13_exp_b-1",
                                  "p53_exp_2p20_e16_N15", "p53_exp_ragged", "p53_log_sqrt2_e16", "p53_exp_delta1"])
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
