"""The CPU oracle (oracle/hr_oracle.c) pinned against fixtures produced by
the reference itself (tests/golden/make_golden.py).  CPU-only."""

from fractions import Fraction
import random

import numpy as np
import pytest

import oracle
from golden_io import CORE_COLUMNS, batch_of, case, load_search, pipeline_cases

ONE64 = 1 << 64


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


@pytest.mark.parametrize("fixture,one", [("search_w64.npz", ONE64), ("search_w32.npz", 1 << 32),
                                         ("search_grid1024.npz", 1 << 10)])
def test_cores_match_reference(fixture, one):
    g = load_search(fixture)
    for col, (algo, mode) in enumerate(CORE_COLUMNS):
        ok, d, it, pl, ph = oracle.search_batch(algo, mode, one, g["a"], g["b"], g["eps"], g["count"])
        assert np.array_equal(ok, g["ok"][:, col]), (fixture, algo, mode)
        assert np.array_equal(d, g["d"][:, col]), (fixture, algo, mode)
        assert np.array_equal(it, g["it"][:, col]), (fixture, algo, mode)
        assert np.array_equal(pl, g["pts_lo"][:, col]), (fixture, algo, mode)
        assert np.array_equal(ph, g["pts_hi"][:, col]), (fixture, algo, mode)


def test_small_moduli_match_reference():
    rows = load_search("search_small_moduli.npz")["rows"]
    ones, a, b, eps, n = (rows[:, k].astype(np.uint64) for k in range(5))
    res = rows[:, 5:].reshape(len(rows), 8, 4)
    for one in np.unique(ones):
        sel = ones == one
        for col, (algo, mode) in enumerate(CORE_COLUMNS):
            ok, d, it, pl, ph = oracle.search_batch(algo, mode, int(one), a[sel], b[sel], eps[sel], n[sel])
            want = res[sel, col]
            assert np.array_equal(ok, want[:, 0].astype(np.uint8)), (one, algo, mode)
            assert np.array_equal(d, want[:, 1].astype(np.uint64)), (one, algo, mode)
            assert np.array_equal(it, want[:, 2].astype(np.uint64)), (one, algo, mode)
            assert np.array_equal(pl, want[:, 3].astype(np.uint64)), (one, algo, mode)


def test_closed_form_pad_equals_fraction_form():
    """pad = ceil((G + |s2|(n-1)^2)/2^(F-W)) + n + 1 vs pipeline.py:165-166."""
    rng = random.Random(7)
    for _ in range(3000):
        F = rng.choice([64, 80, 96, 112, 128])
        W = rng.choice([32, 64])
        if W > F:
            continue
        eps_p = Fraction(rng.randrange(1, 1 << 60), rng.randrange(1, 1 << 62) * 3) / (1 << rng.randrange(8, 40))
        if eps_p >= Fraction(1, 8):
            continue
        n = rng.choice([1, 2, 3, 64, 1 << 12, 1 << 15])
        s2 = rng.randrange(0, 1 << max(1, F - 36)) * rng.choice([-1, 1])
        e_dp = eps_p + Fraction(abs(s2) * (n - 1) ** 2, 1 << F)
        if e_dp >= Fraction(1, 4):
            continue
        pad = -((-e_dp.numerator << W) // e_dp.denominator) + n + 1
        if 2 * pad >= 1 << (W - 1):
            continue
        s0 = rng.randrange(-(1 << 150), 1 << 150)
        s1 = rng.randrange(-(1 << 100), 1 << 100)
        one_f = 1 << F
        want_b = ((((s0 % one_f) << W) >> F) + pad) & ((1 << W) - 1)
        want_a = (((-s1) % one_f) << W) >> F
        G = -((-eps_p.numerator << F) // eps_p.denominator)
        a, b, e = oracle.boolean_problem(s0, s1, G, abs(s2), n, F, W)
        assert (a, b, e) == (want_a, want_b, 2 * pad)


def _rows_of(res):
    oid, oj, ost, ocnt, ores = res
    return [[int(i), int(j), int(s), int(c)] for i, j, s, c in zip(oid, oj, ost, ocnt)]


@pytest.mark.parametrize("name", [c["name"] for c in pipeline_cases()])
def test_oracle_pipeline_matches_reference(name):
    c = case(name)
    batch = batch_of(c)
    algo = c["cfg"]["algorithm"]
    mode = {"sub": 0, "hybrid": 1, "hw": 2}[c["cfg"]["div_mode"]]
    fails, coef = oracle.phase1(batch, algo, mode, with_coeffs=True)
    # tabulated values (domain_coefficient_sets) mod 2^128
    m128 = (1 << 128) - 1
    for k, dom in enumerate(c["domains"]):
        for j, hx in enumerate(dom[3:]):
            want = int(hx, 16) & m128
            got = int(coef[j, 0, k]) | (int(coef[j, 1, k]) << 64)
            assert got == want, (name, k, j)
    assert fails.tolist() == c["phase1_fail"], name
    rows = oracle.phase2(batch, algo, mode, c["cfg"]["split"], fails)
    assert _rows_of(rows) == [r[:4] for r in c["phase2"]], name
    # shifted residues match the reference's shifted coefficients mod 2^128
    for r, want in zip(rows[4], c["phase2"]):
        for l, hx in enumerate(want[4:]):
            assert (int(r[2 * l]) | (int(r[2 * l + 1]) << 64)) == int(hx, 16) & m128
    m, dist, dom = oracle.phase3(batch, rows)
    p = c["p"]
    got = [[hex((((c["binade"] + 1 + (1 << 15)) << (p - 1)) | int(mi))), int(di), int(ii)]
           for mi, di, ii in zip(m, dist, dom)]
    assert got == c["phase3"], name
