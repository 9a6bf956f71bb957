"""Native host generation and confirmation (libhrbhost.so, hostgen.py).

Pins, in order of strength:
- the reference's own fixtures (tests/golden/pipeline_cases.json, written by
  make_golden.py from /root/reference): for every exp case the native packed
  slice equals the packing of the super-domains the REFERENCE computed
  (taylor_approx + hierarchical_split: r_polys and eps'), and the native
  confirmation of the reference's phase-3 candidates yields exactly the
  reference's records;
- mpmath itself: the restated interval exp equals iv.exp endpoint for
  endpoint, and native decisions equal decide_hr's, on random arguments;
- the Python host path (slices.pack_plan(native=False)) on random
  configurations.
"""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from golden_io import batch_of, case, config_of, pipeline_cases

from paper_1211_3056_b200 import hostgen, slices
from paper_1211_3056_b200.enclosure import _enclose_locked, decide_hr
from paper_1211_3056_b200.fpformat import FpFormat, HrCaseRecord, bits_float
from paper_1211_3056_b200.arith import UFrac
from paper_1211_3056_b200.funnel import _confirm_chunk, confirm_candidates
from paper_1211_3056_b200.taylor import PolyGenConfig

PACKED = ("coef", "G", "s2abs", "n_dom", "dom_n", "last_n", "dom_base", "m0")


def _native_cases():
    return [c["name"] for c in pipeline_cases() if c["fn"] == "exp" and c["binade"] <= 0]


@pytest.mark.parametrize("name", _native_cases())
def test_native_pack_equals_reference_fixture(name):
    c = case(name)
    cfg = config_of(c)
    want = batch_of(c)  # the reference's super-domains, packed
    start, count = c["slice"]
    plan = slices.plan_arrays(c["fn"], c["binade"], cfg.fmt, cfg.polygen, start, count)
    got = slices.pack_plan(plan, cfg.word_bits, workers=2, native=True)
    assert [int(x) for x in plan.bstart] == [s["index_start"] for s in c["supers"]]
    assert [int(x) for x in plan.dom_id0] == [s["dom_id0"] for s in c["supers"]]
    for k in PACKED:
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert np.array_equal(got.shift_bound_ok, want.shift_bound_ok)
    # the lazily rebuilt super-domains carry the reference's r_polys
    for g, w in zip(got.supers, want.supers):
        assert [[int(x) for x in rp.coeffs] for rp in g.r_polys] == \
            [[x.to_int() if hasattr(x, "to_int") else int(x) for x in rp.coeffs] for rp in w.r_polys]


@pytest.mark.parametrize("name", _native_cases())
def test_native_confirm_equals_reference_records(name):
    c = case(name)
    cfg = config_of(c)
    cands = [HrCaseRecord(int(a, 16), UFrac(d, 64), dom) for a, d, dom in c["phase3"]]
    recs = confirm_candidates(c["fn"], cands, cfg.fmt, workers=2, native=True)
    assert [[hex(r.argument), r.distance.raw, r.domain_id, r.undecided] for r in recs] == c["records"]


def test_exp_enclosure_equals_mpmath():
    rng = random.Random(7)
    for _ in range(4000):
        p = rng.choice([53, 53, 24, 13, 64])
        b = rng.choice([0, 0, -1, -5])
        M = (1 << (p - 1)) + rng.getrandbits(p - 1)
        xe = b + 1 - p
        prec = rng.choice([96, 128, 160, 186, 200, 372])
        x = Fraction(M) * Fraction(2) ** xe
        want = _enclose_locked("exp", x, max(prec, x.numerator.bit_length(), x.denominator.bit_length()) + 8)
        assert hostgen.exp_enclose(M, xe, prec) == want, (M, xe, prec)


def test_native_confirm_equals_decide_hr():
    """Random arguments plus arguments whose exp lies close to a p-bit
    rounding boundary (both verdicts, and more than one precision step)."""
    rng = random.Random(11)
    for p, eps_bits, b in ((53, 16, 0), (53, 32, 0), (24, 12, -1), (13, 6, 0)):
        fmt = FpFormat(p, eps_bits)
        idx = [rng.getrandbits(p - 1) for _ in range(600)]
        cfg = hostgen.make_cfg("exp", fmt, PolyGenConfig(), b, 64)
        is_hr, dist, status = hostgen.confirm(cfg, np.array(idx, dtype=np.uint64), 2)
        assert (status == 0).all()
        for i, h, d in zip(idx, is_hr.tolist(), dist.tolist()):
            arg = ((b + 1 + (1 << 15)) << (p - 1)) | i
            dec = decide_hr("exp", bits_float(arg, fmt), fmt, start_prec=2 * (p + eps_bits) + 16)
            assert bool(h) == dec.is_hr
            if h:
                assert d == UFrac.from_fraction(dec.distance_lo).raw
        assert is_hr.any() or eps_bits > 8


def test_native_pack_equals_python_random():
    rng = random.Random(3)
    for _ in range(6):
        p = rng.choice([53, 53, 40])
        fmt = FpFormat(p, rng.choice([16, 20, 32]))
        N = 1 << rng.choice([6, 10, 12, 15])
        mu = 1 << rng.choice([0, 1, 2])
        nu = 1 << rng.choice([1, 2, 3])
        pg = PolyGenConfig(tau=mu * nu, N=N, mu=mu, nu=nu, delta=rng.choice([1, 2]), limbs=rng.choice([6, 8]),
                           frac_bits=rng.choice([64, 96, 128]), guard=rng.choice([16, 32]))
        start = rng.getrandbits(p - 8)
        count = rng.randrange(1, 40) * pg.tau * N + rng.randrange(0, N)
        plan = slices.plan_arrays("exp", 0, fmt, pg, start, count)
        try:
            want = slices.pack_plan(plan, 64, workers=1, native=False)
        except (ValueError, ArithmeticError) as e:
            with pytest.raises(type(e)):
                slices.pack_plan(plan, 64, workers=2, native=True)
            continue
        got = slices.pack_plan(plan, 64, workers=2, native=True)
        for k in PACKED:
            assert np.array_equal(getattr(got, k), getattr(want, k)), k
        assert np.array_equal(got.shift_bound_ok, want.shift_bound_ok)


def test_fallback_raises_like_the_reference():
    """A block the reference rejects (eps'' >= 1/4 at a tiny precision) is
    flagged by the native generator and raised by the exact Python path."""
    fmt = FpFormat(13, 2)
    pg = PolyGenConfig(tau=16, N=1 << 6, mu=4, nu=4, delta=2, limbs=8, frac_bits=96, guard=32)
    plan = slices.plan_arrays("exp", 0, fmt, pg, 0, 1 << 12)
    with pytest.raises(ValueError):
        slices.pack_plan(plan, 64, workers=1, native=False)
    with pytest.raises(ValueError):
        slices.pack_plan(plan, 64, workers=1, native=True)


def _overflow_cases():
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "overflow.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("native", [False, True])
def test_limb_overflow_matches_reference(native):
    """Where the reference's host generation raises MPOverflowError under a
    tight limb budget (tests/golden/make_overflow.py: MPInt.from_int in
    taylor_approx, MPInt products in hierarchical_split), this package's
    planning + packing raises the same class with the same message, on
    both the Python and the native path; where the reference succeeds, so
    does this package, with the same number of domains."""
    from paper_1211_3056_b200.arith import MPOverflowError

    for c in _overflow_cases():
        fmt = FpFormat(c["p"], c["eps_bits"])
        pg = PolyGenConfig(tau=c["tau"], N=c["N"], mu=c["mu"], nu=c["nu"], delta=2, limbs=c["limbs"],
                           frac_bits=c["frac_bits"], guard=32)
        plan = slices.plan_arrays(c["fn"], c["binade"], fmt, pg, 0, 1 << (c["p"] - 1))
        if c["ok"]:
            b = slices.pack_plan(plan, 64 if c["frac_bits"] >= 64 else 32, workers=1, native=native)
            assert b.n_total == c["tasks"], c
        else:
            assert c["error"] == "MPOverflowError"
            with pytest.raises(MPOverflowError) as ei:
                slices.pack_plan(plan, 64 if c["frac_bits"] >= 64 else 32, workers=1, native=native)
            assert str(ei.value) == c["message"], c
