"""High-degree (delta_R >= 3) path: host models, device walk, phases,
records.

Parity chain (the reference rejects delta >= 3, polygen.py:81-82, so the
tabulated values and phase flags are PARITY UNPINNED against it):
- native host models == the specification oracle/wide.py (exact ints);
- device tabulated values (multi-limb packet walk) == the specification's
  r_j(i), for every domain;
- device phases 1-3 (failing ids, subdomain keys, candidates) == the
  specification's exact pipeline (Python ints + the C oracle's search);
- confirmed records == the REFERENCE's exhaustive_hr_search
  (tests/golden/exhaustive.json, oracle.py:77-113) and == the delta = 2
  pipeline's records.
"""
import json
import os
import random

import numpy as np
import pytest

import oracle.wide as spec
from paper_1211_3056_b200 import hostgen
from paper_1211_3056_b200.fpformat import FpFormat
from paper_1211_3056_b200.taylor import PolyGenConfig
from paper_1211_3056_b200.wide import WideGenConfig, plan_wide, prepare_wide

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _limbs(v: int, nl: int) -> list:
    v %= 1 << (32 * nl)
    return [(v >> (32 * k)) & 0xFFFFFFFF for k in range(nl)]


def _models(batch, plan):
    fmt, w = batch.fmt, batch.wcfg
    return [spec.wide_model("exp", fmt.precision, fmt.eps_bits, batch.binade, int(plan.bstart[t]),
                            int(plan.bcount[t]), int(plan.n_p[t]), int(plan.tau[t]), int(plan.e_out[t]), w.delta,
                            w.frac_limbs, w.guard) for t in range(len(plan))]


@pytest.mark.parametrize("delta", [3, 4, 5, 6, 7, 8])
def test_native_models_equal_specification(delta):
    rng = random.Random(delta)
    for _ in range(3):
        fmt = FpFormat(53, rng.choice([16, 24, 32]))
        w = WideGenConfig(delta, tau=1 << rng.randrange(4, 12), N=1 << rng.choice([10, 12, 15]))
        start = rng.getrandbits(50)
        plan = plan_wide("exp", 0, fmt, w, start, w.tau * w.N * 2 + rng.randrange(1, w.N * 3))
        batch = prepare_wide("exp", 0, start, int(plan.bcount.sum()), fmt, w, workers=2)
        for t, m in enumerate(_models(batch, plan)):
            want = [_limbs(x, w.frac_limbs) for r in m.q for x in r]
            assert batch.coef[:, :, t].tolist() == want
            assert int(batch.padg[0, t]) | (int(batch.padg[1, t]) << 64) == m.padg
            assert int(batch.s2b[0, t]) | (int(batch.s2b[1, t]) << 64) == m.s2b
            assert batch.win[:, t].tolist() == _limbs(m.win, w.frac_limbs)


def test_wide_budget_out_of_range_raises():
    # a degree-3 model over 2^43 arguments blows the budget (Lagrange term)
    with pytest.raises(ValueError):
        prepare_wide("exp", 0, 0, 1 << 43, FpFormat(53, 32), WideGenConfig(3, tau=1 << 28, N=1 << 15))


def test_wide_config_validation():
    with pytest.raises(ValueError):
        WideGenConfig(2)
    with pytest.raises(ValueError):
        WideGenConfig(9)
    assert WideGenConfig.for_degree(6).tau * (1 << 15) == 1 << 40


# ------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [3, 4, 5, 6, 7, 8])
def test_wide_tabulated_values_equal_specification(delta):
    from paper_1211_3056_b200.wide import wide_domain_coefficients

    fmt = FpFormat(53, 32)
    w = WideGenConfig(delta, tau=1 << 9, N=1 << 12)
    start = 0x123456789AB
    count = 3 * w.tau * w.N + 5 * w.N + 77  # 4 super-domains, ragged tail
    plan = plan_wide("exp", 0, fmt, w, start, count)
    batch = prepare_wide("exp", 0, start, count, fmt, w, workers=2)
    got = wide_domain_coefficients(batch)
    models = _models(batch, plan)
    for t, m in enumerate(models):
        d0 = int(batch.dom_base[t])
        for i in list(range(0, int(plan.tau[t]), 37)) + [int(plan.tau[t]) - 1]:
            for j in range(delta + 1):
                assert got[j, :, d0 + i].tolist() == _limbs(spec.r_tilde(m.q, j, i), w.frac_limbs), (t, i, j)


def _run_device(batch, split=8):
    from paper_1211_3056_b200.wide import WideDeviceSlice, WideRunner

    runner = WideRunner(WideDeviceSlice(batch), 2, split, sub_cap=batch.n_total * 2 * split, cand_cap=1 << 16)
    runner.launch()
    import torch

    torch.cuda.synchronize()
    return runner.result()


@pytest.mark.gpu
@pytest.mark.parametrize("delta,eps_bits,lgN", [(3, 16, 15), (4, 16, 15), (6, 20, 12), (8, 16, 12), (5, 12, 10)])
def test_wide_phases_equal_specification(delta, eps_bits, lgN):
    fmt = FpFormat(53, eps_bits)
    w = WideGenConfig(delta, tau=8, N=1 << lgN)
    start, count = 0x2000000000, (1 << 20) + 1234
    plan = plan_wide("exp", 0, fmt, w, start, count)
    batch = prepare_wide("exp", 0, start, count, fmt, w, workers=2)
    models = _models(batch, plan)
    geom = [(int(plan.bstart[t]), int(plan.bcount[t]), int(plan.n_p[t]), int(plan.tau[t]), int(plan.dom_id0[t]))
            for t in range(len(plan))]
    fails, subs, cands = spec.pipeline(models, geom, fmt.precision, 0, w.frac_limbs)
    c, fail_ids, sub_keys, cm, cd, cdom = _run_device(batch)
    assert (fail_ids + np.uint64(batch.id0)).tolist() == fails
    assert [(int(k >> np.uint64(8)) + batch.id0, int(k & np.uint64(255))) for k in sub_keys] == \
        [(s[0], s[1]) for s in subs]
    assert list(zip(cm.tolist(), cd.tolist(), (cdom + np.uint64(batch.id0)).tolist())) == cands
    assert int(c[0]) == len(fails) and int(c[2]) == len(cands)


def _records_wide(fn, binade, start, count, fmt, w):
    from paper_1211_3056_b200.funnel import confirm_candidates
    from paper_1211_3056_b200.wide import candidates_of, run_wide_host

    batch = prepare_wide(fn, binade, start, count, fmt, w, workers=2)
    res = run_wide_host(batch)
    return confirm_candidates(fn, candidates_of(batch, res), fmt, workers=2), res


@pytest.mark.gpu
@pytest.mark.parametrize("delta", [3, 4, 6, 8])
def test_wide_records_equal_reference_exhaustive(delta):
    """The reference's exhaustive enumerator (every argument decided
    directly, tests/golden/make_exhaustive.py) is the end-result pin."""
    with open(os.path.join(GOLDEN, "exhaustive.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        fmt = FpFormat(c["p"], c["eps_bits"])
        w = WideGenConfig(delta, tau=8, N=1 << 15)
        recs, _ = _records_wide(c["fn"], c["binade"], c["start"], c["count"], fmt, w)
        assert [[hex(r.argument), r.distance.raw, r.undecided] for r in recs] == c["records"], c["name"]


@pytest.mark.gpu
def test_wide_records_equal_delta2_large():
    """2^34 arguments: delta_R = 4 (one model per 2^30 arguments) and 6
    (one model for the whole range) give the delta = 2 records exactly."""
    from paper_1211_3056_b200 import PhaseConfig, PipelineConfig
    from paper_1211_3056_b200.funnel import run_range

    fmt = FpFormat(53, 24)
    start, count = 0x80000000000, 1 << 34
    pg = PolyGenConfig(tau=512, N=1 << 15, mu=16, nu=32, delta=2, limbs=8, frac_bits=96, guard=32)
    cfg = PipelineConfig("exp", fmt, pg, PhaseConfig("regular", phase2_split=8, N1=1 << 15))
    want = run_range("exp", 0, start, count, cfg, interval_args=1 << 34, workers=4).records
    assert len(want) > 100
    for w in (WideGenConfig(4, tau=1 << 15, N=1 << 15), WideGenConfig(6, tau=1 << 19, N=1 << 15)):
        recs, res = _records_wide("exp", 0, start, count, fmt, w)
        assert [(r.argument, r.distance.raw, r.domain_id) for r in recs] == \
            [(r.argument, r.distance.raw, r.domain_id) for r in want]
