"""Divergence measurement against the reference's own simulate_warps reports
(tests/golden/make_divergence.py).  CPU tests: the problem generator and
the per-warp statistics; GPU tests: the device traces and iteration counts."""

import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_1211_3056_b200.arith import DivisionMode
from paper_1211_3056_b200.divergence import (BRANCH_WEIGHTS, _serialized, linear_problem_batch, mdm, nmdm,
                                             warp_summary)
from paper_1211_3056_b200.fpformat import FpFormat
from paper_1211_3056_b200.search import Algorithm

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "divergence.json")) as fh:
    CASES = {c["name"]: c for c in json.load(fh)}


def F(x):
    return Fraction(int(x[0]), int(x[1]))


def paths_of(run):
    return [[bool((int(h, 16) >> k) & 1) for k in range(n)] for *_, n, h in run["lanes"]]


@pytest.mark.parametrize("name", ["exp_p33_512x1024", "exp_p53_2p15x512"])
def test_linear_problem_batch_matches_reference(name):
    c = CASES[name]
    got = linear_problem_batch("exp", FpFormat(c["p"], c["eps_bits"]), 0, c["domain_size"], c["domain_count"])
    assert [[p.a.raw, p.b.raw, p.eps.raw, p.count] for p in got] == c["problems"]


@pytest.mark.parametrize("name", list(CASES))
def test_warp_statistics_match_reference(name):
    c = CASES[name]
    ww = c["warp_width"]
    for run in c["runs"]:
        its = [lane[2] for lane in run["lanes"]]
        paths = paths_of(run)
        w = BRANCH_WEIGHTS[Algorithm(run["algo"])]
        for k, want in enumerate(run["warps"]):
            lanes = its[k * ww:(k + 1) * ww]
            assert mdm(lanes) == F(want[0]) and nmdm(lanes) == F(want[1]), (name, run["algo"], k)
            assert max(lanes) == want[2]
            assert _serialized(paths[k * ww:(k + 1) * ww], w) == want[3], (name, run["algo"], k)


def test_nmdm_examples():
    assert mdm([10, 20, 30, 40]) == 15 and nmdm([10, 20, 30, 40]) == Fraction(3, 8)
    assert nmdm([0, 0]) == 0 and mdm([5] * 32) == 0
    with pytest.raises(ValueError):
        nmdm([])
    s = warp_summary(np.array([10, 20, 30, 40] * 8, dtype=np.uint64))
    assert abs(s.mean_nmdm - 0.375) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_simulate_warps_equals_reference(name):
    from paper_1211_3056_b200.arith import UFrac
    from paper_1211_3056_b200.divergence import simulate_warps
    from paper_1211_3056_b200.search import SearchProblem

    c = CASES[name]
    probs = [SearchProblem(UFrac(a, 64), UFrac(b, 64), UFrac(e, 64), n) for a, b, e, n in c["problems"]]
    for run in c["runs"]:
        rep = simulate_warps(probs, run["algo"], DivisionMode[run["mode"]], c["warp_width"])
        lanes = [[int(o.success), o.d.raw, it, o.points_placed, len(p)]
                 for t in rep.traces for it, p, o in zip(t.lane_iterations, t.branch_paths, t.outcomes)]
        assert lanes == [l[:5] for l in run["lanes"]], (name, run["algo"], run["mode"])
        got_paths = [list(p) for t in rep.traces for p in t.branch_paths]
        assert got_paths == paths_of(run), (name, run["algo"], run["mode"])
        assert [[s.mdm, s.nmdm, s.serialized_iterations, s.branch_serialized_instructions] for s in rep.warps] == \
            [[F(w[0]), F(w[1]), w[2], w[3]] for w in run["warps"]]
        assert (rep.min_iterations, rep.max_iterations) == (run["min"], run["max"])
        assert rep.mean_iterations == F(run["mean"]) and rep.mean_nmdm == F(run["mean_nmdm"])


@pytest.mark.gpu
def test_search_callables_fill_trace_like_the_reference():
    from paper_1211_3056_b200.arith import UFrac
    from paper_1211_3056_b200.search import SEARCHES, SearchProblem

    c = CASES["exp_p33_w8"]
    for run in c["runs"]:
        for (a, b, e, n), lane in list(zip(c["problems"], run["lanes"]))[:16]:
            tr = []
            out = SEARCHES[Algorithm(run["algo"])](SearchProblem(UFrac(a, 64), UFrac(b, 64), UFrac(e, 64), n),
                                                   mode=DivisionMode[run["mode"]], trace=tr)
            assert (int(out.success), out.d.raw, out.iterations, out.points_placed) == tuple(lane[:4])
            assert tr == [bool((int(lane[5], 16) >> k) & 1) for k in range(lane[4])]
