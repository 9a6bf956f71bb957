"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src; that tree does not exist on the GPU box, which
is why its outputs are committed):

    python tests/golden/make_golden.py

Every value below comes from calling the reference's own functions
(lowerbound.py, polygen.py, pipeline.py, evalf.py); nothing here computes an
expected value itself.  The slice composition `_reference_slice` mirrors
pipeline.py:374-409 (_build_tasks) restricted to an argument-index range and
pipeline.py:412-463 (run_pipeline) for the phases and confirmation; with the
slice equal to the whole binade it reproduces run_pipeline exactly (checked
below for every p=13 case).
"""

from __future__ import annotations

import json
import os
import random
import sys
from fractions import Fraction

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hardround.evalf import decide_hr  # noqa: E402
from hardround.fixedpoint import DivisionMode, UFrac  # noqa: E402
from hardround.fpmodel import Domain, FpFormat, HrCaseRecord, bits_float  # noqa: E402
from hardround.lowerbound import (  # noqa: E402
    _lefevre_core,
    _lefevre_swap_core,
    _regular_core,
    _regular_unrolled_core,
)
from hardround.pipeline import (  # noqa: E402
    DomainTask,
    PhaseConfig,
    PipelineConfig,
    _piece_domain_size,
    output_binade_pieces,
    phase1,
    phase2,
    phase3_exhaustive,
    run_pipeline,
)
from hardround.polygen import (  # noqa: E402
    PolyGenConfig,
    domain_coefficient_sets,
    hierarchical_split,
    taylor_approx,
)

HERE = os.path.dirname(os.path.abspath(__file__))
ONE64 = 1 << 64
MODES = {"sub": DivisionMode.SUBTRACTIVE, "hybrid": DivisionMode.HYBRID, "hw": DivisionMode.HARDWARE}
MODE_CODE = (0, 1, 2)  # lowerbound._mode_code order: SUBTRACTIVE, HYBRID, HARDWARE


def _ci(c) -> int:
    return c.to_int() if hasattr(c, "to_int") else int(c)


# ---------------------------------------------------------------- searches


def _run_all_cores(a, b, eps, n, one):
    """(ok, d, it, pts) for lefevre x3 modes, swap x3 modes, regular, unrolled."""
    out = []
    for mode in MODE_CODE:
        out.append(_lefevre_core(a, b, eps, n, one, mode, None))
    for mode in MODE_CODE:
        out.append(_lefevre_swap_core(a, b, eps, n, one, mode, None))
    out.append(_regular_core(a, b, eps, n, one, None))
    out.append(_regular_unrolled_core(a, b, eps, n, one, None))
    return out


def _pack_search(problems, one, path):
    a = np.array([p[0] for p in problems], dtype=np.uint64)
    b = np.array([p[1] for p in problems], dtype=np.uint64)
    e = np.array([p[2] for p in problems], dtype=np.uint64)
    n = np.array([p[3] for p in problems], dtype=np.uint64)
    res = [_run_all_cores(*p, one) for p in problems]
    k = len(res[0])
    ok = np.array([[r[j][0] for j in range(k)] for r in res], dtype=np.uint8)
    d = np.array([[r[j][1] for j in range(k)] for r in res], dtype=np.uint64)
    it = np.array([[r[j][2] for j in range(k)] for r in res], dtype=np.uint64)
    pl = np.array([[r[j][3] & (ONE64 - 1) for j in range(k)] for r in res], dtype=np.uint64)
    ph = np.array([[r[j][3] >> 64 for j in range(k)] for r in res], dtype=np.uint64)
    np.savez_compressed(path, a=a, b=b, eps=e, count=n, ok=ok, d=d, it=it, pts_lo=pl, pts_hi=ph,
                        one_lo=np.uint64(one & (ONE64 - 1)), one_hi=np.uint64(one >> 64))
    print(f"wrote {path}: {len(problems)} problems x {k} core runs")


def search_goldens():
    rng = random.Random(20121113)
    probs = []
    # random full-width problems at the pipeline's typical sizes
    for _ in range(3000):
        probs.append((rng.randrange(ONE64), rng.randrange(ONE64), rng.randrange(1, ONE64 // 4),
                      rng.choice([1, 2, 3, 64, 1 << 12, 1 << 15, rng.randint(1, 1 << 16)])))
    # small eps (phase-1-like) with tiny pads
    for _ in range(1000):
        probs.append((rng.randrange(ONE64), rng.randrange(ONE64), rng.randrange(1, 1 << 34), 1 << 15))
    # heavy-tail classic inputs: a close to 0 or 1 (long runs of plain reductions)
    for _ in range(200):
        a = rng.choice([rng.randrange(1, 1 << 20), ONE64 - rng.randrange(1, 1 << 20)])
        probs.append((a, rng.randrange(ONE64), rng.randrange(1, 1 << 40), rng.choice([1 << 10, 1 << 15])))
    # edge cases: exhaustion, powers of two, a=1, a=2^64-1, boundaries
    edge_a = [0, 1, 2, 3, 1 << 32, 1 << 63, (1 << 63) + 1, ONE64 - 1, ONE64 - 2, ONE64 // 3,
              ONE64 // 4, (ONE64 // 4) * 3, 0x5555555555555555, 12345]
    edge_b = [0, 1, 7, 1 << 62, ONE64 - 1, ONE64 // 4 + ONE64 // 8, 500]
    edge_e = [1, 100, ONE64 // 8, ONE64 // 4, (1 << 63) - 1]
    edge_n = [1, 2, 4, 1 << 10, 1 << 15]
    for a in edge_a:
        for b in edge_b:
            for e in edge_e:
                for n in edge_n:
                    if rng.random() < 0.35:
                        probs.append((a, b, e, n))
    # huge counts on expansions that terminate quickly for every core
    for a in (1 << 63, 3 << 62, ONE64 // 4, (ONE64 // 4) * 3):
        for _ in range(3):
            probs.append((a, rng.randrange(ONE64), rng.randrange(1, 1 << 40), (1 << 64) - 1))
    # pinned examples of test_lowerbound.py:96-130
    probs += [(ONE64 // 4, ONE64 // 4 + ONE64 // 8, ONE64 // 8, 4),
              (ONE64 // 4, ONE64 // 4, ONE64 // 4, 4),
              (12345, 7, 100, 1 << 20), (0, 500, 100, 1 << 10), (0, 50, 100, 1 << 10),
              (123456789, 500, 100, 1)]
    _pack_search(probs, ONE64, os.path.join(HERE, "search_w64.npz"))

    # W = 32 words
    one32 = 1 << 32
    probs32 = [(rng.randrange(one32), rng.randrange(one32), rng.randrange(1, one32 // 4),
                rng.choice([1, 2, 16, 1 << 12, 1 << 15])) for _ in range(1500)]
    probs32 += [(1, 5, 1, 1 << 10), (one32 - 1, 9, 3, 1 << 15), (1 << 31, 1, 1, 8)]
    _pack_search(probs32, one32, os.path.join(HERE, "search_w32.npz"))

    # small odd/even moduli (test_lowerbound.py:213-254): full sweeps for 7, 24, 45
    # and a deterministic 25% sample at 97
    small = []
    for one in (7, 24, 45, 97):
        for a in range(one):
            for b in range(one):
                if one == 97 and (a * 97 + b) % 4:
                    continue
                for eps in sorted({1, one // 6}):
                    if eps >= (one + 1) // 2:
                        continue
                    for n in (1, 2, 3, 7, 16, 33):
                        small.append((one, a, b, eps, n))
    res = [_run_all_cores(a, b, e, n, one) for one, a, b, e, n in small]
    arr = np.array([[*s, *(x for r in rr for x in r)] for s, rr in zip(small, res)], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "search_small_moduli.npz"), rows=arr)
    print(f"wrote search_small_moduli.npz: {len(small)} problems")

    # criterion-2 grid (test_acceptance.py:93-163): reference cores at one=2^10 on a
    # deterministic sample; the full 12.6M sweep is checked against the C port.
    grid = 1 << 10
    g = []
    for _ in range(4000):
        g.append((rng.randrange(grid), rng.randrange(grid), grid >> 6, rng.choice((16, 256, 1024))))
    _pack_search(g, grid, os.path.join(HERE, "search_grid1024.npz"))


# ---------------------------------------------------------------- pipeline


def _reference_slice(fn, binade, cfg, s_lo, s_cnt):
    """pipeline.py:374-409 restricted to argument indices [s_lo, s_lo+s_cnt),
    then pipeline.py:412-463 phases + confirmation.  Returns a JSON-able dict."""
    fmt, pg = cfg.fmt, cfg.polygen
    m_base = 1 << (fmt.precision - 1)
    supers, tasks = [], []
    next_id = 0
    for start, pcount, e_out in output_binade_pieces(fn, binade, fmt):
        lo, hi = max(start, s_lo), min(start + pcount, s_lo + s_cnt)
        if lo >= hi:
            continue
        piece_dom = Domain(m_base + lo, binade + 1, hi - lo, 0)
        n_p = _piece_domain_size(fn, piece_dom, e_out, cfg)
        block = pg.tau * n_p
        for bstart in range(lo, hi, block):
            bcount = min(block, hi - bstart)
            if bcount == block and n_p == pg.N:
                bcfg = pg
            else:
                tau_t = -(-bcount // n_p)
                bcfg = PolyGenConfig(tau=tau_t, N=n_p, mu=1, nu=tau_t, delta=pg.delta,
                                     limbs=pg.limbs, frac_bits=pg.frac_bits, guard=pg.guard)
            super_dom = Domain(m_base + bstart, binade + 1, bcount, next_id)
            r_t, eps_approx = taylor_approx(fn, super_dom, bcfg, fmt)
            eps_prime = fmt.eps + eps_approx
            r_polys = hierarchical_split(r_t, n_p, bcfg.delta)
            supers.append({
                "index_start": bstart, "count": bcount, "n_p": n_p, "tau": bcfg.tau,
                "mu": bcfg.mu, "nu": bcfg.nu, "dom_id0": next_id, "e_out": e_out,
                "r_t": [hex(_ci(c)) for c in r_t.coeffs],
                "r_polys": [[hex(_ci(c)) for c in rp.coeffs] for rp in r_polys],
                "eps_prime": [str(eps_prime.numerator), str(eps_prime.denominator)],
            })
            for i, coeffs in enumerate(domain_coefficient_sets(r_polys, bcfg)):
                dstart = bstart + i * n_p
                dcount = min(n_p, bstart + bcount - dstart)
                if dcount <= 0:
                    break
                dom = Domain(m_base + dstart, binade + 1, dcount, next_id)
                tasks.append(DomainTask(dom, coeffs, pg.frac_bits, eps_prime, e_out))
                next_id += 1
    algo = cfg.phase.algorithm
    by_id = {t.domain.domain_id: t for t in tasks}
    failing_ids = phase1(tasks, cfg, algo)
    subtasks = phase2([by_id[i] for i in failing_ids], cfg, algo)
    candidates = phase3_exhaustive(subtasks, cfg)
    guard = 2 * (fmt.precision + fmt.eps_bits) + 16
    records = []
    for cand in candidates:
        x = bits_float(cand.argument, fmt)
        dec = decide_hr(fn, x, fmt, start_prec=guard)
        if dec.is_hr:
            records.append(HrCaseRecord(cand.argument, UFrac.from_fraction(dec.distance_lo), cand.domain_id))
    records.sort()
    return {
        "supers": supers,
        "domains": [[t.domain.domain_id, t.domain.m_start - m_base, t.domain.count,
                     *[hex(_ci(c)) for c in t.coeffs]] for t in tasks],
        "phase1_fail": failing_ids,
        "phase2": [[s.parent.domain.domain_id, s.sub_index, s.start, s.count,
                    *[hex(_ci(c)) for c in s.coeffs]] for s in subtasks],
        "phase3": [[hex(c.argument), c.distance.raw, c.domain_id] for c in candidates],
        "records": [[hex(r.argument), r.distance.raw, r.domain_id, r.undecided] for r in records],
        "stats": {"phase1": [len(tasks), len(failing_ids), sum(t.domain.count for t in tasks)],
                  "phase2": [len(failing_ids), len(subtasks),
                             sum(by_id[i].domain.count for i in failing_ids)],
                  "phase3": [len(subtasks), len(candidates), sum(s.count for s in subtasks)],
                  "confirm": [len(candidates), len(records)]},
    }


def _cfg(fn, p, eps_bits, tau, N, mu, nu, algorithm="regular", div_mode="hybrid", split=8,
         word_bits=64, delta=2, frac_bits=96):
    pg = PolyGenConfig(tau=tau, N=N, mu=mu, nu=nu, delta=delta, limbs=8, frac_bits=frac_bits, guard=32)
    ph = PhaseConfig(algorithm=algorithm, div_mode=MODES[div_mode], phase2_split=split, N1=N)
    return PipelineConfig(fn=fn, fmt=FpFormat(p, eps_bits), polygen=pg, phase=ph, word_bits=word_bits)


def _case(name, fn, binade, p, eps_bits, tau, N, mu, nu, s_lo, s_cnt, **kw):
    cfg = _cfg(fn, p, eps_bits, tau, N, mu, nu, **kw)
    out = _reference_slice(fn, binade, cfg, s_lo, s_cnt)
    if s_lo == 0 and s_cnt == 1 << (p - 1):
        # whole binade: the composition must equal run_pipeline
        recs, stats = run_pipeline(binade, cfg)
        want = [[hex(r.argument), r.distance.raw, r.domain_id, r.undecided] for r in recs]
        assert want == out["records"], name
        assert [r.domains_out for r in stats.rows] == [out["stats"][k][1] for k in
                                                       ("phase1", "phase2", "phase3", "confirm")], name
    out.update({"name": name, "fn": fn, "binade": binade, "p": p, "eps_bits": eps_bits,
                "slice": [s_lo, s_cnt],
                "cfg": {"tau": tau, "N": N, "mu": mu, "nu": nu, "delta": kw.get("delta", 2),
                        "limbs": 8, "frac_bits": kw.get("frac_bits", 96), "guard": 32,
                        "algorithm": kw.get("algorithm", "regular"),
                        "div_mode": kw.get("div_mode", "hybrid"), "split": kw.get("split", 8),
                        "word_bits": kw.get("word_bits", 64)}})
    print(f"{name}: {len(out['supers'])} supers, {len(out['domains'])} domains, "
          f"p1 {len(out['phase1_fail'])}, p2 {len(out['phase2'])}, p3 {len(out['phase3'])}, "
          f"HR {len(out['records'])}")
    return out


def pipeline_goldens():
    cases = []
    # p=13 whole binades (test_pipeline.py:30-79 configuration)
    for fn, binade in (("exp", 0), ("log", 0), ("exp2", 0), ("exp", -1), ("log", 1), ("exp2", 1)):
        cases.append(_case(f"p13_{fn}_b{binade}", fn, binade, 13, 8, 16, 64, 4, 4, 0, 1 << 12))
    cases.append(_case("p13_exp_b0_lefevre", "exp", 0, 13, 8, 16, 64, 4, 4, 0, 1 << 12, algorithm="lefevre"))
    cases.append(_case("p13_exp_b0_lefevre_sub", "exp", 0, 13, 8, 16, 64, 4, 4, 0, 1 << 12,
                       algorithm="lefevre", div_mode="sub"))
    cases.append(_case("p13_exp_b0_w32", "exp", 0, 13, 8, 16, 64, 4, 4, 0, 1 << 12, word_bits=32))
    # CLI default (cli.py:86-113): N=16, tau=16, mu=4, nu=4
    cases.append(_case("p13_cli_default", "exp", 0, 13, 8, 16, 16, 4, 4, 0, 1 << 12))
    # p=16 (acceptance criterion 1) binade 1
    cases.append(_case("p16_exp_b1", "exp", 1, 16, 8, 16, 64, 4, 4, 0, 1 << 15))
    # binary64 slices: X in [1, 1 + 2^-32)
    cases.append(_case("p53_exp_2p20_e16_N15", "exp", 0, 53, 16, 8, 1 << 15, 2, 4, 0, 1 << 20))
    cases.append(_case("p53_exp_2p20_e16_N15_lef", "exp", 0, 53, 16, 8, 1 << 15, 2, 4, 0, 1 << 20,
                       algorithm="lefevre"))
    cases.append(_case("p53_exp_2p20_e20_N15", "exp", 0, 53, 20, 8, 1 << 15, 2, 4, 0, 1 << 20))
    cases.append(_case("p53_exp_2p20_e16_N12", "exp", 0, 53, 16, 64, 1 << 12, 8, 8, 0, 1 << 20))
    cases.append(_case("p53_exp_2p20_e16_N12_w32", "exp", 0, 53, 16, 64, 1 << 12, 8, 8, 0, 1 << 20,
                       word_bits=32))
    cases.append(_case("p53_exp_delta1", "exp", 0, 53, 16, 2, 1 << 12, 1, 2, 0, 1 << 18, delta=1))
    # an interior slice with a ragged end (partial super-domain and domain)
    cases.append(_case("p53_exp_ragged", "exp", 0, 53, 16, 16, 1 << 12, 4, 4,
                       0x123456789AB, (1 << 18) + 5000))
    # log near sqrt(2)
    cases.append(_case("p53_log_sqrt2_e16", "log", 0, 53, 16, 8, 1 << 15, 2, 4, 0x6A09E667F3BCD, 1 << 20))
    with open(os.path.join(HERE, "pipeline_cases.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print("wrote pipeline_cases.json")


def extra_goldens():
    """Cases appended to pipeline_cases.json: other grid widths F (the
    device's 128-bit phase-3 path runs for F > 96), a wider phase-2 split,
    exp2 and the classic walk's other division modes at binary64."""
    path = os.path.join(HERE, "pipeline_cases.json")
    with open(path) as fh:
        cases = json.load(fh)
    have = {c["name"] for c in cases}
    extra = [
        ("p53_exp_F128", dict(fn="exp", binade=0, p=53, eps_bits=16, tau=64, N=1 << 12, mu=8, nu=8, s_lo=0,
                              s_cnt=1 << 20, frac_bits=128)),
        ("p53_exp_F64", dict(fn="exp", binade=0, p=53, eps_bits=16, tau=64, N=1 << 12, mu=8, nu=8, s_lo=0,
                             s_cnt=1 << 20, frac_bits=64)),
        ("p53_exp_split16", dict(fn="exp", binade=0, p=53, eps_bits=16, tau=8, N=1 << 15, mu=2, nu=4, s_lo=0,
                                 s_cnt=1 << 20, split=16)),
        ("p53_exp2_e16", dict(fn="exp2", binade=0, p=53, eps_bits=16, tau=8, N=1 << 15, mu=2, nu=4, s_lo=0,
                              s_cnt=1 << 20)),
        ("p53_exp_lef_hw", dict(fn="exp", binade=0, p=53, eps_bits=16, tau=64, N=1 << 12, mu=8, nu=8, s_lo=0,
                                s_cnt=1 << 20, algorithm="lefevre", div_mode="hw")),
    ]
    for name, kw in extra:
        if name in have:
            continue
        args = [kw.pop(k) for k in ("fn", "binade", "p", "eps_bits", "tau", "N", "mu", "nu", "s_lo", "s_cnt")]
        cases.append(_case(name, *args, **kw))
    with open(path, "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))
    print("wrote pipeline_cases.json")


if __name__ == "__main__":
    which = sys.argv[1:] or ["search", "pipeline", "extra"]
    if "search" in which:
        search_goldens()
    if "pipeline" in which:
        pipeline_goldens()
    if "extra" in which:
        extra_goldens()
