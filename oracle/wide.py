"""Specification of the high-degree (delta_R >= 3) path -- TEST
INFRASTRUCTURE ONLY (the checker for libhrbhost.so's hrbh_wide_blocks and
for libhrb200.so's hrb_wrun_slice; never imported by the product).

PARITY UNPINNED against the reference for the tabulated values and the
phase flags: the reference rejects delta >= 3 (polygen.py:81-82,
test_polygen.py:181-182).  What is pinned is the end result: the confirmed
HR records must equal the reference's exhaustive_hr_search
(oracle.py:77-113) and the delta = 2 pipeline's records, because every
filter here is sound.

The model follows the paper's large super-domain generation
(one R_t per super-domain of tau domains, hierarchical
split into r_j of degree delta_R - j, tabulated-difference walks) with the
reference's conventions (polygen.py:193-252 for the Taylor model and its
budget, pipeline.py:141-184 for the Boolean problem):

  y(x) = 2^(p - e) f(X(x)), x = argument offset in the super-domain;
  P(x) = sum_k c_k (x - xc)^k, c_k = mid of f^(k)(X(xc)) 2^(p-e) ulp^k / k!;
  r_j(i) = Delta^j P(i N) (unit difference in x), a polynomial of degree
  delta_R - j in the domain index i, in the binomial basis in i:
  r_j(i) = sum_l rho_{j,l} C(i, l);
  the ONLY rounding: q_{j,l} = round_half_even(rho_{j,l} 2^F), F = 32 NL;
  domain polynomial P_i(x) = sum_j r~_j(i) C(x, j), r~_j(i) = sum_l q_{j,l} C(i, l) / 2^F;
  eps_approx = Lagrange + enclosure radii + sum_{j,l} |rho - q/2^F| C(tau-1, l) C(N-1, j);
  degree >= 2 terms of P_i, for any x < N:
     j = 2:  |r~_2(i)| (n-1)^2 <= S2 (n-1)^2,  S2 = sum_l |q_{2,l}| C(tau-1, l)   (2^-F units)
     j >= 3: <= T3 = sum_{j>=3} sum_l |q_{j,l}| C(tau-1, l) C(N-1, j)             (2^-F units)
  device constants (2^-128 units, rounded up; phases 1-2 use
  pad = ceil((padg + s2b (n-1)^2) / 2^(128-W)) + n + 1, as pad_of with F = 128):
     padg = ceil((ceil(eps' 2^F) + T3) / 2^(F-128)),  s2b = ceil(S2 / 2^(F-128)),
  and the phase-3 window (exact, 2^-F units): win = ceil(eps' 2^F) + 1.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np


@dataclass
class WideModel:
    q: list            # q[j][l], ints (signed), j = 0..D, l = 0..D-j
    eps_approx: Fraction
    eps_prime: Fraction
    S2: int
    T3: int
    padg: int
    s2b: int
    win: int


def _round_half_even(x: Fraction) -> int:
    return round(x)


def wide_model(fn: str, p: int, eps_bits: int, binade: int, i0: int, count: int, n_p: int, tau: int, e_out: int,
               D: int, NL: int, guard: int = 32, word_bits: int = 64) -> WideModel:
    from paper_1211_3056_b200.enclosure import derivative_bound, enclose

    if fn != "exp":
        raise ValueError("the wide specification covers exp")
    F = 32 * NL
    prec = F + guard + 32
    xe = binade + 1 - p
    ulp = Fraction(2) ** xe
    norm = Fraction(2) ** (p - e_out)
    mbase = (1 << (p - 1)) + i0
    xc = count // 2
    Xc = Fraction(mbase + xc) * ulp
    lo, hi = enclose("exp", Xc, prec)
    cm = [(lo + hi) / 2 * norm * ulp ** k / math.factorial(k) for k in range(D + 1)]
    cr = [(hi - lo) / 2 * norm * ulp ** k / math.factorial(k) for k in range(D + 1)]

    def P(x: int) -> Fraction:
        t = x - xc
        return sum((c * t ** k for k, c in enumerate(cm)), Fraction(0))

    vals = {(i, m): P(i * n_p + m) for i in range(D + 1) for m in range(D + 1)}
    q, round_err = [], Fraction(0)
    for j in range(D + 1):
        r = [sum(((-1) ** (j - m)) * math.comb(j, m) * vals[(i, m)] for m in range(j + 1)) for i in range(D - j + 1)]
        rho, cur = [], r
        while True:
            rho.append(cur[0])
            if len(cur) == 1:
                break
            cur = [b - a for a, b in zip(cur, cur[1:])]
        qj = [_round_half_even(x * (1 << F)) for x in rho]
        q.append(qj)
        for l, (x, ql) in enumerate(zip(rho, qj)):
            round_err += abs(x - Fraction(ql, 1 << F)) * math.comb(tau - 1, l) * math.comb(n_p - 1, j)
    t_max = max(xc, count - 1 - xc)
    enc_err = sum((r * t_max ** k for k, r in enumerate(cr)), Fraction(0))
    X_last = Fraction(mbase + count - 1) * ulp
    dsup = derivative_bound("exp", D + 1, Fraction(mbase) * ulp, X_last, prec)
    lagrange = norm * dsup * ulp ** (D + 1) * Fraction(t_max) ** (D + 1) / math.factorial(D + 1)
    eps_approx = lagrange + enc_err + round_err
    eps_prime = Fraction(1, 1 << eps_bits) + eps_approx
    S2 = sum(abs(x) * math.comb(tau - 1, l) for l, x in enumerate(q[2])) if D >= 2 else 0
    T3 = sum(abs(x) * math.comb(tau - 1, l) * math.comb(n_p - 1, j)
             for j in range(3, D + 1) for l, x in enumerate(q[j]))
    g = -((-eps_prime.numerator << F) // eps_prime.denominator)
    sh = F - 128
    padg = -(-(g + T3) >> sh)
    s2b = -(-S2 >> sh)
    return WideModel(q, eps_approx, eps_prime, S2, T3, padg, s2b, g + 1)


def r_tilde(q: list, j: int, i: int) -> int:
    """r~_j(i) 2^F exactly: sum_l q_{j,l} C(i, l)."""
    return sum(x * math.comb(i, l) for l, x in enumerate(q[j]))


def pad_of(padg: int, s2b: int, n: int, W: int = 64) -> int:
    X = padg + s2b * (n - 1) ** 2
    sh = 128 - W
    return -(-X >> sh) + n + 1


def problem(s0: int, s1: int, pad: int, F: int, W: int = 64):
    """_boolean_problem (pipeline.py:149-175) from residues mod 2^F."""
    one = 1 << F
    s0m, s1m = s0 % one, (-s1) % one
    a = (s1m << W) >> F
    b = (((s0m << W) >> F) + pad) & ((1 << W) - 1)
    return a, b, 2 * pad


def pipeline(models, slice_geom, fmt_p: int, binade: int, NL: int, split: int = 8, W: int = 64):
    """Phases 1-3 of a wide slice, exact (Python ints + the C oracle's
    regular search): models[t] = WideModel, slice_geom[t] = (index_start,
    count, n_p, tau, dom_id0).  Returns (fail ids, sub rows (id, j, start,
    cnt), candidates (argument index, dist 2^-64, domain id))."""
    import oracle

    F = 32 * NL
    one = 1 << F
    items = []  # (id, t, i, n)
    for t, (i0, count, n_p, tau, id0) in enumerate(slice_geom):
        for i in range(tau):
            n = min(n_p, count - i * n_p)
            items.append((id0 + i, t, i, n))
    a, b, e, N = [], [], [], []
    for did, t, i, n in items:
        m = models[t]
        s0, s1 = r_tilde(m.q, 0, i), r_tilde(m.q, 1, i)
        aa, bb, ee = problem(s0, s1, pad_of(m.padg, m.s2b, n, W), F, W)
        a.append(aa), b.append(bb), e.append(ee), N.append(n)
    ok = oracle.search_batch("regular", 1, 1 << W, a, b, e, N)[0]
    fails = [it for it, o in zip(items, ok.tolist()) if not o]
    subs = []
    a, b, e, N = [], [], [], []
    for did, t, i, n in fails:
        m = models[t]
        D = len(m.q) - 1
        s = [r_tilde(m.q, j, i) for j in range(D + 1)]
        step = max(n // split, 1)
        for jj, start in enumerate(range(0, n, step)):
            cnt = min(step, n - start)
            s0 = sum(s[k] * math.comb(start, k) for k in range(D + 1))
            s1 = sum(s[k] * math.comb(start, k - 1) for k in range(1, D + 1))
            aa, bb, ee = problem(s0, s1, pad_of(m.padg, m.s2b, cnt, W), F, W)
            subs.append((did, t, i, jj, start, cnt, s))
            a.append(aa), b.append(bb), e.append(ee), N.append(cnt)
    ok = oracle.search_batch("regular", 1, 1 << W, a, b, e, N)[0] if subs else np.zeros(0, np.uint8)
    surv = [sb for sb, o in zip(subs, ok.tolist()) if not o]
    cands = []
    for did, t, i, jj, start, cnt, s in surv:
        m = models[t]
        D = len(s) - 1
        i0, count, n_p, tau, id0 = slice_geom[t]
        # difference column of P_i at x = start: Delta^l P_i(start) = sum_k s_k C(start, k - l)
        col = [sum(s[k] * math.comb(start, k - l) for k in range(l, D + 1)) % one for l in range(D + 1)]
        win = m.win
        for x in range(cnt):
            v = col[0]
            if v < win or v > one - win:
                dist = min(v, one - v)
                cands.append((i0 + i * n_p + start + x, (dist << 64) >> F, did))
            for l in range(D):
                col[l] = (col[l] + col[l + 1]) % one
    return ([f[0] for f in fails], [(sb[0], sb[3], sb[4], sb[5]) for sb in surv], cands)
