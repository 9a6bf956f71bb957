// mpexp.h -- exact restatement of the interval exp the host path depends on.
//
// The reference's Taylor models and its HR confirmation take their values
// from mpmath's interval context (evalf.py:98-121: iv.exp of a point
// interval at `work` bits).  For an argument X of a binade <= 0 that is
//   lo = mpf_exp(X, work, round_floor), hi = mpf_exp(X, work, round_ceiling)
// in mpmath 1.3.0 (the pinned version: pyproject.toml:10-13 requires
// >= 1.2; 1.3.0 is installed), libmp/libelefun.py:
//   mpf_exp (1151-1188): wp = work + 14; |X| < 2 so no ln2 reduction:
//       t = X * 2^wp (exact), man = exp_basecase(t, wp),
//       from_man_exp(man, -wp, work, rnd);
//   exp_basecase (1086-1109), for wp <= EXP_COSH_CUTOFF (600 with the
//       python backend, 400 with gmpy; callers stay <= 400 so both agree):
//       r = isqrt(wp); P = wp + r (t is read at scale 2^P: X / 2^r);
//       even/odd Taylor sums s0, s1 with floor divisions by k;
//       s = s0 + s1 * t; r squarings; result s >> r.
// Every step is integer arithmetic with explicit floors, so the endpoints
// below are bit-identical to mpmath's, not merely close.
#pragma once

#include "bign.h"

namespace hrbh {

constexpr int EXP_MAX_WP = 400;

// mpmath exp_basecase(x, prec) (libelefun.py:1086-1109)
HRBH_HD U exp_basecase(const U& x, int prec) {
    int r = (int)isqrt_u64((uint64_t)prec);
    const int P = prec + r;
    U s0 = pow2(P), s1 = s0;
    uint64_t k = 2;
    U x2 = shr(mul(x, x), P);
    U a = x2;
    while (!a.zero()) {
        a = divmod_u64(a, k);
        s0 = add(s0, a);
        k++;
        a = divmod_u64(a, k);
        s1 = add(s1, a);
        k++;
        a = shr(mul(a, x2), P);
    }
    s1 = shr(mul(s1, x), P);
    U s = add(s0, s1);
    for (int i = 0; i < r; i++) s = shr(mul(s, s), P);
    return shr(s, r);
}

// Enclosure [lo, hi] of exp(X), X = M * 2^xe > 0 with X < 2, exactly as
// evalf.enclose("exp", X, prec) computes it (work = max(prec, bit lengths
// of X's reduced numerator and denominator) + 8).  lo = lm * 2^le,
// hi = hm * 2^he.  Returns false when this restatement does not cover the
// case (X >= 2 uses an ln2 reduction; very high precision another series).
struct Enc {
    U lm, hm;
    int le = 0, he = 0;
};

HRBH_HD int reduced_bits(uint64_t M, int xe, int* den_bits) {
    // X = M 2^xe as a reduced fraction num / den
    int tz = ctz64(M);
    uint64_t num = M >> tz;
    int e = xe + tz;
    int nb = 64 - clz64(num);
    if (e >= 0) {
        *den_bits = 1;
        return nb + e;
    }
    *den_bits = -e + 1;  // bit length of 2^-e
    return nb;
}

HRBH_HD bool exp_enclose(uint64_t M, int xe, int prec, Enc* out) {
    if (M == 0) return false;
    int den_bits;
    int num_bits = reduced_bits(M, xe, &den_bits);
    int work = imax(prec, imax(num_bits, den_bits)) + 8;
    int wp = work + 14;
    // mpmath's mag = bitcount(man) + exp = floor(log2 X) + 1
    int mag = (63 - clz64(M)) + xe + 1;
    if (mag > 1 || mag < -wp || wp > EXP_MAX_WP) return false;
    // t = X * 2^wp; offset = exp + wp where X = man 2^exp (man odd)
    int tz = ctz64(M);
    U man((uint64_t)(M >> tz));
    int offset = xe + tz + wp;
    U t = offset >= 0 ? shl(man, offset) : shr(man, -offset);
    U m = exp_basecase(t, wp);
    // from_man_exp(m, -wp, work, floor / ceiling)
    int bc = m.bitlen();
    int n = bc > work ? bc - work : 0;
    U fl = shr(m, n);
    U ce = (n && !m.low_zero(n)) ? add(fl, U(1)) : fl;
    out->lm = fl;
    out->hm = ce;
    out->le = n - wp;
    out->he = n - wp;
#if defined(__CUDA_ARCH__)
    return true;  // device callers stay within the capacity (confirm.cuh)
#else
    return !overflow_flag();
#endif
}

}  // namespace hrbh
