// polygen.h -- one super-domain of the native generation (host library and
// device kernel share this source; include/hrb_host.h hrbh_pack_blocks,
// include/hrb200.h hrb_pack_blocks).
//
// Per super-domain: the degree-delta Taylor model of y(x) = 2^(p-e) exp(X(x))
// about the block midpoint with its rigorous error budget (the quantities of
// polygen.py:193-252, in exact dyadic arithmetic), the hierarchical split
// into r_0..r_delta (polygen.py:113-131, closed form for delta <= 2), the
// limb-budget / eps'' / pad checks of the reference's phase 1
// (slices.check_super), and the packed hrb_slice columns.
#pragma once

#include "../../../include/hrb_host.h"
#include "bign.h"
#include "mpexp.h"

namespace hrbh {

HRBH_HD uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

HRBH_HD U binom(const U& n, int k) {  // C(n, k) for small k, n >= 0
    if (k == 0) return U(1);
    U acc(1);
    for (int i = 0; i < k; i++) {
        // acc = acc * (n - i) / (i + 1), exact at every step
        U ni = cmp(n, U((uint64_t)i)) >= 0 ? sub(n, U((uint64_t)i)) : U();
        if (ni.zero()) return U();
        acc = divmod_u64(mul(acc, ni), (uint64_t)(i + 1));
    }
    return acc;
}

// two's complement of v over cl 32-bit limbs into column t of rows [row..)
HRBH_HD void put_limbs(const S& v, int cl, uint32_t* coef, int64_t row, int64_t S_, int64_t t) {
    // two's complement: for negative v, 2^(32 cl) - |v|
    U m = v.m;
    U tc;
    if (v.neg) {
        U full = pow2(32 * cl);
        tc = sub(full, low_bits(m, 32 * cl));
        tc = low_bits(tc, 32 * cl);
    } else {
        tc = low_bits(m, 32 * cl);
    }
    for (int l = 0; l < cl; l++) {
        int wi = (32 * l) / 64, sh = (32 * l) % 64;
        uint64_t w = wi < tc.n ? tc.w[wi] : 0;
        coef[(row * cl + l) * S_ + t] = (uint32_t)(w >> sh);
    }
}

struct BlockOut {
    S r[6];  // r0.c0 r0.c1 r0.c2 r1.c0 r1.c1 r2.c0
    U G;
    U s2;
    bool shift_ok;
};

// One super-domain.  Returns false for a fallback item (not covered, or the
// reference would raise on it).
HRBH_HD bool one_block(const hrbh_cfg& c, uint64_t i0, uint64_t count, uint64_t n_p, uint64_t tau, int e_out,
                       BlockOut* o) {
    overflow_flag() = false;
    const int p = c.precision, F = c.frac_bits, delta = c.delta, L = c.limbs, W = c.word_bits;
    if (count < 1 || n_p < 1 || tau < 1 || count > tau * n_p) return false;
    const int prec = F + c.guard + 32;
    const int xe = c.binade + 1 - p;  // X = M 2^xe; also ulp = 2^xe
    const uint64_t mbase = (1ull << (p - 1)) + i0;
    const uint64_t xc = count / 2;
    Enc em, el;
    if (!exp_enclose(mbase + xc, xe, prec, &em) || !exp_enclose(mbase + count - 1, xe, prec, &el)) return false;
    const D lo(S(em.lm), em.le), hi(S(em.hm), em.he);
    const D sum = dadd(lo, hi), dif = dsub(hi, lo);
    const int ne = p - e_out;  // norm = 2^ne
    // mids[k] = (lo + hi)/2 * norm ulp^k / k!, rads[k] = (hi - lo)/2 * ...
    D mids[3], rads[3];
    for (int k = 0; k <= delta; k++) {
        int sh = -1 + ne + k * xe - (k == 2 ? 1 : 0);
        mids[k] = D(sum.m, sum.e + sh);
        rads[k] = D(dif.m, dif.e + sh);
    }
    const S sxc = S(U(xc));
    const D dxc(sxc, 0);
    // monomial about xc -> monomial in x -> binomial basis
    D a0 = dadd(dsub(mids[0], dmul(mids[1], dxc)), dmul(mids[2], dmul(dxc, dxc)));
    D a1 = dsub(mids[1], D(sshl(dmul(mids[2], dxc).m, 1), dmul(mids[2], dxc).e));
    D a2 = mids[2];
    D tg[3] = {a0, dadd(a1, a2), D(sshl(a2.m, 1), a2.e)};
    S q[3];
    D round_err;
    const U cm1(count - 1);
    for (int j = 0; j <= delta; j++) {
        const D& s = tg[j];
        int k = -(s.e + F);
        q[j] = k > 0 ? sround_shr(s.m, k) : sshl(s.m, -k);
        D diff = dabs(dsub(s, D(q[j], -F)));
        round_err = dadd(round_err, dmul_u(diff, binom(cm1, j)));
    }
    const uint64_t tmax = umax64(xc, count - 1 - xc);
    D enc_err;
    for (int k = 0; k <= delta; k++) enc_err = dadd(enc_err, dmul_u(rads[k], upow(U(tmax), k)));
    // lagrange * (delta+1)! = norm * dsup * ulp^(delta+1) * tmax^(delta+1)
    const uint64_t fact = delta == 1 ? 2 : 6;
    D lagr = dmul_u(D(S(el.hm), el.he + ne + (delta + 1) * xe), upow(U(tmax), delta + 1));
    // eps_approx * fact
    D ea = dadd(lagr, dmul_u(dadd(enc_err, round_err), U(fact)));
    // eps_approx >= 1/4  <=>  ea >= fact / 4
    {
        int Z = ea.e < -2 ? -ea.e : 2;
        S lhs = dscaled(ea, Z);                 // ea * 2^Z
        S rhs = sshl(S(U(fact)), Z - 2);        // fact / 4 * 2^Z
        if (scmp(lhs, rhs) >= 0) return false;  // "approximation budget blown"
    }
    // MPInt.from_int(q, L) and the split's intermediates stay under 2^(32 L)
    const int lim = 32 * L;
    U bsplit;
    const U two_s(2 * n_p + 2);
    for (int j = 0; j <= delta; j++) {
        if (q[j].m.bitlen() > lim) return false;
        bsplit = add(bsplit, mul(q[j].m, binom(two_s, j)));
    }
    if (shl(bsplit, 3).bitlen() > lim) return false;
    // hierarchical split (closed form of r_j(i) = Delta^j R_t(i n_p))
    const S ss = S(U(n_p));
    S r[6];
    if (delta == 2) {
        S cs2 = S(divmod_u64(mul(U(n_p), U(n_p - 1)), 2));  // C(n_p, 2)
        r[0] = q[0];
        r[1] = sadd(smul(q[1], ss), smul(q[2], cs2));
        r[2] = smul(q[2], smul(ss, ss));
        r[3] = q[1];
        r[4] = smul(q[2], ss);
        r[5] = q[2];
    } else {
        r[0] = q[0];
        r[1] = smul(q[1], ss);
        r[3] = q[1];
    }
    // slices.check_super: walk bound, eps'' < 1/4, pad
    const U utau(tau);
    U bound;
    {
        const int rows[3][3] = {{0, 1, 2}, {3, 4, -1}, {5, -1, -1}};
        for (int j = 0; j <= delta; j++) {
            U acc;
            U tp(1);
            for (int l = 0; l < 3 && rows[j][l] >= 0 && l <= delta - j; l++) {
                acc = add(acc, mul(r[rows[j][l]].m, tp));
                tp = mul(tp, utau);
            }
            if (cmp(acc, bound) > 0) bound = acc;
        }
    }
    if (bound.bitlen() > lim || mul(utau, utau).bitlen() > lim) return false;  // exact MPInt replay needed
    const uint64_t last = count - (tau - 1) * n_p;
    const uint64_t n = umax64(tau > 1 ? n_p : last, last);
    // eps' * fact = fact 2^-eps_bits + ea
    D epf = dadd(D(S(U(fact)), -c.eps_bits), ea);
    const U s2 = delta == 2 ? q[2].m : U();
    // eps'' * fact = eps' fact + fact |s2| (n-1)^2 2^-F
    D edp = dadd(epf, D(S(mul(mul(s2, U(fact)), mul(U(n - 1), U(n - 1)))), -F));
    {
        int Z = edp.e < -2 ? -edp.e : 2;
        if (scmp(dscaled(edp, Z), sshl(S(U(fact)), Z - 2)) >= 0) return false;  // eps'' >= 1/4
    }
    // pad = ceil(eps'' 2^W) + n + 1 ; 2 pad < 2^(W-1)
    auto ceil_scaled = [&](const D& v, int sh) -> U {  // ceil(v * 2^sh / fact), v > 0
        int e = v.e + sh;
        if (e >= 0) {
            uint64_t rem;
            U qq = divmod_u64(shl(v.m.m, e), fact, &rem);
            return rem ? add(qq, U(1)) : qq;
        }
        uint64_t rem;
        U qq = divmod_u64(v.m.m, fact, &rem);
        if (rem) qq = add(qq, U(1));
        U fl = shr(qq, -e);
        return qq.low_zero(-e) ? fl : add(fl, U(1));
    };
    U pad = add(ceil_scaled(edp, W), U(n + 1));
    if (shl(pad, 1).bitlen() > W - 1) return false;  // "eps must be < 1/2"
    U b2;
    {
        U np_pow(1);
        for (int l = 0; l <= delta; l++) {
            b2 = add(b2, mul(bound, np_pow));
            np_pow = mul(np_pow, U(n_p));
        }
    }
    o->shift_ok = b2.bitlen() <= lim;
    o->G = ceil_scaled(epf, F);
    if (o->G.bitlen() > 128) return false;
    o->s2 = s2.bitlen() > 128 ? sub(pow2(128), U(1)) : s2;
    for (int k = 0; k < 6; k++) o->r[k] = r[k];
    return !overflow_flag();
}

}  // namespace hrbh
