// hrb_host.cpp -- native host half of the hybrid split (include/hrb_host.h).
//
// Per super-domain: the degree-delta Taylor model of y(x) = 2^(p-e) exp(X(x))
// about the block midpoint with its rigorous error budget (the quantities of
// polygen.py:193-252, in exact dyadic arithmetic), the hierarchical split
// into r_0..r_delta (polygen.py:113-131, closed form for delta <= 2), the
// limb-budget / eps'' / pad checks of the reference's phase 1, and the
// packed hrb_slice columns.  Blocks are independent: OpenMP over blocks.
#include "../../../include/hrb_host.h"

#include <omp.h>

#include "bign.h"
#include "mpexp.h"
#include "decide.h"
#include "polygen.h"

using namespace hrbh;

namespace {

constexpr int VERSION = 100;

bool valid(const hrbh_cfg* c) {
    return c && c->fn == HRBH_FN_EXP && c->precision >= 2 && c->precision <= 64 && c->eps_bits >= 1 &&
           c->binade <= 0 && c->binade > -1000 && c->frac_bits >= 8 && c->guard >= 0 && c->limbs >= 1 &&
           c->limbs <= 16 && (c->delta == 1 || c->delta == 2) && (c->word_bits == 32 || c->word_bits == 64);
}

}  // namespace

extern "C" {

int hrbh_version(void) { return VERSION; }

int hrbh_pack_blocks(const hrbh_cfg* cfg, int64_t S_, const uint64_t* index_start, const uint64_t* count,
                     const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out, uint32_t* coef, uint64_t* G,
                     uint64_t* s2abs, uint8_t* status, uint8_t* shift_ok, int threads) {
    if (!valid(cfg) || S_ < 0) return 2;
    const hrbh_cfg c = *cfg;
    const int cl = c.limbs + 1;
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
    for (int64_t t = 0; t < S_; t++) {
        BlockOut o;
        if (!one_block(c, index_start[t], count[t], n_p[t], tau[t], e_out[t], &o)) {
            status[t] = HRBH_FALLBACK;
            continue;
        }
        status[t] = HRBH_OK;
        shift_ok[t] = o.shift_ok ? 1 : 0;
        for (int k = 0; k < 6; k++) put_limbs(o.r[k], cl, coef, k, S_, t);
        G[t] = o.G.n > 0 ? o.G.w[0] : 0;
        G[S_ + t] = o.G.n > 1 ? o.G.w[1] : 0;
        s2abs[t] = o.s2.n > 0 ? o.s2.w[0] : 0;
        s2abs[S_ + t] = o.s2.n > 1 ? o.s2.w[1] : 0;
    }
    return 0;
}

}  // extern "C"

// ------------------------------------------------------------ confirmation

namespace {

}  // namespace

extern "C" {

int hrbh_confirm(const hrbh_cfg* cfg, int64_t n, const uint64_t* index, uint8_t* is_hr, uint64_t* dist_raw,
                 uint8_t* status, int threads) {
    if (!valid(cfg) || n < 0) return 2;
    const hrbh_cfg c = *cfg;
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 8) num_threads(threads)
    for (int64_t i = 0; i < n; i++) {
        uint64_t d = 0;
        int r = decide_exp(c.precision, c.eps_bits, c.binade, index[i], &d);
        status[i] = r < 0 ? HRBH_FALLBACK : HRBH_OK;
        is_hr[i] = r == 1;
        dist_raw[i] = d;
    }
    return 0;
}

int hrbh_exp_enclose(uint64_t M, int xe, int prec, uint64_t* lo_words, int32_t* lo_exp, uint64_t* hi_words,
                     int32_t* hi_exp, int32_t* nwords) {
    overflow_flag() = false;
    Enc en;
    if (!exp_enclose(M, xe, prec, &en) || en.lm.n > 16 || en.hm.n > 16) return HRBH_FALLBACK;
    int nw = std::max(en.lm.n, en.hm.n);
    for (int i = 0; i < nw; i++) {
        lo_words[i] = i < en.lm.n ? en.lm.w[i] : 0;
        hi_words[i] = i < en.hm.n ? en.hm.w[i] : 0;
    }
    *lo_exp = en.le;
    *hi_exp = en.he;
    *nwords = nw;
    return HRBH_OK;
}

}  // extern "C"

// ------------------------------------------------- high-degree super-domains
//
// delta_R = D in 3..8 over super-domains of tau domains (oracle/wide.py is
// the specification; the reference itself rejects delta >= 3,
// polygen.py:81-82).  Exact dyadic arithmetic scaled by K = (D+1)!, which
// clears every 1/k! of the Taylor coefficients and of the Lagrange term.

namespace {

// round_half_even(m 2^e / K) for signed m, K > 0 (Python round(Fraction))
S round_div(const S& m, int e, uint64_t K) {
    // value = num / den with den = K 2^k (k >= 0) and num = m 2^max(e, 0)
    const int k = e < 0 ? -e : 0;
    const S num = e > 0 ? sshl(m, e) : m;
    // floor(num / (K 2^k)) = floor(floor(num / K) / 2^k)
    uint64_t r;
    U q1 = divmod_u64(num.m, K, &r);
    S fl;
    if (!num.neg) {
        fl = sfloor_shr(S(q1), k);
    } else {
        U c1 = r ? add(q1, U(1)) : q1;  // ceil(|num| / K)
        fl = sfloor_shr(S(c1, true), k);
    }
    // rem = num - fl K 2^k in [0, K 2^k); compare 2 rem with K 2^k
    const S flK = S(shl(mul(fl.m, U(K)), k), fl.neg);
    const S rem = ssub(num, flK);
    const U den = shl(U(K), k);
    const int c = cmp(shl(rem.m, 1), den);
    if (c > 0 || (c == 0 && fl.m.bit(0))) return sadd(fl, S(U(1)));
    return fl;
}

// ceil(v 2^sh / K) for v > 0
U ceil_div(const D& v, int sh, uint64_t K) {
    int e = v.e + sh;
    uint64_t rem;
    if (e >= 0) {
        U qq = divmod_u64(shl(v.m.m, e), K, &rem);
        return rem ? add(qq, U(1)) : qq;
    }
    U qq = divmod_u64(v.m.m, K, &rem);
    if (rem) qq = add(qq, U(1));
    U fl = shr(qq, -e);
    return qq.low_zero(-e) ? fl : add(fl, U(1));
}

U ceil_shr(const U& v, int k) {
    if (k <= 0) return shl(v, -k);
    U fl = shr(v, k);
    return v.low_zero(k) ? fl : add(fl, U(1));
}

struct WideOut {
    S q[45];
    U padg, s2b, win;
};

bool wide_block(const hrbh_cfg& c, int Dg, int NL, uint64_t i0, uint64_t count, uint64_t n_p, uint64_t tau, int e_out,
                WideOut* o) {
    overflow_flag() = false;
    const int p = c.precision, F = 32 * NL, W = c.word_bits;
    if (count < 1 || n_p < 1 || tau < 1 || count > tau * n_p) return false;
    const int prec = F + c.guard + 32;
    const int xe = c.binade + 1 - p;
    const uint64_t mbase = (1ull << (p - 1)) + i0;
    const uint64_t xc = count / 2;
    Enc em, el;
    if (!exp_enclose(mbase + xc, xe, prec, &em) || !exp_enclose(mbase + count - 1, xe, prec, &el)) return false;
    uint64_t K = 1;
    for (int k = 2; k <= Dg + 1; k++) K *= (uint64_t)k;
    const D lo(S(em.lm), em.le), hi(S(em.hm), em.he);
    const D sum = dadd(lo, hi), dif = dsub(hi, lo);
    const int ne = p - e_out;
    D cm[9], cr[9];
    uint64_t kf = 1;  // k!
    for (int k = 0; k <= Dg; k++) {
        if (k > 1) kf *= (uint64_t)k;
        const U mult(K / kf);
        cm[k] = dmul_u(D(sum.m, sum.e - 1 + ne + k * xe), mult);
        cr[k] = dmul_u(D(dif.m, dif.e - 1 + ne + k * xe), mult);
    }
    // K P(x) at x = i n_p + m, i, m = 0..D
    auto PK = [&](uint64_t x) {
        const S t = x >= xc ? S(U(x - xc)) : S(U(xc - x), true);
        D acc;
        D tp(S(U(1)), 0);
        for (int k = 0; k <= Dg; k++) {
            acc = dadd(acc, dmul(cm[k], tp));
            tp = dmul(tp, D(t, 0));
        }
        return acc;
    };
    D vals[9][9];
    for (int i = 0; i <= Dg; i++)
        for (int m = 0; m <= Dg; m++) vals[i][m] = PK((uint64_t)i * n_p + (uint64_t)m);
    const U cnp(n_p - 1), ctau(tau - 1);
    D round_err;  // scaled by K
    int ci = 0;
    for (int j = 0; j <= Dg; j++) {
        D r[9];
        for (int i = 0; i <= Dg - j; i++) {
            D acc;
            for (int m = 0; m <= j; m++) {
                D term = dmul_u(vals[i][m], binom(U((uint64_t)j), m));
                acc = ((j - m) & 1) ? dsub(acc, term) : dadd(acc, term);
            }
            r[i] = acc;
        }
        // forward differences in i: rho_{j,l} = Delta^l r (0)
        const int len = Dg - j + 1;
        const U bj = binom(cnp, j);
        for (int l = 0; l < len; l++) {
            const D rho = r[0];
            const S q = round_div(rho.m, rho.e + F, K);
            o->q[ci + l] = q;
            // |rho K - q K 2^-F| C(tau-1, l) C(n_p-1, j)
            const D err = dabs(dsub(rho, D(smul(q, S(U(K))), -F)));
            round_err = dadd(round_err, dmul_u(dmul_u(err, binom(ctau, l)), bj));
            for (int i = 0; i + 1 < len - l; i++) r[i] = dsub(r[i + 1], r[i]);
        }
        ci += len;
    }
    const uint64_t tmax = std::max(xc, count - 1 - xc);
    D enc_err;
    for (int k = 0; k <= Dg; k++) enc_err = dadd(enc_err, dmul_u(cr[k], upow(U(tmax), k)));
    // lagrange K = norm dsup ulp^(D+1) tmax^(D+1)   (K = (D+1)!)
    const D lagr = dmul_u(D(S(el.hm), el.he + ne + (Dg + 1) * xe), upow(U(tmax), Dg + 1));
    const D ea = dadd(lagr, dadd(enc_err, round_err));
    auto ge_quarter = [&](const D& v) {  // v / K >= 1/4
        int Z = v.e < -2 ? -v.e : 2;
        return scmp(dscaled(v, Z), sshl(S(U(K)), Z - 2)) >= 0;
    };
    if (ge_quarter(ea)) return false;
    const D ep = dadd(D(S(U(K)), -c.eps_bits), ea);
    const U g = ceil_div(ep, F, K);  // ceil(eps' 2^F)
    // S2 and T3 (2^-F units)
    U S2, T3;
    ci = 0;
    for (int j = 0; j <= Dg; j++) {
        const int len = Dg - j + 1;
        for (int l = 0; l < len; l++) {
            const U a = mul(o->q[ci + l].m, binom(ctau, l));
            if (j == 2) S2 = add(S2, a);
            if (j >= 3) T3 = add(T3, mul(a, binom(cnp, j)));
        }
        ci += len;
    }
    // eps'' at the largest count: eps' + (T3 + S2 (n-1)^2) 2^-F < 1/4
    const uint64_t last = count - (tau - 1) * n_p;
    const uint64_t n = std::max(tau > 1 ? n_p : last, last);
    const U tr = add(T3, mul(S2, mul(U(n - 1), U(n - 1))));
    if (ge_quarter(dadd(ep, D(S(mul(tr, U(K))), -F)))) return false;
    o->padg = ceil_shr(add(g, T3), F - 128);
    o->s2b = ceil_shr(S2, F - 128);
    o->win = add(g, U(1));
    // the device forms padg + s2b (n-1)^2 in 128 bits; pad < 2^(W-2)
    const U X = add(o->padg, mul(o->s2b, mul(U(n - 1), U(n - 1))));
    if (X.bitlen() > 128) return false;
    const U pad = add(ceil_shr(X, 128 - W), U(n + 1));
    if (shl(pad, 1).bitlen() > W - 1) return false;
    if (o->win.bitlen() > F) return false;
    return !overflow_flag();
}

}  // namespace

extern "C" {

int hrbh_wide_blocks(const hrbh_cfg* cfg, int degree, int frac_limbs, int64_t S_, const uint64_t* index_start,
                     const uint64_t* count, const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out,
                     uint32_t* coef, uint64_t* padg, uint64_t* s2b, uint32_t* win, uint8_t* status, int threads) {
    if (!cfg || cfg->fn != HRBH_FN_EXP || cfg->binade > 0 || cfg->precision < 2 || cfg->precision > 64 ||
        degree < 3 || degree > 8 || frac_limbs < 4 || frac_limbs > 8 || cfg->word_bits != 64 || S_ < 0)
        return 2;
    const hrbh_cfg c = *cfg;
    const int ncoef = (degree + 1) * (degree + 2) / 2;
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t t = 0; t < S_; t++) {
        WideOut o;
        if (!wide_block(c, degree, frac_limbs, index_start[t], count[t], n_p[t], tau[t], e_out[t], &o)) {
            status[t] = HRBH_FALLBACK;
            continue;
        }
        status[t] = HRBH_OK;
        for (int k = 0; k < ncoef; k++) put_limbs(o.q[k], frac_limbs, coef, k, S_, t);
        padg[t] = o.padg.n > 0 ? o.padg.w[0] : 0;
        padg[S_ + t] = o.padg.n > 1 ? o.padg.w[1] : 0;
        s2b[t] = o.s2b.n > 0 ? o.s2b.w[0] : 0;
        s2b[S_ + t] = o.s2b.n > 1 ? o.s2b.w[1] : 0;
        put_limbs(S(o.win), frac_limbs, win, 0, S_, t);
    }
    return 0;
}

}  // extern "C"
