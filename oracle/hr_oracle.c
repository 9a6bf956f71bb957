/*
 * hr_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links this file:
 * it is loaded by tests/, by __graft_entry__.smoke() as the checker, and by
 * bench.py's cpu_baseline / --impl reference legs.  It restates, in plain C
 * with exact 128-bit (and multi-limb) integer arithmetic, the algorithms of
 * the reference package (PUBLIC reference at /root/reference/pkg/src/hardround):
 *
 *   or_lefevre_core          lowerbound.py:88-163   (_lefevre_core)
 *   or_lefevre_swap_core     lowerbound.py:166-225  (_lefevre_swap_core)
 *   or_regular_core          lowerbound.py:228-267  (_regular_core)
 *   or_regular_unrolled_core lowerbound.py:270-308  (_regular_unrolled_core)
 *   tabulated walk           polygen.py:134-158, 255-280 (tabulated_shift_step,
 *                            straightforward_shift, generate_packets,
 *                            domain_coefficient_sets) on MPInt semantics
 *                            (fixedpoint.py:140-305: |x| < 2^(32L) or overflow)
 *   boolean problem          pipeline.py:141-175 (_truncation_eps, _boolean_problem)
 *   phase1 / phase2 / phase3 pipeline.py:213-293
 *
 * Arithmetic domain: the search cores take a general modulus `one` <= 2^64
 * (so the small-modulus sweeps of test_lowerbound.py:213-254 run here too);
 * all quantities live in unsigned/signed __int128, which covers the 65-bit
 * point counts of the reference (e.g. a=1 gives 2^64+1 points).
 *
 * The pad of the Boolean problem is evaluated in the closed form
 *     pad = ceil((G + |s2|*(n-1)^2) / 2^(F-W)) + n + 1,  G = ceil(eps' * 2^F)
 * which equals ceil(eps''*2^W) + n + 1 of pipeline.py:165-166 exactly (the
 * identity ceil(X/M) = ceil(ceil(X)/M) for integer M); tests pin it against
 * the Fraction form.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------ */
/* search cores                                                         */
/* ------------------------------------------------------------------ */

typedef struct {
    int ok;
    u128 d;
    uint64_t it;
    u128 pts;
} core_out;

static inline core_out mk(int ok, u128 d, uint64_t it, u128 pts) {
    core_out o;
    o.ok = ok;
    o.d = d;
    o.it = it;
    o.pts = pts;
    return o;
}

/* ceil(need / den) for need > 0, den > 0 */
static inline u128 ceil_div(u128 need, u128 den) { return (need + den - 1) / den; }

/* lowerbound.py:88-163.  mode: 0 subtractive, 1 hybrid, 2 hardware (the
 * reference's _mode_code); anything else behaves like 2 (mode None). */
core_out or_lefevre_core(u128 a, u128 b, u128 eps, u128 N, u128 one, int mode) {
    u128 d = b;
    if (d < eps) return mk(0, d, 0, 1);
    if (a == 0) return mk(1, d, 0, N);
    if (N == 1) return mk(1, d, 0, 1);
    u128 p = a, q = one - a, u = 1, v = 1;
    uint64_t it = 0;
    for (;;) {
        if (d < p) {
            it++;
            u128 k = q / p;
            i128 need = (i128)N - (i128)u - (i128)v;
            u128 kc = need > 0 ? ceil_div((u128)need, v) : 0;
            if (k >= kc) return mk(1, d, it, u + kc * v + v);
            q -= k * p;
            u += k * v;
            if (q == 0) return mk(1, d, it, N);
            p -= q;
            v += u;
        } else {
            it++;
            d -= p;
            if (d < eps) return mk(0, d, it, u + v);
            u128 k = p / q;
            if (k == 0) {
                if (u + v >= N) return mk(1, d, it, u + v);
                q -= p;
                u += v;
                if (mode != 0) {
                    int extra = 0;
                    while (d >= p && q > p) {
                        if (mode == 1 && !extra) {
                            it++;
                            extra = 1;
                        }
                        d -= p;
                        if (d < eps) return mk(0, d, it, u + v);
                        if (u + v >= N) return mk(1, d, it, u + v);
                        q -= p;
                        u += v;
                    }
                }
            } else {
                i128 need = (i128)N - (i128)u - (i128)v;
                u128 kc = need > 0 ? ceil_div((u128)need, u) : 0;
                if (k >= kc) return mk(1, d, it, u + v + kc * u);
                p -= k * q;
                v += k * u;
                if (p == 0) return mk(1, d, it, N);
                q -= p;
                u += v;
            }
        }
    }
}

/* lowerbound.py:166-225 */
core_out or_lefevre_swap_core(u128 a, u128 b, u128 eps, u128 N, u128 one, int mode) {
    u128 d = b, t;
    if (d < eps) return mk(0, d, 0, 1);
    if (a == 0) return mk(1, d, 0, N);
    if (N == 1) return mk(1, d, 0, 1);
    u128 p = a, q = one - a, u = 1, v = 1;
    int swapped = d >= p;
    if (swapped) {
        t = p; p = q; q = t;
        t = u; u = v; v = t;
    }
    uint64_t it = 0;
    for (;;) {
        it++;
        if (swapped) {
            d -= q;
            if (d < eps) return mk(0, d, it, u + v);
        }
        u128 k = q / p;
        i128 need = (i128)N - (i128)u - (i128)v;
        u128 kc = need > 0 ? ceil_div((u128)need, v) : 0;
        if (k >= kc) return mk(1, d, it, u + kc * v + v);
        q -= k * p;
        u += k * v;
        if (q == 0) return mk(1, d, it, N);
        p -= q;
        v += u;
        if (swapped && k == 0 && mode != 0) {
            int extra = 0;
            while (d >= q && q < p) {
                if (mode == 1 && !extra) {
                    it++;
                    extra = 1;
                }
                d -= q;
                if (d < eps) return mk(0, d, it, u + v);
                if (u + v >= N) return mk(1, d, it, u + v);
                p -= q;
                v += u;
            }
        }
        int nxt = d >= (swapped ? q : p);
        if (nxt != swapped) {
            t = p; p = q; q = t;
            t = u; u = v; v = t;
            swapped = nxt;
        }
    }
}

static inline u128 umax(u128 x, u128 y) { return x > y ? x : y; }

/* lowerbound.py:228-267 */
core_out or_regular_core(u128 a, u128 b, u128 eps, u128 N, u128 one) {
    u128 d = b;
    if (d < eps) return mk(0, d, 0, 1);
    if (a == 0) return mk(d > eps, d, 0, N);
    u128 p = a, q = one, u = 1, v = 0;
    if (N <= 1) return mk(d > eps, d, 0, 1);
    uint64_t it = 0;
    for (;;) {
        it++;
        if (p < q) {
            u128 k = q / p;
            q -= k * p;
            v += k * u;
            d %= p;
            if (q == 0) return mk(d > eps, d, it, umax(u + v, N));
        } else {
            u128 k = p / q;
            p -= k * q;
            u += k * v;
            if (d >= p) d = (d - p) % q;
            if (p == 0) return mk(d > eps, d, it, umax(u + v, N));
        }
        if (u + v >= N) return mk(d > eps, d, it, u + v);
    }
}

/* lowerbound.py:270-308 */
core_out or_regular_unrolled_core(u128 a, u128 b, u128 eps, u128 N, u128 one) {
    u128 d = b;
    if (d < eps) return mk(0, d, 0, 1);
    if (a == 0) return mk(d > eps, d, 0, N);
    u128 p = a, q = one, u = 1, v = 0;
    if (N <= 1) return mk(d > eps, d, 0, 1);
    uint64_t it = 0;
    for (;;) {
        it++;
        u128 k = q / p;
        q -= k * p;
        v += k * u;
        d %= p;
        if (q == 0) return mk(d > eps, d, it, umax(u + v, N));
        if (u + v >= N) return mk(d > eps, d, it, u + v);
        k = p / q;
        p -= k * q;
        u += k * v;
        if (d >= p) d = (d - p) % q;
        if (p == 0) return mk(d > eps, d, it, umax(u + v, N));
        if (u + v >= N) return mk(d > eps, d, it, u + v);
    }
}

enum { ALG_LEFEVRE = 0, ALG_LEFEVRE_SWAP = 1, ALG_REGULAR = 2, ALG_REGULAR_UNROLLED = 3 };

static core_out run_core(int algo, int mode, u128 a, u128 b, u128 eps, u128 N, u128 one) {
    switch (algo) {
    case ALG_LEFEVRE: return or_lefevre_core(a, b, eps, N, one, mode);
    case ALG_LEFEVRE_SWAP: return or_lefevre_swap_core(a, b, eps, N, one, mode);
    case ALG_REGULAR: return or_regular_core(a, b, eps, N, one);
    default: return or_regular_unrolled_core(a, b, eps, N, one);
    }
}

static int g_threads = 0; /* 0 = OpenMP default */

void or_set_threads(int n) { g_threads = n; }

int or_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Batched cores over SoA inputs.  `one` = one_lo + 2^64*one_hi (<= 2^64).
 * count may be any u64 >= 1.  Outputs: ok, d (low 64 bits; d < one), it,
 * points as (lo, hi).
 */
void or_search_batch(int algo, int mode, uint64_t one_lo, uint64_t one_hi, int64_t n,
                     const uint64_t* a, const uint64_t* b, const uint64_t* eps,
                     const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* it,
                     uint64_t* pts_lo, uint64_t* pts_hi) {
    u128 one = ((u128)one_hi << 64) | one_lo;
    int nt = or_get_threads();
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nt)
    for (int64_t i = 0; i < n; i++) {
        core_out o = run_core(algo, mode, a[i], b[i], eps[i], count[i], one);
        ok[i] = (uint8_t)o.ok;
        d[i] = (uint64_t)o.d;
        it[i] = o.it;
        pts_lo[i] = (uint64_t)o.pts;
        pts_hi[i] = (uint64_t)(o.pts >> 64);
    }
}

/* ------------------------------------------------------------------ */
/* multi-limb signed integers (MPInt semantics, fixedpoint.py:140-305)  */
/* ------------------------------------------------------------------ */

#define NW 12 /* 384-bit two's complement working width; supports L <= 11 */

typedef struct {
    uint32_t w[NW];
} big;

static void big_from_limbs(big* x, const uint32_t* limbs, int cl) {
    /* cl-limb two's complement input, sign-extended */
    uint32_t ext = (limbs[cl - 1] & 0x80000000u) ? 0xFFFFFFFFu : 0;
    for (int i = 0; i < NW; i++) x->w[i] = i < cl ? limbs[i] : ext;
}

static void big_add(big* r, const big* x, const big* y) {
    uint64_t c = 0;
    for (int i = 0; i < NW; i++) {
        uint64_t s = (uint64_t)x->w[i] + y->w[i] + c;
        r->w[i] = (uint32_t)s;
        c = s >> 32;
    }
}

/* r = x * m for unsigned 64-bit m (signed x) */
static void big_mul_u64(big* r, const big* x, uint64_t m) {
    int neg = (x->w[NW - 1] >> 31) & 1;
    big mag;
    if (neg) {
        uint64_t c = 1;
        for (int i = 0; i < NW; i++) {
            uint64_t s = (uint64_t)(uint32_t)~x->w[i] + c;
            mag.w[i] = (uint32_t)s;
            c = s >> 32;
        }
    } else {
        mag = *x;
    }
    big out;
    memset(&out, 0, sizeof out);
    uint32_t ml = (uint32_t)m, mh = (uint32_t)(m >> 32);
    for (int i = 0; i < NW; i++) {
        u128 carry = 0;
        /* accumulate mag.w[i]*m into out starting at limb i */
        u128 prod = (u128)mag.w[i] * ml + ((u128)mag.w[i] * mh << 32);
        for (int j = i; j < NW && (prod || carry); j++) {
            u128 s = (u128)out.w[j] + (uint32_t)prod + carry;
            out.w[j] = (uint32_t)s;
            carry = s >> 32;
            prod >>= 32;
        }
    }
    if (neg) {
        uint64_t c = 1;
        for (int i = 0; i < NW; i++) {
            uint64_t s = (uint64_t)(uint32_t)~out.w[i] + c;
            out.w[i] = (uint32_t)s;
            c = s >> 32;
        }
    }
    *r = out;
}

/* |x| >= 2^(32L): MPInt overflow (fixedpoint.py:238-252, 291, 300) */
static int big_overflows(const big* x, int L) {
    int neg = (x->w[NW - 1] >> 31) & 1;
    if (!neg) {
        for (int i = L; i < NW; i++)
            if (x->w[i]) return 1;
        return 0;
    }
    /* negative: |x| >= 2^(32L)  <=>  x <= -2^(32L)  <=> upper limbs not all-ones,
     * or all-ones upper with low L limbs all zero */
    for (int i = L; i < NW; i++)
        if (x->w[i] != 0xFFFFFFFFu) return 1;
    for (int i = 0; i < L; i++)
        if (x->w[i]) return 0;
    return 1;
}

/* low 128 bits (mod 2^128) */
static u128 big_lo128(const big* x) {
    return ((u128)x->w[3] << 96) | ((u128)x->w[2] << 64) | ((u128)x->w[1] << 32) | x->w[0];
}

/*
 * straightforward_shift (polygen.py:143-158) of a degree<=2 binomial-basis
 * polynomial c[0..deg] by i, with MPInt overflow tracking on every
 * intermediate (coefficient x binomial product, then each partial sum).
 */
static void shift_poly(big* out, const big* c, int deg, uint64_t i, int L, int* ovf) {
    uint64_t binom[3];
    binom[0] = 1;
    binom[1] = i;
    /* C(i,2) = i*(i-1)/2; i < 2^33 in every supported configuration */
    binom[2] = (uint64_t)(((u128)i * (i > 0 ? i - 1 : 0)) / 2);
    if (i == 0) binom[2] = 0;
    for (int l = 0; l <= deg; l++) {
        big acc = c[l];
        for (int m = l + 1; m <= deg; m++) {
            big term;
            /* MPInt coercion of the int binomial (fixedpoint.py:165-167) */
            if (L < 2 && (binom[m - l] >> (32 * L))) *ovf = 1;
            big_mul_u64(&term, &c[m], binom[m - l]);
            if (big_overflows(&term, L)) *ovf = 1;
            big_add(&acc, &acc, &term);
            if (big_overflows(&acc, L)) *ovf = 1;
        }
        out[l] = acc;
    }
}

/* ------------------------------------------------------------------ */
/* slice phases                                                         */
/* ------------------------------------------------------------------ */

/*
 * Slice description shared with the device path (see include/hrb200.h):
 *   coef   : uint32 [6][CL][S] two's complement, coefficient order
 *            r0.c0, r0.c1, r0.c2, r1.c0, r1.c1, r2.c0 (binomial basis in the
 *            packet variable i, polygen.py:113-131), limb-major SoA
 *   G      : ceil(eps' * 2^F) as (lo, hi) u64 pairs  [2][S]
 *   s2abs  : |r2| saturated to 2^128-1               [2][S]
 *   n_dom  : domains in the super-domain             [S]
 *   dom_n  : domain size N_t                         [S]
 *   last_n : size of the last domain                 [S]
 *   nu     : reference packet length (overflow order) [S]
 *   dom_id0: global id of the first domain           [S]
 *   m0     : binade index of the first argument      [S]
 */
typedef struct {
    int64_t S;
    int CL, L, F, W, delta;
    const uint32_t* coef;
    const uint64_t* G;
    const uint64_t* s2abs;
    const uint32_t* n_dom;
    const uint32_t* dom_n;
    const uint32_t* last_n;
    const uint32_t* nu;
    const uint64_t* dom_id0;
    const uint64_t* m0;
} slice_t;

static void load_coef(const slice_t* s, int64_t t, int c, big* out) {
    uint32_t limbs[NW];
    for (int l = 0; l < s->CL; l++) limbs[l] = s->coef[((int64_t)c * s->CL + l) * s->S + t];
    big_from_limbs(out, limbs, s->CL);
}

static inline u128 mask_f(int F) { return F >= 128 ? ~(u128)0 : (((u128)1 << F) - 1); }

/* pad of pipeline.py:165-166 in closed form (see header) */
static u128 pad_of(u128 G, u128 s2abs, uint64_t n, int F, int W) {
    u128 nm1 = n - 1;
    u128 T = s2abs * nm1 * nm1;
    u128 X = G + T;
    int sh = F - W;
    u128 q = sh > 0 ? (X >> sh) + ((X & (((u128)1 << sh) - 1)) != 0) : X;
    return q + n + 1;
}

typedef struct {
    u128 a, b, eps;
} bprob;

/* _boolean_problem (pipeline.py:149-175) from residues s0, s1 (full ints) */
static bprob boolean_problem(const big* s0, const big* s1, u128 pad, int F, int W) {
    u128 m = mask_f(F);
    u128 s0m = big_lo128(s0) & m;
    u128 s1m = (((u128)0 - big_lo128(s1))) & m; /* (-s1) mod 2^F */
    u128 wmask = W >= 128 ? ~(u128)0 : (((u128)1 << W) - 1);
    bprob r;
    /* (s << W) >> F  ==  s >> (F - W) for F >= W */
    r.b = ((s0m >> (F - W)) + pad) & wmask;
    r.a = s1m >> (F - W);
    r.eps = 2 * pad;
    return r;
}

/* per-domain full coefficients of super-domain t via the reference packet
 * walk; returns the values for domain index i (and flags overflow seen
 * anywhere in the walk up to i) -- used for phase 1 sequentially. */
typedef struct {
    big col[3][3]; /* col[j][l]: Delta^l r_j at current i */
} walk_t;

/*
 * Phase 1 over the slice: tabulated walk (generate_packets order), boolean
 * problem, search; failing global domain ids ascending (pipeline.py:213-231).
 * Returns the number of failures written (<= cap), or -1 on MPInt overflow,
 * -2 on capacity exhaustion.  coef_out (optional, may be NULL) receives the
 * per-domain residues s_j mod 2^128 as [3][2][n_total] u64 (for parity).
 */
int64_t or_phase1(const slice_t* s, int algo, int mode, uint64_t* fail_ids, int64_t cap,
                  uint64_t* coef_out, int64_t n_total) {
    int64_t S = s->S;
    int deg_r[3] = {s->delta, s->delta - 1, s->delta - 2};
    int nt = or_get_threads();
    int64_t* counts = (int64_t*)calloc((size_t)S, sizeof(int64_t));
    uint64_t** lists = (uint64_t**)calloc((size_t)S, sizeof(uint64_t*));
    int ovf_any = 0;
    int64_t* dom_base = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1));
    dom_base[0] = 0;
    for (int64_t t = 0; t < S; t++) dom_base[t + 1] = dom_base[t] + s->n_dom[t];
    u128 one = (u128)1 << s->W;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt) reduction(| : ovf_any)
    for (int64_t t = 0; t < S; t++) {
        big r[3][3];
        memset(r, 0, sizeof r);
        for (int j = 0; j <= s->delta; j++)
            for (int l = 0; l <= deg_r[j]; l++) load_coef(s, t, (j == 0 ? 0 : j == 1 ? 3 : 5) + l, &r[j][l]);
        uint32_t tau = s->n_dom[t], nu = s->nu[t];
        uint32_t mu = (tau + nu - 1) / nu;
        u128 G = ((u128)s->G[S + t] << 64) | s->G[t];
        u128 s2a = ((u128)s->s2abs[S + t] << 64) | s->s2abs[t];
        uint64_t* list = (uint64_t*)malloc(sizeof(uint64_t) * (tau ? tau : 1));
        int64_t nf = 0;
        int ovf = 0;
        big vals[3];
        /* the reference walks j outer, u, i inner; values are independent of
         * that order, so walk u outer and all j together */
        for (uint32_t u = 0; u < mu; u++) {
            big col[3][3];
            for (int j = 0; j <= s->delta; j++) shift_poly(col[j], r[j], deg_r[j], (uint64_t)u * nu, s->L, &ovf);
            for (uint32_t i = 0; i < nu; i++) {
                if (i) {
                    for (int j = 0; j <= s->delta; j++)
                        for (int l = 0; l < deg_r[j]; l++) {
                            big_add(&col[j][l], &col[j][l], &col[j][l + 1]);
                            if (big_overflows(&col[j][l], s->L)) ovf = 1;
                        }
                }
                uint64_t idx = (uint64_t)u * nu + i;
                if (idx >= tau) continue; /* reference sets[] has exactly tau rows */
                for (int j = 0; j < 3; j++) {
                    if (j <= s->delta) vals[j] = col[j][0];
                    else memset(&vals[j], 0, sizeof(big));
                }
                uint64_t n = idx == tau - 1 ? s->last_n[t] : s->dom_n[t];
                u128 pad = pad_of(G, s->delta >= 2 ? s2a : 0, n, s->F, s->W);
                bprob bp = boolean_problem(&vals[0], &vals[1], pad, s->F, s->W);
                core_out o = run_core(algo, mode, bp.a, bp.b, bp.eps, n, one);
                if (!o.ok) list[nf++] = s->dom_id0[t] + idx;
                if (coef_out) {
                    int64_t g = dom_base[t] + (int64_t)idx;
                    for (int j = 0; j < 3; j++) {
                        u128 lo = big_lo128(&vals[j]);
                        coef_out[((int64_t)j * 2 + 0) * n_total + g] = (uint64_t)lo;
                        coef_out[((int64_t)j * 2 + 1) * n_total + g] = (uint64_t)(lo >> 64);
                    }
                }
            }
        }
        counts[t] = nf;
        lists[t] = list;
        ovf_any |= ovf;
    }
    int64_t total = 0;
    int full = 0;
    for (int64_t t = 0; t < S; t++) {
        for (int64_t k = 0; k < counts[t]; k++) {
            if (total < cap) fail_ids[total] = lists[t][k];
            else full = 1;
            total++;
        }
        free(lists[t]);
    }
    free(lists);
    free(counts);
    free(dom_base);
    if (ovf_any) return -1;
    if (full) return -2;
    return total;
}

/* locate super-domain of a global domain id (dom_id0 ascending) */
static int64_t find_super(const slice_t* s, uint64_t id) {
    int64_t lo = 0, hi = s->S - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (s->dom_id0[mid] <= id) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

/* full coefficients (s0, s1, s2) of domain i of super-domain t: the domain
 * polynomial P_{t+i} = straightforward_shift of each r_j to i (values equal
 * the tabulated walk exactly). */
static void domain_coeffs(const slice_t* s, int64_t t, uint64_t i, big* vals, int* ovf) {
    int deg_r[3] = {s->delta, s->delta - 1, s->delta - 2};
    for (int j = 0; j < 3; j++) memset(&vals[j], 0, sizeof(big));
    for (int j = 0; j <= s->delta; j++) {
        big r[3], col[3];
        memset(r, 0, sizeof r);
        for (int l = 0; l <= deg_r[j]; l++) load_coef(s, t, (j == 0 ? 0 : j == 1 ? 3 : 5) + l, &r[l]);
        shift_poly(col, r, deg_r[j], i, s->L, ovf);
        vals[j] = col[0];
    }
}

/*
 * Phase 2 (pipeline.py:234-257): for each failing domain id (ascending),
 * split `split` ways, straightforward-shift the domain polynomial to each
 * subdomain start, re-test.  Output rows (domain id, sub index j, start, cnt)
 * plus the shifted residues mod 2^128 [3][2] per row.  Returns count, -1 on
 * overflow, -2 on capacity.
 */
int64_t or_phase2(const slice_t* s, int algo, int mode, int split, const uint64_t* ids, int64_t n_ids,
                  uint64_t* out_id, uint32_t* out_j, uint32_t* out_start, uint32_t* out_cnt,
                  uint64_t* out_res, int64_t cap) {
    int nt = or_get_threads();
    int64_t* counts = (int64_t*)calloc((size_t)(n_ids ? n_ids : 1), sizeof(int64_t));
    uint64_t** rows = (uint64_t**)calloc((size_t)(n_ids ? n_ids : 1), sizeof(uint64_t*));
    int ovf_any = 0;
    u128 one = (u128)1 << s->W;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt) reduction(| : ovf_any)
    for (int64_t k = 0; k < n_ids; k++) {
        int ovf = 0;
        uint64_t id = ids[k];
        int64_t t = find_super(s, id);
        uint64_t i = id - s->dom_id0[t];
        big vals[3];
        int ovf_dom = 0; /* already checked by the phase-1 walk */
        domain_coeffs(s, t, i, vals, &ovf_dom);
        uint64_t n = i == s->n_dom[t] - 1 ? s->last_n[t] : s->dom_n[t];
        uint64_t step = n / (uint64_t)split;
        if (step < 1) step = 1;
        u128 G = ((u128)s->G[s->S + t] << 64) | s->G[t];
        u128 s2a = ((u128)s->s2abs[s->S + t] << 64) | s->s2abs[t];
        uint64_t nsub = (n + step - 1) / step;
        uint64_t* row = (uint64_t*)malloc(sizeof(uint64_t) * 10 * (nsub ? nsub : 1));
        int64_t nr = 0;
        int deg = s->delta;
        for (uint64_t j = 0; j < nsub; j++) {
            uint64_t start = j * step;
            uint64_t cnt = n - start < step ? n - start : step;
            big sh[3];
            shift_poly(sh, vals, deg, start, s->L, &ovf);
            for (int l = deg + 1; l < 3; l++) memset(&sh[l], 0, sizeof(big));
            u128 pad = pad_of(G, deg >= 2 ? s2a : 0, cnt, s->F, s->W);
            bprob bp = boolean_problem(&sh[0], &sh[1], pad, s->F, s->W);
            core_out o = run_core(algo, mode, bp.a, bp.b, bp.eps, cnt, one);
            if (!o.ok) {
                uint64_t* r = row + 10 * nr;
                r[0] = id;
                r[1] = j;
                r[2] = start;
                r[3] = cnt;
                for (int l = 0; l < 3; l++) {
                    u128 lo = big_lo128(&sh[l]);
                    r[4 + 2 * l] = (uint64_t)lo;
                    r[5 + 2 * l] = (uint64_t)(lo >> 64);
                }
                nr++;
            }
        }
        counts[k] = nr;
        rows[k] = row;
        ovf_any |= ovf;
    }
    int64_t total = 0;
    int full = 0;
    for (int64_t k = 0; k < n_ids; k++) {
        for (int64_t r = 0; r < counts[k]; r++) {
            uint64_t* x = rows[k] + 10 * r;
            if (total < cap) {
                out_id[total] = x[0];
                out_j[total] = (uint32_t)x[1];
                out_start[total] = (uint32_t)x[2];
                out_cnt[total] = (uint32_t)x[3];
                for (int l = 0; l < 6; l++) out_res[6 * total + l] = x[4 + l];
            } else {
                full = 1;
            }
            total++;
        }
        free(rows[k]);
    }
    free(rows);
    free(counts);
    if (ovf_any) return -1;
    if (full) return -2;
    return total;
}

/*
 * Phase 3 (pipeline.py:260-293): exact second-order walk of each surviving
 * subdomain mod 2^F; emit arguments inside the eps' window.  Inputs are the
 * phase-2 rows.  Output: argument binade index, distance floored to 2^-64,
 * domain id, ascending by argument (input rows ascending).  Returns count or
 * -2 on capacity.
 */
int64_t or_phase3(const slice_t* s, int64_t n_rows, const uint64_t* row_id, const uint32_t* row_start,
                  const uint32_t* row_cnt, const uint64_t* row_res, uint64_t* out_m, uint64_t* out_dist,
                  uint64_t* out_id, int64_t cap) {
    int F = s->F;
    u128 m = mask_f(F);
    u128 oneF = F >= 128 ? 0 : ((u128)1 << F); /* F == 128 wraps to 0: handled by mask */
    int nt = or_get_threads();
    int64_t* counts = (int64_t*)calloc((size_t)(n_rows ? n_rows : 1), sizeof(int64_t));
    uint64_t** lists = (uint64_t**)calloc((size_t)(n_rows ? n_rows : 1), sizeof(uint64_t*));
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (int64_t r = 0; r < n_rows; r++) {
        uint64_t id = row_id[r];
        int64_t t = find_super(s, id);
        uint64_t i = id - s->dom_id0[t];
        u128 G = ((u128)s->G[s->S + t] << 64) | s->G[t];
        u128 window = G + 1;
        const uint64_t* res = row_res + 6 * r;
        u128 v = (((u128)res[1] << 64) | res[0]) & m;
        u128 d1 = (((u128)res[3] << 64) | res[2]) & m;
        u128 d2 = (((u128)res[5] << 64) | res[4]) & m;
        uint64_t cnt = row_cnt[r];
        uint64_t base = s->m0[t] + i * (uint64_t)s->dom_n[t] + row_start[r];
        int64_t cap_l = 16, nl = 0;
        uint64_t* l = (uint64_t*)malloc(sizeof(uint64_t) * 3 * (size_t)cap_l);
        for (uint64_t x = 0; x < cnt; x++) {
            if (v < window || v > ((oneF - window) & m)) {
                u128 comp = (oneF - v) & m; /* 2^F - v for v in (0, 2^F) */
                u128 dist = (v == 0 || v < comp) ? v : comp;
                uint64_t d64 = F >= 64 ? (uint64_t)(dist >> (F - 64)) : (uint64_t)(dist << (64 - F));
                if (nl == cap_l) {
                    cap_l *= 2;
                    l = (uint64_t*)realloc(l, sizeof(uint64_t) * 3 * (size_t)cap_l);
                }
                l[3 * nl] = base + x;
                l[3 * nl + 1] = d64;
                l[3 * nl + 2] = id;
                nl++;
            }
            v = (v + d1) & m;
            d1 = (d1 + d2) & m;
        }
        counts[r] = nl;
        lists[r] = l;
    }
    int64_t total = 0;
    int full = 0;
    for (int64_t r = 0; r < n_rows; r++) {
        for (int64_t k = 0; k < counts[r]; k++) {
            if (total < cap) {
                out_m[total] = lists[r][3 * k];
                out_dist[total] = lists[r][3 * k + 1];
                out_id[total] = lists[r][3 * k + 2];
            } else {
                full = 1;
            }
            total++;
        }
        free(lists[r]);
    }
    free(lists);
    free(counts);
    if (full) return -2;
    return total;
}

/* flat-argument wrappers for ctypes (slice passed field by field) */
#define SLICE_ARGS                                                                                  \
    int64_t S, int CL, int L, int F, int W, int delta, const uint32_t *coef, const uint64_t *G,      \
        const uint64_t *s2abs, const uint32_t *n_dom, const uint32_t *dom_n, const uint32_t *last_n, \
        const uint32_t *nu, const uint64_t *dom_id0, const uint64_t *m0
#define SLICE_INIT                                                                                 \
    slice_t s = {S, CL, L, F, W, delta, coef, G, s2abs, n_dom, dom_n, last_n, nu, dom_id0, m0};

int64_t or_phase1_flat(SLICE_ARGS, int algo, int mode, uint64_t* fail_ids, int64_t cap, uint64_t* coef_out,
                       int64_t n_total) {
    SLICE_INIT
    return or_phase1(&s, algo, mode, fail_ids, cap, coef_out, n_total);
}

int64_t or_phase2_flat(SLICE_ARGS, int algo, int mode, int split, const uint64_t* ids, int64_t n_ids,
                       uint64_t* out_id, uint32_t* out_j, uint32_t* out_start, uint32_t* out_cnt,
                       uint64_t* out_res, int64_t cap) {
    SLICE_INIT
    return or_phase2(&s, algo, mode, split, ids, n_ids, out_id, out_j, out_start, out_cnt, out_res, cap);
}

int64_t or_phase3_flat(SLICE_ARGS, int64_t n_rows, const uint64_t* row_id, const uint32_t* row_start,
                       const uint32_t* row_cnt, const uint64_t* row_res, uint64_t* out_m, uint64_t* out_dist,
                       uint64_t* out_id, int64_t cap) {
    SLICE_INIT
    return or_phase3(&s, n_rows, row_id, row_start, row_cnt, row_res, out_m, out_dist, out_id, cap);
}

/* the (a, b, eps) of the Boolean problem for given residues and pad inputs
 * (exposed so tests can pin the closed-form pad against Fraction arithmetic) */
void or_boolean_problem(uint64_t s0_lo, uint64_t s0_hi, uint64_t s1_lo, uint64_t s1_hi, uint64_t G_lo,
                        uint64_t G_hi, uint64_t s2_lo, uint64_t s2_hi, uint64_t n, int F, int W,
                        uint64_t* out3) {
    big s0, s1;
    memset(&s0, 0, sizeof s0);
    memset(&s1, 0, sizeof s1);
    u128 v0 = ((u128)s0_hi << 64) | s0_lo, v1 = ((u128)s1_hi << 64) | s1_lo;
    for (int i = 0; i < 4; i++) {
        s0.w[i] = (uint32_t)(v0 >> (32 * i));
        s1.w[i] = (uint32_t)(v1 >> (32 * i));
    }
    u128 pad = pad_of(((u128)G_hi << 64) | G_lo, ((u128)s2_hi << 64) | s2_lo, n, F, W);
    bprob bp = boolean_problem(&s0, &s1, pad, F, W);
    out3[0] = (uint64_t)bp.a;
    out3[1] = (uint64_t)bp.b;
    out3[2] = (uint64_t)bp.eps;
    out3[3] = (uint64_t)(bp.eps >> 64);
}
