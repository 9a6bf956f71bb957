// confirm.cuh -- the rigorous confirmation of phase-3 candidates on the
// device (decide_hr for exp, evalf.py:286-327 at the pipeline's start
// precision, pipeline.py:446-461).
//
// Two forms of the same computation:
//   confirm_exp_kernel       one thread per candidate runs csrc/host/decide.h
//                            -- the SAME source as the host library's
//                            hrbh_confirm (generic capacity, all precisions)
//   confirm_exp_fast_kernel  the first precision step only, in fixed-width
//                            registers (NL 64-bit limbs): mpmath's
//                            exp_basecase (libelefun.py:1086-1109) with its
//                            floor divisions by small k done by
//                            multiply-high with ceil(2^64 / k), then the
//                            from_man_exp rounding, the distance enclosure
//                            and the decision of decide.h.  Bit-identical
//                            steps; a candidate it cannot settle at that
//                            precision gets status 1 (the host continues
//                            with the doubled precision).
#include "host/decide.h"

__global__ void __launch_bounds__(128) confirm_exp_kernel(int precision, int eps_bits, int binade, int64_t n,
                                                          const uint64_t* index, uint8_t* is_hr, uint64_t* dist,
                                                          uint8_t* status) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t d = 0;
        const int r = hrbh::decide_exp(precision, eps_bits, binade, index[i], &d);
        status[i] = r < 0 ? 1 : 0;
        is_hr[i] = r == 1 ? 1 : 0;
        dist[i] = d;
    }
}

namespace fw {

// ceil(2^64 / d) for d = 2..127 (d = 1 is skipped by the callers)
__constant__ uint64_t c_inv[128];

template <int NL>
struct W {
    uint64_t w[NL];
};

template <int NL>
__device__ __forceinline__ W<NL> zero() {
    W<NL> r;
#pragma unroll
    for (int i = 0; i < NL; i++) r.w[i] = 0;
    return r;
}

template <int NL>
__device__ __forceinline__ bool is_zero(const W<NL>& a) {
    uint64_t o = 0;
#pragma unroll
    for (int i = 0; i < NL; i++) o |= a.w[i];
    return o == 0;
}

template <int NL>
__device__ __forceinline__ W<NL> pow2(int k) {
    W<NL> r;
#pragma unroll
    for (int i = 0; i < NL; i++) r.w[i] = (i == (k >> 6)) ? (1ull << (k & 63)) : 0;
    return r;
}

template <int NL>
__device__ __forceinline__ W<NL> add(const W<NL>& a, const W<NL>& b) {
    W<NL> r;
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        const uint64_t s = a.w[i] + b.w[i];
        const uint64_t c1 = s < a.w[i];
        r.w[i] = s + c;
        c = c1 | (r.w[i] < s);
    }
    return r;
}

template <int NL>
__device__ __forceinline__ W<NL> sub(const W<NL>& a, const W<NL>& b) {  // a >= b
    W<NL> r;
    uint64_t br = 0;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        const uint64_t d = a.w[i] - b.w[i];
        const uint64_t b1 = a.w[i] < b.w[i];
        r.w[i] = d - br;
        br = b1 | (d < br);
    }
    return r;
}

template <int NL>
__device__ __forceinline__ int cmp(const W<NL>& a, const W<NL>& b) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < NL; i++) c = a.w[i] != b.w[i] ? (a.w[i] < b.w[i] ? -1 : 1) : c;
    return c;
}

template <int NL>
__device__ __forceinline__ int bitlen(const W<NL>& a) {
    int b = 0;
#pragma unroll
    for (int i = 0; i < NL; i++) b = a.w[i] ? 64 * i + 64 - __clzll((long long)a.w[i]) : b;
    return b;
}

template <int NL>
__device__ __forceinline__ int tz(const W<NL>& a) {
    int t = 0;
    bool found = false;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        if (!found && a.w[i]) {
            t = 64 * i + __ffsll((long long)a.w[i]) - 1;
            found = true;
        }
    }
    return t;
}

// floor(a / 2^k), k >= 0 (register-resident: word offset by selects)
template <int NLI, int NLO>
__device__ __forceinline__ W<NLO> shr(const W<NLI>& a, int k) {
    const int q = k >> 6, s = k & 63;
    W<NLO> r;
#pragma unroll
    for (int i = 0; i < NLO; i++) {
        uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int j = 0; j < NLI; j++) {
            lo = (j == i + q) ? a.w[j] : lo;
            hi = (j == i + q + 1) ? a.w[j] : hi;
        }
        r.w[i] = s ? (lo >> s) | (hi << (64 - s)) : lo;
    }
    return r;
}

template <int NL>
__device__ __forceinline__ W<NL> shl(const W<NL>& a, int k) {  // a 2^k (fits by the caller's sizing)
    const int q = k >> 6, s = k & 63;
    W<NL> r;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int j = 0; j < NL; j++) {
            lo = (j == i - q) ? a.w[j] : lo;
            hi = (j == i - q - 1) ? a.w[j] : hi;
        }
        r.w[i] = s ? (lo << s) | (hi >> (64 - s)) : lo;
    }
    return r;
}

template <int NL>
__device__ __forceinline__ bool low_zero(const W<NL>& a, int k) {  // low k bits all zero
    bool z = true;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        const int lo = 64 * i;
        if (k >= lo + 64) z = z && a.w[i] == 0;
        else if (k > lo) z = z && (a.w[i] & ((1ull << (k - lo)) - 1)) == 0;
    }
    return z;
}

template <int NL>
__device__ __forceinline__ W<NL> low_bits(const W<NL>& a, int k) {
    W<NL> r;
#pragma unroll
    for (int i = 0; i < NL; i++) {
        const int lo = 64 * i;
        r.w[i] = k >= lo + 64 ? a.w[i] : (k > lo ? a.w[i] & ((1ull << (k - lo)) - 1) : 0);
    }
    return r;
}

// (a b) >> P, the product kept in 2 NL words
template <int NL>
__device__ __forceinline__ W<NL> mul_shr(const W<NL>& a, const W<NL>& b, int P) {
    W<2 * NL> p = zero<2 * NL>();
#pragma unroll
    for (int i = 0; i < NL; i++) {
        uint64_t c = 0;
#pragma unroll
        for (int j = 0; j < NL; j++) {
            const uint64_t lo = a.w[i] * b.w[j], hi = __umul64hi(a.w[i], b.w[j]);
            const uint64_t s1 = p.w[i + j] + lo;
            const uint64_t c1 = s1 < lo;
            const uint64_t s2 = s1 + c;
            const uint64_t c2 = s2 < c;
            p.w[i + j] = s2;
            c = hi + c1 + c2;
        }
        p.w[i + NL] = c;
    }
    return shr<2 * NL, NL>(p, P);
}

// floor(a / d), 2 <= d < 128: per 32-bit half, q = umulhi(cur, ceil(2^64/d))
// is exact for cur < d 2^32 (error < cur 2^-64 < 1/d)
template <int NL>
__device__ __forceinline__ W<NL> div_small(const W<NL>& a, uint32_t d) {
    const uint64_t m = c_inv[d];
    W<NL> r;
    uint64_t rem = 0;
#pragma unroll
    for (int i = NL - 1; i >= 0; i--) {
        uint64_t cur = (rem << 32) | (a.w[i] >> 32);
        uint64_t q1 = __umul64hi(cur, m);
        rem = cur - q1 * d;
        cur = (rem << 32) | (a.w[i] & 0xFFFFFFFFull);
        uint64_t q0 = __umul64hi(cur, m);
        rem = cur - q0 * d;
        r.w[i] = (q1 << 32) | q0;
    }
    return r;
}

// mpmath exp_basecase(x, wp) (libelefun.py:1086-1109), r = isqrt(wp)
template <int NL>
__device__ __forceinline__ W<NL> exp_basecase(const W<NL>& x, int wp, int r, bool* ok) {
    const int P = wp + r;
    W<NL> s0 = pow2<NL>(P), s1 = s0;
    const W<NL> x2 = mul_shr<NL>(x, x, P);
    W<NL> a = x2;
    uint32_t k = 2;
    *ok = true;
    while (!is_zero<NL>(a)) {
        if (k > 124) {  // beyond the reciprocal table (never at these precisions)
            *ok = false;
            break;
        }
        a = div_small<NL>(a, k);
        s0 = add<NL>(s0, a);
        k++;
        a = div_small<NL>(a, k);
        s1 = add<NL>(s1, a);
        k++;
        a = mul_shr<NL>(a, x2, P);
    }
    s1 = mul_shr<NL>(s1, x, P);
    W<NL> s = add<NL>(s0, s1);
    for (int i = 0; i < r; i++) s = mul_shr<NL>(s, s, P);
    return shr<NL, NL>(s, r);
}

// decide.h's dist_range
template <int NL>
__device__ __forceinline__ void dist_range(const W<NL>& off, const W<NL>& width, const W<NL>& grid, W<NL>* dlo,
                                           W<NL>* dhi) {
    const W<NL> end = add<NL>(off, width);
    const W<NL> half = shr<NL, NL>(grid, 1);
    if (cmp<NL>(end, grid) >= 0) {
        *dlo = zero<NL>();
        if (cmp<NL>(off, half) <= 0) {
            *dhi = half;
        } else {
            const W<NL> a = sub<NL>(grid, off), eg = sub<NL>(end, grid);
            const W<NL> b = cmp<NL>(eg, half) < 0 ? eg : half;
            *dhi = cmp<NL>(a, b) > 0 ? a : b;
        }
        return;
    }
    const W<NL> go = sub<NL>(grid, off), ge = sub<NL>(grid, end);
    const W<NL> d0 = cmp<NL>(off, go) < 0 ? off : go;
    const W<NL> d1 = cmp<NL>(end, ge) < 0 ? end : ge;
    *dlo = cmp<NL>(d0, d1) < 0 ? d0 : d1;
    *dhi = (cmp<NL>(off, half) <= 0 && cmp<NL>(half, end) <= 0) ? half : (cmp<NL>(d0, d1) > 0 ? d0 : d1);
}

__device__ __forceinline__ int den_bits_of(int tzm, int e) {
    const int ee = e + tzm;
    return ee >= 0 ? 1 : -ee + 1;
}

}  // namespace fw

// The first precision step of decide_exp in NL-limb registers.  The host
// sizes NL so that every value fits (P + 3 bits; see hrb_confirm_exp).
template <int NL>
__global__ void __launch_bounds__(128) confirm_exp_fast_kernel(int precision, int eps_bits, int binade, int prec,
                                                               int64_t n, const uint64_t* index, uint8_t* is_hr,
                                                               uint64_t* dist, uint8_t* status) {
    using namespace fw;
    const int p = precision;
    const int xe = binade + 1 - p;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t M = (1ull << (p - 1)) + index[i];
        int den_b;
        const int num_b = hrbh::reduced_bits(M, xe, &den_b);
        const int work = max(prec, max(num_b, den_b)) + 8;
        const int wp = work + 14;
        const int r = (int)hrbh::isqrt_u64((uint64_t)wp);
        const int tzM = __ffsll((long long)M) - 1;
        // t = X 2^wp (X < 2: no reduction; the host checked mag <= 1)
        W<NL> man = zero<NL>();
        man.w[0] = M >> tzM;
        const int offset = xe + tzM + wp;
        const W<NL> t = offset >= 0 ? shl<NL>(man, offset) : shr<NL, NL>(man, -offset);
        bool ok;
        const W<NL> m = exp_basecase<NL>(t, wp, r, &ok);
        // from_man_exp(m, -wp, work, floor / ceiling)
        const int bc = bitlen<NL>(m);
        const int nsh = bc > work ? bc - work : 0;
        const W<NL> fl = shr<NL, NL>(m, nsh);
        W<NL> one = zero<NL>();
        one.w[0] = 1;
        const W<NL> ce = (nsh && !low_zero<NL>(m, nsh)) ? add<NL>(fl, one) : fl;
        const int le = nsh - wp;
        uint8_t st = 1, hr = 0;
        uint64_t dd = 0;
        if (ok && cmp<NL>(fl, ce) != 0) {
            const int sc = max(max(den_bits_of(tz<NL>(fl), le), den_bits_of(tz<NL>(ce), le)), prec) + 4;
            const W<NL> nlo = le + sc >= 0 ? shl<NL>(fl, le + sc) : shr<NL, NL>(fl, -(le + sc));
            W<NL> nhi;
            if (le + sc >= 0) {
                nhi = shl<NL>(ce, le + sc);
            } else {
                const int k = -(le + sc);
                nhi = shr<NL, NL>(ce, k);
                if (!low_zero<NL>(ce, k)) nhi = add<NL>(nhi, one);
            }
            const int bl = bitlen<NL>(nlo);
            if (bl == bitlen<NL>(nhi)) {
                const int gbits = bl - p;  // sc + (bl - sc) - p
                if (gbits > 0) {
                    const W<NL> grid = pow2<NL>(gbits);
                    W<NL> dlo, dhi;
                    dist_range<NL>(low_bits<NL>(nlo, gbits), sub<NL>(nhi, nlo), grid, &dlo, &dhi);
                    const bool ge_eps_bits = gbits >= eps_bits;
                    const W<NL> epsg = pow2<NL>(ge_eps_bits ? gbits - eps_bits : 0);
                    const bool hi_lt = ge_eps_bits ? cmp<NL>(dhi, epsg) < 0 : is_zero<NL>(dhi);
                    const bool lo_lt = ge_eps_bits ? cmp<NL>(dlo, epsg) < 0 : is_zero<NL>(dlo);
                    if (hi_lt) {
                        const W<NL> rr = gbits >= 64 ? shr<NL, NL>(dlo, gbits - 64) : shl<NL>(dlo, 64 - gbits);
                        dd = rr.w[0];
                        hr = 1;
                        st = 0;
                    } else if (!lo_lt) {
                        st = 0;
                    }
                }
            }
        }
        status[i] = st;
        is_hr[i] = hr;
        dist[i] = dd;
    }
}
