// tile_search.cuh -- throughput form of the regular search for the phases.
//
// A warp owns a tile of 32*NU work items (lane l takes items l, l+32, ...).
// Each lane advances TWO searches in lockstep (items k and k+1): two
// independent dependency chains per thread hide the FP64 / conversion
// latencies of the quotient estimate, while the regular algorithm's nearly
// constant iteration count (NMDM 0.1%) keeps the 64
// searches of a warp in step.  Each half-step is straight-line code: the
// role swap is unconditional (so the compiler renames instead of moving),
// the d-reduction offset is a select, and the only branches are one rarely
// taken exact-division fallback and the loop exit.
//
// Restates _regular_core (lowerbound.py:228-267) bit-exactly for the
// verdict, d and the iteration count, for counts N < 2^32 (always true on
// the pipeline path: domain and subdomain sizes are 32-bit).
#pragma once
#include <stdint.h>

#include "search_core.cuh"

namespace hrb {

constexpr double TWO32 = 4294967296.0;

__device__ __forceinline__ double rcp_refined(double xd) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(xd));
    double e = fma(-xd, r, 1.0);
    return fma(r, e, r);
}

// one search in flight, role form (see search_core.cuh RegState)
struct Slot {
    uint64_t S, L, d;
    float Sf, Lf;  // S, L rounded to float: only ever used for quotient estimates
    uint32_t cS, cL;
};

// Quotient estimate from the FP32 reciprocal: with M = 1.5 * 2^23 the FFMA
// y*rcp(x) + (M - 1) lands in [2^23, 2^24) where floats are the integers, so
// its single rounding IS round-to-nearest(y/x - 1 + e) with |e| < 2^-22 y/x;
// for y/x < 2^20 that is floor(y/x) or floor(y/x) - 1 (possibly -1 when the
// quotient is 0), read straight from the bit pattern -- no F2I on the
// conversion pipe.  Quotients >= 2^20 are reported for the exact path.
__device__ __forceinline__ int32_t qest(float yf, float rcp) {
    const float kf = fmaf(yf, rcp, 12582911.0f);  // 1.5 * 2^23 - 1
    return (int32_t)(__float_as_uint(kf) - 0x4B400000u);
}

// r = y - k x with k in {K-1, K} (K = floor(y/x)), fixed to the exact
// remainder; returns the exact quotient.  k = -1 (K = 0) is clamped to 0,
// where y < x already holds, so the products stay unsigned 32x64.
__device__ __forceinline__ uint32_t qfix(uint64_t y, uint64_t x, int32_t k, uint64_t& r) {
    const uint32_t ku = (uint32_t)max(k, 0);
    const uint64_t rr = y - (uint64_t)ku * x;
    const bool c = rr >= x;
    r = c ? rr - x : rr;
    return ku + (c ? 1u : 0u);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // <= 1 ulp
    return r;
}

constexpr int32_t QMAX = 1 << 20;

// One half-step; THEN selects the reference's `p < q` body (d %= p) versus
// the `p >= q` body (d reduced past the new p).  Returns true when the
// search ended (verdict d > eps); the state is advanced unconditionally, so
// a finished slot keeps computing harmless garbage.  Invariant S <= 2^63
// (S is a remainder of 2^W by a, or smaller).
template <bool THEN>
__device__ __forceinline__ bool half_step(Slot& s, uint32_t N) {
    const uint64_t S = s.S, L = s.L;
    const float rcp = rcp_approx(s.Sf);
    const int32_t ke = qest(s.Lf, rcp);
    uint64_t Lp;
    const uint32_t k = qfix(L, S, ke, Lp);
    uint64_t cLp = (uint64_t)k * s.cS + s.cL;
    // d reduction: then-body d mod S; else-body (d >= Lp ? d - Lp : d) mod S
    // (when d < Lp, d < S already and the mod is the identity)
    uint64_t x = (!THEN && s.d >= Lp) ? s.d - Lp : s.d;
    const int32_t ke2 = qest(__ull2float_rn(x), rcp);
    uint64_t dn;
    qfix(x, S, ke2, dn);
    if (ke >= QMAX || ke2 >= QMAX) {  // rare: a quotient >= 2^20 (exact path)
        const uint64_t kk = S ? L / S : 0;
        Lp = L - kk * S;
        cLp = kk * (uint64_t)s.cS + s.cL;  // true value <= 2^64; == 2^64 only if Lp == 0 and S == 1
        x = (!THEN && s.d >= Lp) ? s.d - Lp : s.d;
        dn = S ? x % S : x;
    }
    s.d = dn;
    const bool done = Lp == 0 || cLp >= (uint64_t)(N - s.cS);
    s.L = S;
    s.Lf = s.Sf;
    s.S = Lp;
    s.Sf = __ull2float_rn(Lp);
    s.cL = s.cS;
    s.cS = (uint32_t)cLp;
    return done;
}

// _regular_core up to and including the first (then-) half-step against
// one = 2^W.  Returns true if the search ended there (*ok, *it set);
// otherwise `s` holds the state before the first else-half.
template <int W>
__device__ __forceinline__ bool reg_start(uint64_t a, uint64_t b, uint64_t eps, uint32_t N, Slot& s, bool* ok,
                                          uint32_t* it) {
    if (b < eps) {
        *ok = false;
        *it = 0;
        return true;
    }
    if (a == 0 || N <= 1) {
        *ok = b > eps;
        *it = 0;
        return true;
    }
    // k = one / a, rem = one mod a (one = 2^W); the quotient is >= 1 since a < one
    const double ad = __ull2double_rn(a);
    const double inv = rcp_refined(ad);
    const double kd = fma(W == 64 ? 18446744073709551616.0 : 4294967296.0, inv, -0.5);
    uint64_t k, rem, d;
    if (kd < TWO32) {
        uint32_t k0 = __double2uint_rz(kd);
        k0 = k0 ? k0 : 1u;
        rem = (W == 64) ? (0ull - (uint64_t)k0 * a) : ((1ull << 32) - (uint64_t)k0 * a);
        const bool c = rem >= a;
        rem = c ? rem - a : rem;
        k = k0 + (c ? 1u : 0u);
        const double kd2 = fma(__ull2double_rn(b), inv, -0.5);
        if (kd2 < TWO32) {
            const uint32_t k2 = __double2uint_rz(kd2);
            d = b - (uint64_t)k2 * a;
            d = d >= a ? d - a : d;
        } else {
            d = b % a;
        }
    } else {
        if (W == 64 && a == 1) {  // k = 2^64: q -> 0, d = 0, exhausted
            *ok = false;
            *it = 1;
            return true;
        }
        if (W == 64) {
            const uint64_t k0 = ~0ull / a, r0 = ~0ull - k0 * a;
            k = (r0 == a - 1) ? k0 + 1 : k0;
            rem = (r0 == a - 1) ? 0 : r0 + 1;
        } else {
            k = (1ull << 32) / a;
            rem = (1ull << 32) - k * a;
        }
        d = b % a;
    }
    if (rem == 0 || k >= (uint64_t)N - 1) {
        *ok = d > eps;
        *it = 1;
        return true;
    }
    s.S = rem;
    s.L = a;
    s.d = d;
    s.Sf = __ull2float_rn(rem);
    s.Lf = __ull2float_rn(a);
    s.cS = (uint32_t)k;
    s.cL = 1;
    return false;
}

// All items of one lane, two searches at a time in lockstep.
//   src.build(k, a, b, eps, N) builds item k; called for k = 0, 1, 2, ... in
//   order, exactly once each; returns false for an invalid item.
// Returns the lane's failure bits (bit k = item k failed) and adds the
// items' iteration counts (halved and rounded up for the unrolled variant)
// to *iters.
template <int W, int NU, class Src>
__device__ __forceinline__ uint32_t lane_items(Src& src, unsigned long long* iters, bool halve, uint32_t n_items = NU) {
    uint32_t fails = 0, its = 0;
    const int kend = n_items < (uint32_t)NU ? (int)n_items : NU;
#pragma unroll 1
    for (int k = 0; k < kend; k += 2) {
        Slot s0, s1;
        uint64_t a, b, e0 = 0, e1 = 0;
        uint32_t n0 = 0, n1 = 0, it;
        bool ok, act0 = false, act1 = false;
        if (src.build(k, a, b, e0, n0)) {
            if (reg_start<W>(a, b, e0, n0, s0, &ok, &it)) {
                its += halve ? (it + 1) >> 1 : it;
                fails |= ok ? 0u : 1u << k;
            } else {
                act0 = true;
            }
        }
        if (src.build(k + 1, a, b, e1, n1)) {
            if (reg_start<W>(a, b, e1, n1, s1, &ok, &it)) {
                its += halve ? (it + 1) >> 1 : it;
                fails |= ok ? 0u : 2u << k;
            } else {
                act1 = true;
            }
        }
        if (!act0) {  // keep the idle chain's arithmetic well defined
            s0 = s1;
            n0 = n1;
        }
        if (!act1) {
            s1 = s0;
            n1 = n0;
        }
        uint32_t h = 1;  // half-steps so far (both slots start after their first then-half)
        while (act0 || act1) {
            bool f0 = half_step<false>(s0, n0);
            bool f1 = half_step<false>(s1, n1);
            h++;
            if (act0 && f0) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                act1 = false;
            }
            f0 = half_step<true>(s0, n0);
            f1 = half_step<true>(s1, n1);
            h++;
            if (act0 && f0) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                act1 = false;
            }
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
