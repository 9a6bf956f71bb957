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
    double Sd, Ld;
    uint32_t cS, cL, it;
};

// One half-step; THEN selects the reference's `p < q` body (d %= p) versus
// the `p >= q` body (d reduced past the new p).  Returns true when the
// search ended (verdict d > eps, iterations s.it); the state is advanced
// unconditionally, so a finished slot keeps computing harmless garbage.
template <bool THEN>
__device__ __forceinline__ bool half_step(Slot& s, uint32_t N) {
    const uint64_t S = s.S, L = s.L;
    const double inv = rcp_refined(s.Sd);
    // quotient of the continued fraction: estimate, then one fix-up
    const double kd = fma(s.Ld, inv, -0.5);
    uint32_t k = __double2uint_rz(kd);
    uint64_t Lp = L - (uint64_t)k * S;
    const bool c = Lp >= S;
    Lp = c ? Lp - S : Lp;
    k += c ? 1u : 0u;
    uint64_t cLp = (uint64_t)k * s.cS + s.cL;
    // d reduction: then-body d mod S; else-body (d >= Lp ? d - Lp : d) mod S
    // (when d < Lp, d < S already and the mod is the identity)
    uint64_t x = (!THEN && s.d >= Lp) ? s.d - Lp : s.d;
    const double kd2 = fma(__ull2double_rn(x), inv, -0.5);
    const uint32_t k2 = __double2uint_rz(kd2);
    uint64_t dn = x - (uint64_t)k2 * S;
    dn = dn >= S ? dn - S : dn;
    if (!(fmax(kd, kd2) < TWO32)) {  // rare: a quotient >= 2^32 (exact path)
        const uint64_t kk = S ? L / S : 0;
        Lp = L - kk * S;
        cLp = kk * (uint64_t)s.cS + s.cL;  // true value <= 2^64; == 2^64 only if Lp == 0 and S == 1
        x = (!THEN && s.d >= Lp) ? s.d - Lp : s.d;
        dn = S ? x % S : x;
    }
    s.d = dn;
    s.it++;
    const bool done = Lp == 0 || cLp >= (uint64_t)(N - s.cS);
    s.L = S;
    s.Ld = s.Sd;
    s.S = Lp;
    s.Sd = __ull2double_rn(Lp);
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
    s.Sd = __ull2double_rn(rem);
    s.Ld = ad;
    s.cS = (uint32_t)k;
    s.cL = 1;
    s.it = 1;
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
        while (act0 || act1) {
            bool f0 = half_step<false>(s0, n0);
            bool f1 = half_step<false>(s1, n1);
            if (act0 && f0) {
                its += halve ? (s0.it + 1) >> 1 : s0.it;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (s1.it + 1) >> 1 : s1.it;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                act1 = false;
            }
            f0 = half_step<true>(s0, n0);
            f1 = half_step<true>(s1, n1);
            if (act0 && f0) {
                its += halve ? (s0.it + 1) >> 1 : s0.it;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (s1.it + 1) >> 1 : s1.it;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                act1 = false;
            }
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
