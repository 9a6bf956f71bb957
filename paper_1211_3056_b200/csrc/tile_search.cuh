// tile_search.cuh -- throughput form of the regular search for the phases.
//
// A warp owns a tile of 32*NU work items (lane l takes items l, l+32, ...).
// Each lane advances TWO searches in lockstep (items k and k+1): two
// independent dependency chains per thread hide the MUFU / conversion
// latencies of the quotient estimates, while the regular algorithm's nearly
// constant iteration count (NMDM 0.1%) keeps the 64
// searches of a warp in step.  Each half-step is straight-line code: the
// (p, q) roles alternate between two fixed registers, quotients come from
// one FP32 reciprocal with round-down estimates, and every correction (a
// near-integer estimate, a quotient >= 2^20, the first step's divisor above
// 2^63) is taken by the whole warp on one vote-gated exact path; the loop
// branches are warp-uniform.
//
// Restates _regular_core (lowerbound.py:228-267) bit-exactly for the
// verdict, d and the iteration count, for counts N < 2^32 (always true on
// the pipeline path: domain and subdomain sizes are 32-bit).
#pragma once
#include <stdint.h>

#include "search_core.cuh"

namespace hrb {

// One search in flight.  The reference's (p, q) pair lives in two fixed
// registers A, B whose roles alternate: before each else-half A is the
// divisor (S) and B the dividend (L); the else-half replaces B by B mod A,
// the following then-half replaces A by A mod B.  A loop iteration is one
// (else, then) pair, so the state returns to the same registers with no
// role-swap moves.  cA, cB are the matching point counts; Af, Bf the values
// rounded to float (used only for quotient estimates).
struct Slot {
    uint64_t A, B, d;
    float Af, Bf;
    uint32_t cA, cB;
};

// floor(y/x + e) from the FP32 reciprocal in one round-down FFMA: with
// M = 1.5 * 2^23, y*rcp + M rounded toward -inf lands on the integer grid of
// [2^23, 2^24), i.e. M + floor(y*rcp) while y*rcp < 2^22.  The error of
// y*rcp against y/x is |e| < 2^-21 y/x, so for y/x < 2^20 the result is
// floor(y/x) except when y/x lies within |e| of an integer: then it can be
// off by one either way, which the caller detects (remainder outside [0, x))
// and repairs on its rare exact path.
__device__ __forceinline__ int32_t qfloor(float yf, float rcp) {
    const float kf = __fmaf_rd(yf, rcp, 12582912.0f);
    return (int32_t)(__float_as_uint(kf) - 0x4B400000u);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // <= 1 ulp
    return r;
}

constexpr int32_t QMAX = 1 << 20;

// One half-step, fast path: Lp = L mod S with its quotient k, and the
// reduced d, from one FP32 reciprocal of S and round-down quotient estimates
// that are exact except in rare near-integer cases.  THEN selects the
// reference's `p < q` body (d %= p) versus the `p >= q` body (d reduced past
// the new p; when d < Lp, d < S already and the mod is the identity).
// `bad` flags a step the estimates may have got wrong -- a remainder outside
// [0, S) or a quotient >= 2^20 -- which hs_exact redoes; nothing is fixed up
// on the fast path.  Invariants on an active slot: S < L, d < L, S <= 2^63.
//
// FIRST: the first step of a search, the only one whose divisor (a) may
// exceed 2^63 and whose dividend (one - a) may be below it.  Its quotient
// estimate is clamped at 0 and a wrapped subtraction is caught directly
// (result above its minuend), since ">= S" no longer implies a wrap there.
template <bool THEN, bool FIRST = false>
__device__ __forceinline__ void hs_fast(uint64_t L, uint64_t S, float Lf, float Sf, uint64_t d, uint64_t& Lp,
                                        uint64_t& dn, uint32_t& k, bool& bad) {
    const float rcp = rcp_approx(Sf);
    // floor(L/S) >= 1 except on a first step, so the estimate is >= 0
    const int32_t ke = FIRST ? max(qfloor(Lf, rcp), 0) : qfloor(Lf, rcp);
    const uint64_t r = L - (uint64_t)(uint32_t)ke * S;
    uint64_t x = d;
    if (!THEN && x >= r) x -= r;
    // the quotient of x by S is >= 0; an estimate of -1 (x/S within |e| of
    // 0 from above) is clamped to 0, which is then exact
    const uint32_t ke2 = (uint32_t)max(qfloor(__ull2float_rn(x), rcp), 0);
    const uint64_t y = x - (uint64_t)ke2 * S;
    bad = (ke >= QMAX) | (r >= S) | (y >= S);
    if (FIRST) bad |= (r > L) | (y > x);
    Lp = r;
    dn = y;
    k = (uint32_t)ke;
}

// The same half-step with hardware 64-bit division (rare: a quotient >= 2^20
// or an estimate that missed by one).
// k saturates at 2^32 - 1: any quotient that large ends the search (cS >= 1
// makes cLp >= 2^32 - 1 >= N - cS), exactly as the reference's u + v >= N.
// Out of line and by value, so the hot loop keeps its registers.
struct ExactStep {
    uint64_t Lp, dn;
    uint32_t k;
};

__device__ __noinline__ ExactStep hs_exact(uint64_t L, uint64_t S, uint64_t d, bool then_body) {
    ExactStep e;
    const uint64_t kk = L / S;
    e.Lp = L - kk * S;
    const uint64_t x = (!then_body && d >= e.Lp) ? d - e.Lp : d;
    e.dn = x % S;
    e.k = kk > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)kk;
    return e;
}

// Commit a half-step in place (L <- Lp, cL <- k cS + cL, d <- dn) and report
// whether the search ended: expansion exhausted (Lp == 0) or the count
// reaches N.  A finished slot keeps computing harmless garbage.
__device__ __forceinline__ bool hs_commit(uint64_t& L, float& Lf, uint32_t& cL, uint32_t cS, uint64_t& d, uint32_t N,
                                          uint64_t Lp, uint64_t dn, uint32_t k) {
    const uint64_t cLp = (uint64_t)k * cS + cL;
    const bool done = Lp == 0 || cLp >= (uint64_t)(N - cS);
    L = Lp;
    Lf = __ull2float_rn(Lp);
    cL = (uint32_t)cLp;
    d = dn;
    return done;
}

// Both slots of a lane advance one half-step: the else-half divides B by A,
// the then-half A by B.  Must be called by all 32 lanes of the warp
// (warp-uniform control flow): the rare exact path is entered by the whole
// warp through one vote, so the hot path carries no divergent branch.
//
// FIRST marks the first then-half of a search (see hs_fast).
template <bool THEN, bool FIRST = false>
__device__ __forceinline__ void pair_step(Slot& s0, Slot& s1, uint32_t n0, uint32_t n1, bool act0, bool act1,
                                          bool& f0, bool& f1) {
    uint64_t& L0 = THEN ? s0.A : s0.B;
    uint64_t& L1 = THEN ? s1.A : s1.B;
    const uint64_t S0 = THEN ? s0.B : s0.A, S1 = THEN ? s1.B : s1.A;
    float& Lf0 = THEN ? s0.Af : s0.Bf;
    float& Lf1 = THEN ? s1.Af : s1.Bf;
    const float Sf0 = THEN ? s0.Bf : s0.Af, Sf1 = THEN ? s1.Bf : s1.Af;
    uint32_t& cL0 = THEN ? s0.cA : s0.cB;
    uint32_t& cL1 = THEN ? s1.cA : s1.cB;
    const uint32_t cS0 = THEN ? s0.cB : s0.cA, cS1 = THEN ? s1.cB : s1.cA;
    uint64_t Lp0, dn0, Lp1, dn1;
    uint32_t k0, k1;
    bool b0, b1;
    hs_fast<THEN, FIRST>(L0, S0, Lf0, Sf0, s0.d, Lp0, dn0, k0, b0);
    hs_fast<THEN, FIRST>(L1, S1, Lf1, Sf1, s1.d, Lp1, dn1, k1, b1);
    b0 = b0 && act0;
    b1 = b1 && act1;
    if (__any_sync(0xffffffffu, b0 || b1)) {
        if (b0) {
            const ExactStep e = hs_exact(L0, S0, s0.d, THEN);
            Lp0 = e.Lp, dn0 = e.dn, k0 = e.k;
        }
        if (b1) {
            const ExactStep e = hs_exact(L1, S1, s1.d, THEN);
            Lp1 = e.Lp, dn1 = e.dn, k1 = e.k;
        }
    }
    f0 = hs_commit(L0, Lf0, cL0, cS0, s0.d, n0, Lp0, dn0, k0);
    f1 = hs_commit(L1, Lf1, cL1, cS1, s1.d, n1, Lp1, dn1, k1);
}

// Set up a slot for _regular_core (lowerbound.py:228-267).  Returns true if
// the search ends before its loop (b < eps; a == 0 or N <= 1: 0 iterations)
// with *ok, *dout set.  Otherwise the slot holds (one - a, a) with counts
// (1, 1): its first then-half divides one - a by a, which yields the
// reference's first quotient floor(one / a) minus one, the count k + 1 and
// the remainder one mod a -- the whole first iteration on the lockstep path
// (no 65-bit `one` needed).
template <int W>
__device__ __forceinline__ bool slot_init(uint64_t a, uint64_t b, uint64_t eps, uint32_t N, Slot& s, bool* ok,
                                          uint64_t* dout) {
    if (b < eps) {
        *ok = false;
        *dout = b;
        return true;
    }
    if (a == 0 || N <= 1) {
        *ok = b > eps;
        *dout = b;
        return true;
    }
    s.A = (W == 64) ? (0ull - a) : ((1ull << 32) - a);
    s.B = a;
    s.d = b;
    s.Af = __ull2float_rn(s.A);
    s.Bf = __ull2float_rn(a);
    s.cA = 1;
    s.cB = 1;
    return false;
}

// All items of one lane, two searches at a time in lockstep.
//   src.build(k, a, b, eps, N) builds item k; called for k = 0, 1, 2, ... in
//   order, exactly once each; returns false for an invalid item.
//   src.done(k, ok, d, iterations) reports each valid item's outcome (the
//   phase kernels ignore it; the verdict batch stores it).
// Returns the lane's failure bits (bit k = item k failed) and adds the
// items' iteration counts (halved and rounded up for the unrolled variant)
// to *iters.
//
// Must be called by all 32 lanes of a warp: the item and step loops run to the
// warp's maximum (items past a lane's own count build as invalid), which keeps
// the vote in pair_step legal and the loop branches uniform.
template <int W, int NU, class Src>
__device__ __forceinline__ uint32_t lane_items(Src& src, unsigned long long* iters, bool halve, uint32_t n_items = NU) {
    uint32_t fails = 0, its = 0;
    const uint32_t mine = n_items < (uint32_t)NU ? n_items : (uint32_t)NU;
    const int kend = (int)__reduce_max_sync(0xffffffffu, mine);
#pragma unroll 1
    for (int k = 0; k < kend; k += 2) {
        Slot s0, s1;
        uint64_t a, b, e0 = 0, e1 = 0;
        uint32_t n0 = 0, n1 = 0;
        bool ok, act0 = false, act1 = false;
        uint64_t d_early;
        if (src.build(k, a, b, e0, n0)) {
            if (slot_init<W>(a, b, e0, n0, s0, &ok, &d_early)) {
                fails |= ok ? 0u : 1u << k;
                src.done(k, ok, d_early, 0);
            } else {
                act0 = true;
            }
        }
        if (src.build(k + 1, a, b, e1, n1)) {
            if (slot_init<W>(a, b, e1, n1, s1, &ok, &d_early)) {
                fails |= ok ? 0u : 2u << k;
                src.done(k + 1, ok, d_early, 0);
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
        {  // iteration 1: the then-half against one (see slot_init)
            bool f0, f1;
            pair_step<true, true>(s0, s1, n0, n1, act0, act1, f0, f1);
            if (act0 && f0) {
                its += 1;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                src.done(k, s0.d > e0, s0.d, 1);
                act0 = false;
            }
            if (act1 && f1) {
                its += 1;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                src.done(k + 1, s1.d > e1, s1.d, 1);
                act1 = false;
            }
        }
        uint32_t h = 1;  // half-steps so far (both slots start after their first then-half)
        while (__any_sync(0xffffffffu, act0 || act1)) {
            bool f0, f1;
            pair_step<false>(s0, s1, n0, n1, act0, act1, f0, f1);
            h++;
            if (act0 && f0) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                src.done(k, s0.d > e0, s0.d, halve ? (h + 1) >> 1 : h);
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                src.done(k + 1, s1.d > e1, s1.d, halve ? (h + 1) >> 1 : h);
                act1 = false;
            }
            pair_step<true>(s0, s1, n0, n1, act0, act1, f0, f1);
            h++;
            if (act0 && f0) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s0.d > e0) ? 0u : 1u << k;
                src.done(k, s0.d > e0, s0.d, halve ? (h + 1) >> 1 : h);
                act0 = false;
            }
            if (act1 && f1) {
                its += halve ? (h + 1) >> 1 : h;
                fails |= (s1.d > e1) ? 0u : 2u << k;
                src.done(k + 1, s1.d > e1, s1.d, halve ? (h + 1) >> 1 : h);
                act1 = false;
            }
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
