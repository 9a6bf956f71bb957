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
// role-swap moves.  cA, cB are the matching point counts and M the budget
// left, N - cA - cB (>= 0 while the search runs); Af, Bf the values rounded
// to float (quotient estimates, and the fast path's r < S and L == 0 tests).
struct Slot {
    uint64_t A, B, d;
    float Af, Bf;
    uint32_t cA, cB, M;
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

// x - y and whether it did not borrow (x >= y), from one carry chain: the
// comparison the else-half needs comes free with the subtraction.
__device__ __forceinline__ uint64_t sub_nb(uint64_t x, uint64_t y, bool& ge) {
    uint32_t lo, hi, c;
    asm("sub.cc.u32 %0, %3, %5;\n\t"
        "subc.cc.u32 %1, %4, %6;\n\t"
        "subc.u32 %2, 0, 0;"
        : "=r"(lo), "=r"(hi), "=r"(c)
        : "r"((uint32_t)x), "r"((uint32_t)(x >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32)));
    ge = c == 0;
    return ((uint64_t)hi << 32) | lo;
}

constexpr int32_t QMAX = 1 << 20;

// x + k * y mod 2^64 for a 32-bit k.  With y = -S precomputed once per
// half-step, both of its products (L - k S and x - k2 S) compile to one wide
// multiply-add on the low word and one multiply-add on the high word.
__device__ __forceinline__ uint64_t madd64(uint64_t x, uint32_t k, uint64_t y) { return x + (uint64_t)k * y; }

// One half-step, fast path: Lp = L mod S with its quotient k, and the
// reduced d, from one FP32 reciprocal of S and round-down quotient estimates
// that are exact except in rare near-integer cases.  THEN selects the
// reference's `p < q` body (d %= p) versus the `p >= q` body (d reduced past
// the new p; when d < Lp, d < S already and the mod is the identity).
// `bad` flags a step the estimates may have got wrong -- a remainder outside
// [0, S) or a quotient >= 2^20 -- which hs_redo redoes; nothing is fixed up
// on the fast path.  r < S is proved in float: rounding is monotone, so
// float(r) < float(S) implies r < S (equal floats are flagged, rarely and
// harmlessly).  Invariants on an active slot: S < L, d < L, S <= 2^63.
//
// FIRST: the first step of a search, the only one whose divisor (a) may
// exceed 2^63 and whose dividend (one - a) may be below it.  Its quotient
// estimate is clamped at 0 and a wrapped subtraction is caught directly
// (result above its minuend), since ">= S" no longer implies a wrap there.
template <bool THEN, bool FIRST = false>
__device__ __forceinline__ void hs_fast(uint64_t& L, uint64_t S, float& Lf, float Sf, uint64_t& d, uint32_t& k,
                                        uint32_t& k2, bool& sub, bool& bad) {
    const float rcp = rcp_approx(Sf);
    // floor(L/S) >= 1 except on a first step, so the estimate is >= 0
    const int32_t ke = FIRST ? max(qfloor(Lf, rcp), 0) : qfloor(Lf, rcp);
    const uint64_t nS = 0 - S;
    const uint64_t r = madd64(L, (uint32_t)ke, nS);
    uint64_t x = d;
    if (THEN) {
        sub = false;
    } else {
        const uint64_t t = sub_nb(d, r, sub);
        x = sub ? t : d;
    }
    // the quotient of x by S is >= 0; an estimate of -1 (x/S within |e| of
    // 0 from above) is clamped to 0, which is then exact
    const uint32_t ke2 = (uint32_t)max(qfloor(__ull2float_rn(x), rcp), 0);
    const uint64_t y = madd64(x, ke2, nS);
    const float rf = __ull2float_rn(r);
    // 0 < r < S, proved in float by one product: (rf - Sf) rf < 0 exactly
    // when 0 < rf < Sf (rf = 0, rf >= Sf and an overflow to +inf all fail
    // it).  r == 0 -- the expansion exhausted, rare before the count limit --
    // is left to the exact path, whose commit ends the search.
    bad = (ke >= QMAX) | !(__fmul_rn(rf - Sf, rf) < 0.0f) | (y >= S);
    if (FIRST) bad |= (r > L) | (y > x);
    // in place: the old L and d are recoverable from (r, y, ke, ke2, sub)
    // on the exact path, so no copy of them stays live across the vote
    L = r;
    Lf = rf;
    d = y;
    k = (uint32_t)ke;
    k2 = ke2;
}

// The same half-step with hardware 64-bit division (rare: a quotient >= 2^20
// or an estimate that missed by one).
// k saturates at 2^32 - 1: any quotient that large ends the search (cS >= 1
// makes k cS >= 2^32 - 1 >= M), exactly as the reference's u + v >= N.
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

// Finish a half-step (L, Lf and d already updated): cL <- k cS + cL, and
// report whether the search ended: expansion exhausted (L == 0, i.e.
// Lf == 0) or the count reaches N, i.e. k cS >= M = N - cL - cS (the
// reference's u + v >= N).  The budget then shrinks by k cS.  A finished
// slot keeps computing harmless garbage.
__device__ __forceinline__ uint64_t mul_wide(uint32_t a, uint32_t b) {
    uint64_t p;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
    return p;
}

template <bool ZERO = true>
__device__ __forceinline__ bool hs_commit(float Lf, uint32_t& cL, uint32_t cS, uint32_t& M, uint32_t k) {
    const uint64_t P = mul_wide(k, cS);
    // ZERO = false: the fast loop's commit, where r == 0 was flagged bad
    const bool done = (ZERO && Lf == 0.0f) | (P >= M);
    cL += (uint32_t)P;
    M -= (uint32_t)P;
    return done;
}

// Undo hs_fast's in-place update (all arithmetic mod 2^64 is exact) and
// redo the half-step with hardware division.
__device__ __forceinline__ void hs_redo(uint64_t& L, uint64_t S, float& Lf, uint64_t& d, uint32_t& k, uint32_t k2,
                                        bool sub, bool then_body) {
    const uint64_t L_old = L + (uint64_t)k * S;
    const uint64_t d_old = d + (uint64_t)k2 * S + (sub ? L : 0);
    const ExactStep e = hs_exact(L_old, S, d_old, then_body);
    L = e.Lp;
    Lf = __ull2float_rn(e.Lp);
    d = e.dn;
    k = e.k;
}

// Both slots of a lane advance one half-step: the else-half divides B by A,
// the then-half A by B.  Must be called by all 32 lanes of the warp
// (warp-uniform control flow): the rare exact path is entered by the whole
// warp through one vote, so the hot path carries no divergent branch.
//
// FIRST marks the first then-half of a search (see hs_fast).
template <bool THEN, bool FIRST = false>
__device__ __forceinline__ void pair_step(Slot& s0, Slot& s1, bool act0, bool act1, bool& f0, bool& f1) {
    uint64_t& L0 = THEN ? s0.A : s0.B;
    uint64_t& L1 = THEN ? s1.A : s1.B;
    const uint64_t S0 = THEN ? s0.B : s0.A, S1 = THEN ? s1.B : s1.A;
    float& Lf0 = THEN ? s0.Af : s0.Bf;
    float& Lf1 = THEN ? s1.Af : s1.Bf;
    const float Sf0 = THEN ? s0.Bf : s0.Af, Sf1 = THEN ? s1.Bf : s1.Af;
    uint32_t& cL0 = THEN ? s0.cA : s0.cB;
    uint32_t& cL1 = THEN ? s1.cA : s1.cB;
    const uint32_t cS0 = THEN ? s0.cB : s0.cA, cS1 = THEN ? s1.cB : s1.cA;
    uint32_t k0, k1, q0, q1;
    bool b0, b1, u0, u1;
    hs_fast<THEN, FIRST>(L0, S0, Lf0, Sf0, s0.d, k0, q0, u0, b0);
    hs_fast<THEN, FIRST>(L1, S1, Lf1, Sf1, s1.d, k1, q1, u1, b1);
    b0 = b0 && act0;
    b1 = b1 && act1;
    if (__any_sync(0xffffffffu, b0 || b1)) {
        if (b0) hs_redo(L0, S0, Lf0, s0.d, k0, q0, u0, THEN);
        if (b1) hs_redo(L1, S1, Lf1, s1.d, k1, q1, u1, THEN);
    }
    f0 = hs_commit(Lf0, cL0, cS0, s0.M, k0);
    f1 = hs_commit(Lf1, cL1, cS1, s1.M, k1);
}

// The lockstep loop's two building blocks.  fast_pair advances both slots
// by one half-step in place and votes: it returns true when some active
// lane's estimate may be wrong, in which case the caller leaves the loop
// (no commit) and finishes the pair on the exact path -- keeping every
// repair out of the loop body, whose registers then never merge with it.
template <bool THEN>
__device__ __forceinline__ bool fast_pair(Slot& s0, Slot& s1, bool act0, bool act1, uint32_t& k0, uint32_t& k1,
                                          uint32_t& q0, uint32_t& q1, bool& u0, bool& u1, bool& b0, bool& b1) {
    uint64_t& L0 = THEN ? s0.A : s0.B;
    uint64_t& L1 = THEN ? s1.A : s1.B;
    hs_fast<THEN>(L0, THEN ? s0.B : s0.A, THEN ? s0.Af : s0.Bf, THEN ? s0.Bf : s0.Af, s0.d, k0, q0, u0, b0);
    hs_fast<THEN>(L1, THEN ? s1.B : s1.A, THEN ? s1.Af : s1.Bf, THEN ? s1.Bf : s1.Af, s1.d, k1, q1, u1, b1);
    b0 = b0 && act0;
    b1 = b1 && act1;
    return __any_sync(0xffffffffu, b0 || b1);
}

template <bool THEN>
__device__ __forceinline__ bool commit_slot(Slot& s, uint32_t k) {
    return THEN ? hs_commit<false>(s.Af, s.cA, s.cB, s.M, k) : hs_commit<false>(s.Bf, s.cB, s.cA, s.M, k);
}

// One exact half-step of parity `th` from a slot's committed state.
__device__ __forceinline__ bool exact_half(Slot& s, bool th) {
    if (th) {
        const ExactStep e = hs_exact(s.A, s.B, s.d, true);
        s.A = e.Lp;
        s.Af = __ull2float_rn(e.Lp);
        s.d = e.dn;
        return hs_commit(s.Af, s.cA, s.cB, s.M, e.k);
    }
    const ExactStep e = hs_exact(s.B, s.A, s.d, false);
    s.B = e.Lp;
    s.Bf = __ull2float_rn(e.Lp);
    s.d = e.dn;
    return hs_commit(s.Bf, s.cB, s.cA, s.M, e.k);
}

// Rare path: repair the half-step of parity `th` that fast_pair left
// uncommitted (redo it exactly where it was flagged), commit it, then run
// the slot's search to its end with exact half-steps.  Returns the
// half-step count at the end.
__device__ __noinline__ uint32_t slow_finish(Slot& s, bool bad, uint32_t k, uint32_t q, bool u, bool th, uint32_t h) {
    uint64_t& L = th ? s.A : s.B;
    float& Lf = th ? s.Af : s.Bf;
    const uint64_t S = th ? s.B : s.A;
    if (bad) hs_redo(L, S, Lf, s.d, k, q, u, th);
    bool f = th ? hs_commit(s.Af, s.cA, s.cB, s.M, k) : hs_commit(s.Bf, s.cB, s.cA, s.M, k);
    h++;
    while (!f) {
        th = !th;
        f = exact_half(s, th);
        h++;
    }
    return h;
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
    s.M = N - 2;  // N >= 2 here
    return false;
}

// All items of one lane, two searches at a time in lockstep.
//   src.build2(k, ...) builds items k and k + 1 (k = 0, 2, 4, ... in order,
//   exactly once each) and flags each valid or not.
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
    Slot s0 = {}, s1 = {};
    // a slot whose search ended after h half-steps: record its outcome
    auto finish = [&](int item, const Slot& s, uint64_t e, uint32_t h) {
        const uint32_t it = halve ? (h + 1) >> 1 : h;
        its += it;
        fails |= (s.d > e) ? 0u : 1u << item;
        src.done(item, s.d > e, s.d, it);
    };
#pragma unroll 1
    for (int k = 0; k < kend; k += 2) {
        uint64_t ia0, ib0, ia1, ib1, e0 = 0, e1 = 0;
        uint32_t n0 = 0, n1 = 0;
        bool ok, v0, v1, act0 = false, act1 = false;
        uint64_t d_early;
        src.build2(k, v0, ia0, ib0, e0, n0, v1, ia1, ib1, e1, n1);
        if (v0) {
            if (slot_init<W>(ia0, ib0, e0, n0, s0, &ok, &d_early)) {
                fails |= ok ? 0u : 1u << k;
                src.done(k, ok, d_early, 0);
            } else {
                act0 = true;
            }
        }
        if (v1) {
            if (slot_init<W>(ia1, ib1, e1, n1, s1, &ok, &d_early)) {
                fails |= ok ? 0u : 2u << k;
                src.done(k + 1, ok, d_early, 0);
            } else {
                act1 = true;
            }
        }
        // An idle slot keeps whatever state it holds: its arithmetic may be
        // garbage (integer ops do not trap, and an idle slot's `bad` flag is
        // masked), so nothing is copied into it.
        {  // iteration 1: the then-half against one (see slot_init)
            bool f0, f1;
            pair_step<true, true>(s0, s1, act0, act1, f0, f1);
            f0 = f0 && act0;
            f1 = f1 && act1;
            if (f0) finish(k, s0, e0, 1);
            if (f1) finish(k + 1, s1, e1, 1);
            act0 = act0 && !f0;
            act1 = act1 && !f1;
        }
        uint32_t h = 1;  // half-steps so far (both slots start after their first then-half)
        int pending = 0;  // 1 / 2: left the loop with an uncommitted else- / then-half
        uint32_t k0, k1, q0, q1;
        bool u0, u1, b0, b1;
        while (__any_sync(0xffffffffu, act0 || act1)) {
            if (fast_pair<false>(s0, s1, act0, act1, k0, k1, q0, q1, u0, u1, b0, b1)) {
                pending = 1;
                break;
            }
            bool f0 = commit_slot<false>(s0, k0) && act0, f1 = commit_slot<false>(s1, k1) && act1;
            h++;
            if (f0 || f1) {  // one branch for both slots (rare: a search ends)
                if (f0) finish(k, s0, e0, h);
                if (f1) finish(k + 1, s1, e1, h);
                act0 = act0 && !f0;
                act1 = act1 && !f1;
            }
            if (fast_pair<true>(s0, s1, act0, act1, k0, k1, q0, q1, u0, u1, b0, b1)) {
                pending = 2;
                break;
            }
            f0 = commit_slot<true>(s0, k0) && act0;
            f1 = commit_slot<true>(s1, k1) && act1;
            h++;
            if (f0 || f1) {
                if (f0) finish(k, s0, e0, h);
                if (f1) finish(k + 1, s1, e1, h);
                act0 = act0 && !f0;
                act1 = act1 && !f1;
            }
        }
        if (pending) {  // rare (warp-uniform entry): finish the pair's searches exactly
            const bool th = pending == 2;
            if (act0) finish(k, s0, e0, slow_finish(s0, b0, k0, q0, u0, th, h));
            if (act1) finish(k + 1, s1, e1, slow_finish(s1, b1, k1, q1, u1, th, h));
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
