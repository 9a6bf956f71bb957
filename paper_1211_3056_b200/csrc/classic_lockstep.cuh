// classic_lockstep.cuh -- throughput form of the classic (Lefevre) search
// for the phases: lowerbound.py:88-225 (_lefevre_core / _lefevre_swap_core,
// which agree on the full outcome, test_lowerbound.py:236-238) restated for
// warp-uniform control flow.
//
// Each lane runs TWO searches at a time (two dependency chains) over its
// items, and a slot whose search ends takes the lane's next item at once
// (the classic walk's iteration counts vary widely: NMDM ~20 %,
// PAPER.md:1653-1664).  Only the verdict and the per-mode iteration count
// are produced (what the phases read, pipeline.py:200-201, 228); the general
// core (search_core.cuh) keeps the full outcome for the search ABI.
//
// The step is the swap form (_lefevre_swap_core 166-225) as straight-line
// code:
//   if swapped: d -= q, a failure when d < eps
//   k = q // p;  success when k v >= M  (M = max(N - u - v, 0), the
//                reference's k >= ceil((N - u - v) / v))
//   q -= k p, u += k v;  success when q == 0
//   p -= q, v += u, M = max(M - k v - u, 0)
//   swap (p, q), (u, v) when d >= (swapped ? q : p) changes `swapped`.
// The batched plain-reduction loop of the reference (170-222) is the same
// state evolution as a run of swapped steps with k == 0 -- the loop runs
// while d >= q (the slot stays swapped) and q < p (the next k is 0) -- and
// differs only in its counting: the run's first step is a normal one, then
// mode 1 counts one more step and mode 2 none (mode 0 never batches).  A
// run counter in the slot (0, 1, 2+) reproduces that.
//
// The quotient comes from one FP32 reciprocal with a round-down estimate
// (tile_search.cuh's qfloor).  A wrong estimate leaves the remainder r =
// q - k p (mod 2^64) outside (0, p): (rf - pf) rf < 0 proves 0 < r < p in
// float by monotone rounding.  With the estimate below 2^20 it is off by at
// most one; k + 1 wraps r to 2^64 + r - p, which is >= p unless p > 2^63,
// and then q < p (p + q <= one throughout), so the estimate errs only when
// q is within 2^-21 of p, where 2^64 + q - p >= p.  A flagged step (or r
// == 0, the expansion exhausted) is redone with the hardware division, the
// whole warp entering that path through one vote.
#pragma once
#include <stdint.h>

#include "search_core.cuh"
#include "tile_search.cuh"

namespace hrb {

struct CSlot {
    uint64_t p, q, d, eps;
    float pf, qf;      // float(p), float(q)
    uint32_t u, v, M;  // M = max(N - u - v, 0)
    uint32_t it;       // per-mode iteration count
    uint32_t st;       // bit 0: swapped; bits 1-2: swapped k == 0 steps just before (0, 1, 2+)
    int item;
};

// lef_begin (search_core.cuh / lowerbound.py:166-181): true when the search
// ends before its loop, with *ok
template <int W>
__device__ __forceinline__ bool cslot_init(uint64_t a, uint64_t b, uint64_t eps, uint32_t N, CSlot& s, bool* ok) {
    if (b < eps) {
        *ok = false;
        return true;
    }
    if (a == 0 || N == 1) {
        *ok = true;
        return true;
    }
    const uint64_t c = (W == 64) ? (0ull - a) : ((1ull << 32) - a);  // one - a
    const bool sw = b >= a;
    s.p = sw ? c : a;
    s.q = sw ? a : c;
    s.pf = __ull2float_rn(s.p);
    s.qf = __ull2float_rn(s.q);
    s.u = 1;
    s.v = 1;
    s.M = N >= 2 ? N - 2 : 0;
    s.d = b;
    s.eps = eps;
    s.it = 0;
    s.st = sw ? 1u : 0u;
    return false;
}

// The step up to its quotient: d -= q when swapped (and the failure test),
// k = floor(q / p) estimated, r = q - k p, and whether the estimate may be
// wrong.  p, q are left untouched for a redo.
__device__ __forceinline__ void cslot_pre(CSlot& s, bool& fail, uint64_t& r, float& rf, uint32_t& k, bool& bad) {
    const bool sw = s.st & 1u;
    if (sw) s.d -= s.q;
    fail = sw && s.d < s.eps;
    const float rcp = rcp_approx(s.pf);
    const int32_t ke = qfloor(s.qf, rcp);  // >= 0: qf * rcp >= 0
    r = madd64(s.q, (uint32_t)ke, 0 - s.p);
    rf = __ull2float_rn(r);
    k = (uint32_t)ke;
    bad = (ke >= QMAX) | !(__fmul_rn(rf - s.pf, rf) < 0.0f);
}

// the rare exact quotient (k saturates at 2^32 - 1: v >= 1 makes k v >= M,
// the end the reference reaches with the full quotient)
__device__ __noinline__ uint64_t cslot_exact_quot(uint64_t q, uint64_t p) { return q / p; }

__device__ __forceinline__ void cslot_exact(const CSlot& s, uint64_t& r, float& rf, uint32_t& k, bool& zero) {
    const uint64_t kk = cslot_exact_quot(s.q, s.p);
    r = s.q - kk * s.p;
    rf = __ull2float_rn(r);
    k = kk > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)kk;
    zero = r == 0;
}

// The rest of the step with the step's quotient k and remainder r: counts,
// updates, the role swap.  Returns 0 running, 1 failure, 2 success.
// lim = 3 - mode: a swapped k == 0 step with `lim` such steps just before it
// is a batched step the mode does not count.
__device__ __forceinline__ int cslot_post(CSlot& s, bool fail, uint64_t r, float rf, uint32_t k, bool zero,
                                          uint32_t lim) {
    const bool sw = s.st & 1u;
    const uint32_t run = s.st >> 1;
    const bool k0 = k == 0;
    s.it += (sw && k0 && run >= lim) ? 0u : 1u;
    const uint64_t P = mul_wide(k, s.v);
    const bool done = P >= s.M;
    const uint32_t u1 = s.u + (uint32_t)P;
    const uint32_t M1 = s.M - (uint32_t)P;
    const uint64_t p1 = s.p - r;
    const float p1f = __ull2float_rn(p1);
    const uint32_t v1 = s.v + u1;
    const uint32_t M2 = M1 - min(M1, u1);
    const bool nxt = s.d >= (sw ? r : p1);
    const bool x = nxt != sw;
    s.p = x ? r : p1;
    s.q = x ? p1 : r;
    s.pf = x ? rf : p1f;
    s.qf = x ? p1f : rf;
    s.u = x ? v1 : u1;
    s.v = x ? u1 : v1;
    s.M = M2;
    s.st = (nxt ? 1u : 0u) | ((sw && k0) ? (min(run + 1u, 2u) << 1) : 0u);
    return fail ? 1 : ((done || zero) ? 2 : 0);
}

// All items of one lane, two searches at a time; a slot whose search ended
// takes the lane's next item.  src.build(k, a, b, eps, N) builds item k
// (called in order k = 0, 1, 2, ..., once each) and reports whether it is
// valid.  Returns the lane's failure bits (bit k = item k failed) and adds
// the per-mode iteration counts to *iters.  Must be called by all 32 lanes
// (the votes).
template <int W, int NU, class Src>
__device__ __forceinline__ uint32_t lane_items_classic(Src& src, unsigned long long* iters, int mode,
                                                       uint32_t n_items = NU) {
    uint32_t fails = 0, its = 0;
    const int mine = (int)(n_items < (uint32_t)NU ? n_items : (uint32_t)NU);
    const uint32_t lim = 3u - (uint32_t)mode;
    int next = 0;
    CSlot s0, s1;
    // the next item that starts a real search (immediate outcomes recorded)
    auto refill = [&](CSlot& s) -> bool {
        while (next < mine) {
            uint64_t a, b, e;
            uint32_t N;
            const int k = next++;
            if (!src.build(k, a, b, e, N)) continue;
            bool ok;
            if (cslot_init<W>(a, b, e, N, s, &ok)) {
                fails |= ok ? 0u : 1u << k;
                continue;
            }
            s.item = k;
            return true;
        }
        return false;
    };
    bool act0 = refill(s0), act1 = refill(s1);
    while (__any_sync(0xffffffffu, act0 || act1)) {
        bool f0, f1, b0, b1, z0 = false, z1 = false;
        uint64_t r0, r1;
        float rf0, rf1;
        uint32_t k0, k1;
        cslot_pre(s0, f0, r0, rf0, k0, b0);
        cslot_pre(s1, f1, r1, rf1, k1, b1);
        b0 = b0 && act0;
        b1 = b1 && act1;
        if (__any_sync(0xffffffffu, b0 || b1)) {  // rare: the hardware division
            if (b0) cslot_exact(s0, r0, rf0, k0, z0);
            if (b1) cslot_exact(s1, r1, rf1, k1, z1);
        }
        const int e0 = cslot_post(s0, f0, r0, rf0, k0, z0, lim);
        const int e1 = cslot_post(s1, f1, r1, rf1, k1, z1, lim);
        if (act0 && e0) {
            fails |= e0 == 1 ? 1u << s0.item : 0u;
            its += s0.it;
            act0 = refill(s0);
        }
        if (act1 && e1) {
            fails |= e1 == 1 ? 1u << s1.item : 0u;
            its += s1.it;
            act1 = refill(s1);
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
