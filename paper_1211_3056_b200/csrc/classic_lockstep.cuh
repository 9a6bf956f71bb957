// classic_lockstep.cuh -- throughput form of the classic (Lefevre) search
// for the phases: lowerbound.py:88-225 (_lefevre_core / _lefevre_swap_core,
// which agree on the full outcome, test_lowerbound.py:236-238) in the
// role-swapped single-body form of search_core.cuh's lef_step, restated for
// warp-uniform control flow.
//
// Each lane runs TWO searches at a time (two dependency chains) over its
// items.  The step body is straight-line: the swap / batched-reduction
// decisions of the reference become selects, the quotient floor(q / p) comes
// from one FP32 reciprocal with a round-down estimate (tile_search.cuh's
// qfloor), and a possibly wrong estimate (remainder outside [0, p), or a
// quotient >= 2^20) sends the whole warp through one vote to an exact
// division.  The classic walk's iteration counts vary widely (NMDM ~20 %,
// PAPER.md:1653-1664), so a slot whose search ends is refilled at once with
// the lane's next item instead of waiting for the slowest search of the
// warp.  Only the verdict and the per-mode iteration count are produced
// (what the phases read, pipeline.py:200-201, 228); the general core
// (search_core.cuh) keeps the full outcome for the search ABI.
#pragma once
#include <stdint.h>

#include "search_core.cuh"
#include "tile_search.cuh"

namespace hrb {

struct CSlot {
    uint64_t p, q, d, eps;
    uint32_t u, v, N, it;
    uint32_t fl;  // bit 0 swapped, bit 1 in_batch, bit 2 extra
    int item;
};

constexpr uint32_t CF_SWAP = 1, CF_BATCH = 2, CF_EXTRA = 4;

// lef_begin (search_core.cuh / lowerbound.py:88-107): true when the search
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
    s.p = a;
    s.q = (W == 64) ? (0ull - a) : ((1ull << 32) - a);
    s.u = 1;
    s.v = 1;
    s.d = b;
    s.eps = eps;
    s.N = N;
    s.it = 0;
    s.fl = 0;
    return false;
}

// One classic step, fast path (lef_step, branch-free).  Returns the search's
// end: 0 running, 1 failure (d < eps), 2 success.  `bad` flags a quotient
// estimate that may be wrong; the caller then redoes the step exactly from
// the saved pre-step state (cslot_step with EXACT).
template <bool EXACT>
__device__ __forceinline__ int cslot_step(CSlot& s, int mode, bool& bad) {
    const bool swapped0 = s.fl & CF_SWAP, in_batch = s.fl & CF_BATCH, extra = s.fl & CF_EXTRA;
    const bool batched = in_batch && s.d >= s.q && s.q < s.p;
    // the main branch: swap the roles when d crosses the current threshold
    const bool nxt = s.d >= (swapped0 ? s.q : s.p);
    const bool doswap = !batched && nxt != swapped0;
    const uint64_t p = doswap ? s.q : s.p, q = doswap ? s.p : s.q;
    const uint32_t u = doswap ? s.v : s.u, v = doswap ? s.u : s.v;
    const bool swapped = batched ? swapped0 : nxt;
    s.it += batched ? ((mode == 1 && !extra) ? 1u : 0u) : 1u;
    const bool extra1 = batched ? (extra || mode == 1) : extra;
    // swapped: d -= q, and a failure as soon as d < eps
    const uint64_t d = swapped ? s.d - q : s.d;
    const bool fail = swapped && d < s.eps;
    // k = floor(q / p) when q >= p
    uint64_t k;
    if (EXACT) {
        k = q >= p ? q / p : 0;
        bad = false;
    } else {
        const float pf = __ull2float_rn(p);
        const int32_t ke = max(qfloor(__ull2float_rn(q), rcp_approx(pf)), 0);
        const uint64_t r = q - (uint64_t)(uint32_t)ke * p;
        const bool big = q >= p;
        bad = big && ((ke >= QMAX) | (r >= p) | (r > q));
        k = big ? (uint64_t)(uint32_t)ke : 0;
    }
    // counts: u + v reaching N ends the walk (success), as does a quotient
    // that would overshoot it (k v >= N - u - v)
    const uint64_t sv = (uint64_t)u + v;
    const uint64_t need = sv < s.N ? s.N - sv : 0;
    const bool over = sv >= s.N || (k >> 32) != 0 || (uint64_t)(uint32_t)k * v >= need;
    const uint64_t qn = q - k * p;
    const uint32_t un = u + (uint32_t)k * v;
    const bool q0 = qn == 0;
    s.p = p - qn;
    s.q = qn;
    s.u = un;
    s.v = v + un;
    s.d = d;
    const bool enter = !batched && swapped && k == 0 && mode != 0;
    s.fl = (swapped ? CF_SWAP : 0u) | ((enter || (batched && in_batch)) ? CF_BATCH : 0u) |
           ((enter ? false : extra1) ? CF_EXTRA : 0u);
    return fail ? 1 : ((over || q0) ? 2 : 0);
}

// All items of one lane, two searches at a time, each slot refilled with
// the lane's next item as soon as its search ends.  src.build(k, a, b, eps,
// N) builds item k (called in order k = 0, 1, 2, ..., once each) and
// reports whether it is valid.  Returns the lane's failure bits (bit k =
// item k failed) and adds the per-mode iteration counts to *iters.  Must
// be called by all 32 lanes (the votes).
template <int W, int NU, class Src>
__device__ __forceinline__ uint32_t lane_items_classic(Src& src, unsigned long long* iters, int mode,
                                                       uint32_t n_items = NU) {
    uint32_t fails = 0, its = 0;
    const int mine = (int)(n_items < (uint32_t)NU ? n_items : (uint32_t)NU);
    int next = 0;
    CSlot s0, s1;
    // next item that starts a real search (immediate outcomes recorded)
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
        const CSlot o0 = s0, o1 = s1;
        bool b0, b1;
        int r0 = cslot_step<false>(s0, mode, b0);
        int r1 = cslot_step<false>(s1, mode, b1);
        b0 = b0 && act0;
        b1 = b1 && act1;
        if (__any_sync(0xffffffffu, b0 || b1)) {  // rare: exact division from the saved state
            bool x;
            if (b0) {
                s0 = o0;
                r0 = cslot_step<true>(s0, mode, x);
            }
            if (b1) {
                s1 = o1;
                r1 = cslot_step<true>(s1, mode, x);
            }
        }
        if (act0 && r0) {
            fails |= r0 == 1 ? 1u << s0.item : 0u;
            its += s0.it;
            act0 = refill(s0);
        }
        if (act1 && r1) {
            fails |= r1 == 1 ? 1u << s1.item : 0u;
            its += s1.it;
            act1 = refill(s1);
        }
    }
    *iters += its;
    return fails;
}

}  // namespace hrb
