// search_core.cuh -- device lower-bound searches for min{(b - a*x) mod 1 : x < N}.
//
// Restates, for one lane, the four reference cores of
// /root/reference/pkg/src/hardround/lowerbound.py:
//   regular family  (_regular_core 228-267, _regular_unrolled_core 270-308)
//   classic family  (_lefevre_core 88-163, _lefevre_swap_core 166-225)
// bit-exactly (verdict, d, iterations, points_placed) at word width W in
// {32, 64}, in 64-bit registers.  The reference uses unbounded Python ints;
// the only quantities that leave 64 bits are handled explicitly:
//   * the first regular quotient 2^W / a (q starts at one = 2^W),
//   * a = 1 (first quotient 2^64, v = 2^64),
//   * exhaustion with divisor 1 (count 2^64, from the circle identity
//     cS*L + cL*S = 2^W that every half-step preserves),
//   * 65-bit point totals, returned as (lo, hi).
//
// Division: quotients are Gauss-Kuzmin distributed (mostly 1..3), so a
// quotient is estimated from an FP32 reciprocal of the divisor (one per
// divisor, shared by the two divisions of a regular half-step) and fixed with
// one compare; quotients >= 2^20 take the exact hardware path.
#pragma once
#include <stdint.h>

namespace hrb {

enum { ALGO_LEFEVRE = 0, ALGO_LEFEVRE_SWAP = 1, ALGO_REGULAR = 2, ALGO_REGULAR_UNROLLED = 3 };

struct Outcome {
    uint64_t d;
    uint64_t it;
    uint64_t pts_lo;
    uint32_t pts_hi;
    bool ok;
};

__device__ __forceinline__ Outcome mk_out(bool ok, uint64_t d, uint64_t it, uint64_t lo, uint32_t hi) {
    Outcome o;
    o.ok = ok;
    o.d = d;
    o.it = it;
    o.pts_lo = lo;
    o.pts_hi = hi;
    return o;
}

// Branch-decision recorders: the device form of the reference cores' optional
// `trace` list (lowerbound.py:88-308; consumed by divergence.py:243-248).
struct NoTrace {
    __device__ __forceinline__ void rec(bool) {}
};

struct BitTrace {  // decisions as bits, LSB first; len counts every decision
    uint64_t* words;
    uint32_t cap_bits;
    uint32_t len;
    __device__ __forceinline__ void rec(bool b) {
        if (len < cap_bits) {
            const uint64_t m = 1ull << (len & 63);
            if (b) words[len >> 6] |= m;
            else words[len >> 6] &= ~m;
        }
        len++;
    }
};

// FP32 reciprocal of x (<= 1 ulp; MUFU.RCP), shared by the divisions of a step.
__device__ __forceinline__ float recip_f32(uint64_t x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__ull2float_rn(x)));
    return r;
}

// k = floor(y / x), r = y - k x, given rcp ~ 1/x.  With M = 1.5 * 2^23 the
// FFMA y*rcp + (M - 1) lands on the integer grid of [2^23, 2^24), so its
// single rounding is round(y/x - 1 + e) with |e| < 2^-21 y/x: for y/x < 2^20
// that is floor(y/x) or floor(y/x) - 1 (-1 clamped to 0, where y < x), read
// from the bit pattern; one compare finishes it.  Larger quotients (and
// estimates off the grid) take the hardware division.
__device__ __forceinline__ uint64_t divmod_est(uint64_t y, uint64_t x, float rcp, uint64_t& r) {
    const float kf = fmaf(__ull2float_rn(y), rcp, 12582911.0f);
    const int32_t ke = (int32_t)(__float_as_uint(kf) - 0x4B400000u);
    if (ke < (1 << 20)) {
        const uint32_t k = (uint32_t)max(ke, 0);
        const uint64_t rr = y - (uint64_t)k * x;
        const bool c = rr >= x;
        r = c ? rr - x : rr;
        return (uint64_t)k + (c ? 1u : 0u);
    }
    const uint64_t k = y / x;
    r = y - k * x;
    return k;
}

__device__ __forceinline__ uint64_t mod_est(uint64_t y, uint64_t x, float rcp) {
    uint64_t r;
    divmod_est(y, x, rcp, r);
    return r;
}

// 65-bit sum helpers
__device__ __forceinline__ void add65(uint64_t x, uint64_t y, uint64_t& lo, uint32_t& hi) {
    lo = x + y;
    hi = lo < x ? 1u : 0u;
}

// ---------------------------------------------------------------------------
// regular family (lowerbound.py:228-308)
//
// State after each half-step, in role form: S (current divisor), L (current
// dividend), cS, cL (their point counts).  The reference alternates strictly
// between its `p < q` and `p >= q` bodies; role form makes both the same
// body, except the d-reduction offset (0 for the then-body, the new p for
// the else-body).  `it` counts half-steps (= _regular_core iterations);
// _regular_unrolled_core reports ceil(it / 2).
// ---------------------------------------------------------------------------

struct RegState {
    uint64_t S, L, cS, cL, d, eps, N, it;
    bool then_next;  // next half-step is the reference's `p < q` body
};

// Start a search.  Returns true if the search finished during setup (early
// exits and the first half-step against one = 2^W) with *out filled.
template <int W, class Tr = NoTrace>
__device__ __forceinline__ bool reg_begin(uint64_t a, uint64_t b, uint64_t eps, uint64_t N, RegState& st,
                                          Outcome* out, Tr* tr = nullptr, bool unrolled = false) {
    uint64_t d = b;
    if (d < eps) {
        *out = mk_out(false, d, 0, 1, 0);
        return true;
    }
    if (a == 0) {
        *out = mk_out(d > eps, d, 0, N, 0);
        return true;
    }
    if (N <= 1) {
        *out = mk_out(d > eps, d, 0, 1, 0);
        return true;
    }
    uint64_t k, rem;
    if (tr && !unrolled) tr->rec(true);  // iteration 1 is the then-body (p = a < q = one)
    if (W == 64) {
        if (a == 1) {
            // k = 2^64, q -> 0: d = b mod 1 = 0, points max(1 + 2^64, N) = 2^64 + 1
            *out = mk_out(false, 0, 1, 1, 1);
            return true;
        }
        uint64_t k0 = ~0ull / a;
        uint64_t r0 = ~0ull - k0 * a;
        if (r0 == a - 1) {
            k = k0 + 1;
            rem = 0;
        } else {
            k = k0;
            rem = r0 + 1;
        }
    } else {
        k = (1ull << 32) / a;
        rem = (1ull << 32) - k * a;
    }
    d = d % a;
    // counts after the first then-body: u = 1, v = k   (k <= 2^63 here)
    if (rem == 0) {
        uint64_t s = 1 + k;
        *out = mk_out(d > eps, d, 1, s > N ? s : N, 0);
        return true;
    }
    if (k >= N - 1) {
        *out = mk_out(d > eps, d, 1, 1 + k, 0);
        return true;
    }
    st.S = rem;
    st.L = a;
    st.cS = k;
    st.cL = 1;
    st.d = d;
    st.eps = eps;
    st.N = N;
    st.it = 1;
    st.then_next = false;
    return false;
}

// One half-step.  Returns true when the search finished (*out filled).
template <int W, class Tr = NoTrace>
__device__ __forceinline__ bool reg_step(RegState& st, Outcome* out, Tr* tr = nullptr, bool unrolled = false) {
    const uint64_t S = st.S;
    const float sinv = recip_f32(S);
    uint64_t Lp;
    uint64_t k = divmod_est(st.L, S, sinv, Lp);
    uint64_t cLp = st.cL + k * st.cS;  // exact unless exhausted with S == 1 (see below)
    uint64_t d = st.d;
    uint64_t off = st.then_next ? 0 : Lp;
    if (tr) {
        // _regular_core: one decision per iteration (p < q);
        // _regular_unrolled_core: the d >= p guard of each second half
        if (!unrolled) tr->rec(st.then_next);
        else if (!st.then_next) tr->rec(d >= Lp);
    }
    if (d >= off) d = mod_est(d - off, S, sinv);
    st.it++;
    if (Lp == 0) {
        // exhausted: cLp * S = 2^W exactly
        uint64_t lo;
        uint32_t hi;
        if (W == 64 && S == 1) {
            lo = st.cS;
            hi = 1;
        } else {
            add65(st.cS, cLp, lo, hi);
        }
        if (hi == 0 && lo < st.N) lo = st.N;
        *out = mk_out(d > st.eps, d, st.it, lo, hi);
        return true;
    }
    if (cLp >= st.N - st.cS) {  // cS < N holds on entry
        uint64_t lo;
        uint32_t hi;
        add65(st.cS, cLp, lo, hi);
        *out = mk_out(d > st.eps, d, st.it, lo, hi);
        return true;
    }
    st.L = S;
    st.S = Lp;
    st.cL = st.cS;
    st.cS = cLp;
    st.d = d;
    st.then_next = !st.then_next;
    return false;
}

template <int W, class Tr = NoTrace>
__device__ Outcome regular_search(uint64_t a, uint64_t b, uint64_t eps, uint64_t N, Tr* tr = nullptr,
                                  bool unrolled = false) {
    RegState st;
    Outcome o;
    if (reg_begin<W, Tr>(a, b, eps, N, st, &o, tr, unrolled)) return o;
    while (!reg_step<W, Tr>(st, &o, tr, unrolled)) {
    }
    return o;
}

// ---------------------------------------------------------------------------
// classic family (lowerbound.py:88-225), in the role-swapped single-body
// form of _lefevre_swap_core with its batched plain-reduction loop folded
// into the main loop: a "batched" step is a main step with k = 0 that the
// reference executes inside its inner while-loop, so only the iteration
// accounting differs (mode 0: no batching; 1: first batched step counted;
// 2: none counted).  _lefevre_core and _lefevre_swap_core agree on the full
// (ok, d, it, points) tuple (test_lowerbound.py:236-238).
// ---------------------------------------------------------------------------

struct LefState {
    uint64_t p, q, u, v, d, eps, N, it;
    bool swapped, in_batch, extra;
};

template <int W>
__device__ __forceinline__ bool lef_begin(uint64_t a, uint64_t b, uint64_t eps, uint64_t N, LefState& st,
                                          Outcome* out) {
    if (b < eps) {
        *out = mk_out(false, b, 0, 1, 0);
        return true;
    }
    if (a == 0) {
        *out = mk_out(true, b, 0, N, 0);
        return true;
    }
    if (N == 1) {
        *out = mk_out(true, b, 0, 1, 0);
        return true;
    }
    st.p = a;
    st.q = (W == 64) ? (0ull - a) : ((1ull << 32) - a);
    st.u = 1;
    st.v = 1;
    st.d = b;
    st.eps = eps;
    st.N = N;
    st.it = 0;
    st.swapped = false;
    st.in_batch = false;
    st.extra = false;
    return false;
}

// trace polarity: _lefevre_swap_core records `swapped` (d >= p of the plain
// walk), _lefevre_core records its complement (d < p); batched extras are
// swapped-state decisions (lowerbound.py:109-148, 187-214)
template <int W, class Tr = NoTrace>
__device__ __forceinline__ bool lef_step(LefState& st, int mode, Outcome* out, Tr* tr = nullptr,
                                         bool swap_polarity = false) {
    bool batched = st.in_batch && st.d >= st.q && st.q < st.p;
    if (batched) {
        if (mode == 1 && !st.extra) {
            st.it++;
            st.extra = true;
            if (tr) tr->rec(swap_polarity);
        }
    } else {
        st.in_batch = false;
        bool nxt = st.d >= (st.swapped ? st.q : st.p);
        if (nxt != st.swapped) {
            uint64_t t = st.p;
            st.p = st.q;
            st.q = t;
            t = st.u;
            st.u = st.v;
            st.v = t;
            st.swapped = nxt;
        }
        st.it++;
        if (tr) tr->rec(swap_polarity ? st.swapped : !st.swapped);
    }
    if (st.swapped) {
        st.d -= st.q;
        if (st.d < st.eps) {
            uint64_t lo;
            uint32_t hi;
            add65(st.u, st.v, lo, hi);
            *out = mk_out(false, st.d, st.it, lo, hi);
            return true;
        }
    }
    uint64_t k = 0;
    if (st.q >= st.p) {
        uint64_t r;
        k = divmod_est(st.q, st.p, recip_f32(st.p), r);
    }
    uint64_t s = st.u + st.v;
    bool c = s < st.u;
    if (c || s >= st.N) {  // need <= 0: kc = 0
        *out = mk_out(true, st.d, st.it, s, c ? 1u : 0u);
        return true;
    }
    uint64_t need = st.N - s;
    if (__umul64hi(k, st.v) != 0 || k * st.v >= need) {
        uint64_t kc = (need - 1) / st.v + 1;
        unsigned __int128 pts = (unsigned __int128)st.u + (unsigned __int128)kc * st.v + st.v;
        *out = mk_out(true, st.d, st.it, (uint64_t)pts, (uint32_t)(pts >> 64));
        return true;
    }
    st.q -= k * st.p;
    st.u += k * st.v;
    if (st.q == 0) {
        *out = mk_out(true, st.d, st.it, st.N, 0);
        return true;
    }
    st.p -= st.q;
    st.v += st.u;
    if (!batched && st.swapped && k == 0 && mode != 0) {
        st.in_batch = true;
        st.extra = false;
    }
    return false;
}

template <int W, class Tr = NoTrace>
__device__ Outcome lefevre_search(uint64_t a, uint64_t b, uint64_t eps, uint64_t N, int mode, Tr* tr = nullptr,
                                  bool swap_polarity = false) {
    LefState st;
    Outcome o;
    if (lef_begin<W>(a, b, eps, N, st, &o)) return o;
    while (!lef_step<W, Tr>(st, mode, &o, tr, swap_polarity)) {
    }
    return o;
}

template <int W>
__device__ __forceinline__ Outcome run_search(int algo, int mode, uint64_t a, uint64_t b, uint64_t eps,
                                              uint64_t N) {
    if (algo >= ALGO_REGULAR) {
        Outcome o = regular_search<W>(a, b, eps, N);
        if (algo == ALGO_REGULAR_UNROLLED) o.it = (o.it + 1) >> 1;
        return o;
    }
    return lefevre_search<W>(a, b, eps, N, mode);
}

}  // namespace hrb
