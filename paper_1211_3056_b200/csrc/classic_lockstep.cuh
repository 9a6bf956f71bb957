// classic_lockstep.cuh -- throughput form of the classic (Lefevre) search
// for the phases: lowerbound.py:88-225 (_lefevre_core / _lefevre_swap_core,
// which agree on the full outcome, test_lowerbound.py:236-238) restated for
// warp-uniform control flow.
//
// Each lane runs TWO searches at a time (two dependency chains).  The
// classic walk's iteration counts vary widely (NMDM ~20 %,
// PAPER.md:1653-1664), so a slot whose search ends takes the next entry of
// a per-warp queue of searches at once (see lane_items_classic_m).  Only
// the verdict and the per-mode iteration count are produced (what the
// phases read, pipeline.py:200-201, 228); the general core (search_core.cuh)
// keeps the full outcome for the search ABI.
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
// mode 1 counts one more step and mode 2 none (mode 0 never batches).  Two
// run bits in the slot reproduce that; the mode is a template parameter.
//
// The quotient comes from one FP32 reciprocal with a round-down estimate
// (tile_search.cuh's qfloor).  A wrong estimate leaves the remainder r =
// q - k p (mod 2^64) outside (0, p): (rf - pf) rf < 0 proves 0 < r < p in
// float by monotone rounding.  An estimate k + 1 wraps r to 2^64 + r - p,
// which is >= p unless p > 2^63; then q < p (p + q <= one throughout), so
// the estimate errs only when q is within 2^-21 of p, where 2^64 + q - p >=
// p.  A flagged step (or r == 0, the expansion exhausted) is redone with
// the hardware division, the whole warp entering that path through one
// vote.
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
    // CF_SW: swapped.  CF_FAIL: the swapped step's d -= q, applied to d by
    // the step before it (which decides the swap: the comparison d >= q is
    // that subtraction's borrow), failed.  CF_R1 / CF_R2: the last one / two
    // steps were swapped with k == 0 (the reference's batched run).
    uint32_t fl;
    int item;
};

constexpr uint32_t CF_SW = 1, CF_FAIL = 2, CF_R1 = 4, CF_R2 = 8;

// lef_begin (search_core.cuh / lowerbound.py:166-181): true when the search
// ends before its loop, with *ok; otherwise the slot holds its start, with
// the first swapped step's d -= q applied
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
    s.d = sw ? b - a : b;
    s.eps = eps;
    s.it = 0;
    s.fl = sw ? (CF_SW | ((b - a < eps) ? CF_FAIL : 0u)) : 0u;
    return false;
}

// The step up to its quotient: k = floor(q / p) estimated and q replaced by
// r = q - k p in place (a redo recovers q = r + k p), and whether the
// estimate may be wrong.  No bound on k is tested: below q/p = 2^22 the
// estimate is within 2 of k and 3p <= 2^64 keeps a wrapped r >= p; past it
// the float leaves the integer grid and the estimate falls below k (r >= p).
__device__ __forceinline__ void cslot_pre(CSlot& s, float& rf, uint32_t& k, bool& bad) {
    const float rcp = rcp_approx(s.pf);
    const int32_t ke = qfloor(s.qf, rcp);  // >= 0: qf * rcp >= 0
    s.q = madd64(s.q, (uint32_t)ke, 0 - s.p);
    rf = __ull2float_rn(s.q);
    k = (uint32_t)ke;
    bad = !(__fmul_rn(rf - s.pf, rf) < 0.0f);
}

// the rare exact quotient (k saturates at 2^32 - 1: v >= 1 makes k v >= M,
// the end the reference reaches with the full quotient)
__device__ __noinline__ uint64_t cslot_exact_quot(uint64_t q, uint64_t p) { return q / p; }

__device__ __forceinline__ void cslot_exact(CSlot& s, float& rf, uint32_t& k, bool& zero) {
    const uint64_t q = s.q + (uint64_t)k * s.p;
    const uint64_t kk = cslot_exact_quot(q, s.p);
    s.q = q - kk * s.p;
    rf = __ull2float_rn(s.q);
    k = kk > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)kk;
    zero = s.q == 0;
}

// The rest of the step with its quotient k (q already the remainder r):
// count, updates, the role swap and the next step's d -= q.  Returns true
// when the search ended (CF_FAIL of the old flags tells a failure).  MODE
// fixes which swapped k == 0 steps go uncounted: mode 1 those after two such
// steps, mode 2 after one, mode 0 none.
template <int MODE>
__device__ __forceinline__ bool cslot_post(CSlot& s, float rf, uint32_t k, bool zero, uint32_t& fl_old) {
    const uint32_t fl = s.fl;
    fl_old = fl;
    const bool sw = fl & CF_SW;
    if (MODE != 0) {
        const uint32_t um = CF_SW | (MODE == 1 ? CF_R2 : CF_R1);
        s.it += (k == 0 && (fl & um) == um) ? 0u : 1u;
    } else {
        s.it += 1;
    }
    const uint64_t P = mul_wide(k, s.v);
    const bool done = P >= s.M;
    const uint64_t r = s.q, p0 = s.p;
    const uint32_t u1 = s.u + (uint32_t)P;
    const uint32_t M1 = s.M - (uint32_t)P;
    const uint64_t p1 = p0 - r;
    const float p1f = __ull2float_rn(p1);
    const uint32_t v1 = s.v + u1;
    s.M = M1 - min(M1, u1);
    // next: swapped iff d >= (swapped ? q : p), whose q is then exactly that
    bool nxt;
    const uint64_t dn = sub_nb(s.d, sw ? r : p1, nxt);
    const bool x = nxt != sw;
    const uint64_t pn = x ? r : p1;
    s.p = pn;
    s.q = p0 - pn;  // the other of r, p1 (r + p1 = p)
    s.pf = x ? rf : p1f;
    s.qf = x ? p1f : rf;
    const uint32_t un = x ? v1 : u1;
    s.v = (u1 + v1) - un;
    s.u = un;
    s.d = nxt ? dn : s.d;
    uint32_t f = nxt ? (CF_SW | (dn < s.eps ? CF_FAIL : 0u)) : 0u;
    if (MODE != 0 && sw && k == 0) f |= CF_R1 | (MODE == 1 ? ((fl << 1) & CF_R2) : 0u);
    s.fl = f;
    return (fl & CF_FAIL) || done || zero;
}

// Per-warp work queue in shared memory: the searches of the lanes' next
// items, built and set up by all lanes together, taken in order by
// whichever slot of the warp frees up.
#ifndef HRB_CL_CHUNK
#define HRB_CL_CHUNK 4  // items per lane per build pass
#endif
struct ClQueue {  // the searches' initial states, structure of arrays
    uint64_t p[32 * HRB_CL_CHUNK], q[32 * HRB_CL_CHUNK], d[32 * HRB_CL_CHUNK], e[32 * HRB_CL_CHUNK];
    float pf[32 * HRB_CL_CHUNK], qf[32 * HRB_CL_CHUNK];
    uint32_t M[32 * HRB_CL_CHUNK], tag[32 * HRB_CL_CHUNK];  // tag: owner lane | item << 8 | flags << 16
    uint32_t fails[32];
};

// All items of the warp's lanes, two searches at a time per lane.  Building
// an item (the tabulated walk) costs several times a step, and a slot's
// search ends at an unpredictable step, so items are built in warp-wide
// passes -- each lane its next HRB_CL_CHUNK items, immediate outcomes
// recorded on the spot -- into a queue of the searches that remain, and a
// slot that frees up takes the queue's next entry: the divergent part of a
// refill is only the slot's setup, and every slot of the warp stays busy
// until the queue runs dry (no lane waits on its own slowest items).
// src.build(k, a, b, eps, N) builds the lane's item k (called in order
// k = 0, 1, 2, ..., once each) and reports whether it is valid.  Returns the
// lane's failure bits (bit k = the lane's item k failed) and adds the
// per-mode iteration counts of the searches this lane ran to *iters.  Must
// be called by all 32 lanes (the votes, the shared queue).
template <int W, int NU, int MODE, class Src>
__device__ __forceinline__ uint32_t lane_items_classic_m(Src& src, ClQueue* qu, unsigned long long* iters,
                                                         uint32_t n_items) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t its = 0;
    const int mine = (int)(n_items < (uint32_t)NU ? n_items : (uint32_t)NU);
    int next = 0;
    qu->fails[lane] = 0;
    uint32_t qh = 0, qn = 0;  // queue head and length (warp-uniform)
    CSlot s0, s1;
    bool act0 = false, act1 = false;
    while (true) {
        // refill idle slots from the queue, building the next items first
        // when it is empty
        const uint32_t w0 = __ballot_sync(0xffffffffu, !act0), w1 = __ballot_sync(0xffffffffu, !act1);
        if (w0 | w1) {
            // (a pass may yield only immediate outcomes: build until the
            // queue has entries or the lanes' items run out)
            while (qh == qn && __any_sync(0xffffffffu, next < mine)) {
                __syncwarp();
                qh = 0;
                qn = 0;
#pragma unroll 1
                for (int j = 0; j < HRB_CL_CHUNK; j++) {
                    uint64_t a = 0, b = 0, e = 0;
                    uint32_t N = 0;
                    const int k = next;
                    const bool valid = k < mine && src.build(k, a, b, e, N);
                    next += k < mine ? 1 : 0;
                    if (valid && b < e) qu->fails[lane] |= 1u << k;  // own word: no race
                    CSlot t;
                    bool ok;
                    const bool real = valid && !cslot_init<W>(a, b, e, N, t, &ok);
                    const uint32_t m = __ballot_sync(0xffffffffu, real);
                    if (real) {
                        const uint32_t pos = qn + __popc(m & lt);
                        qu->p[pos] = t.p;
                        qu->q[pos] = t.q;
                        qu->d[pos] = t.d;
                        qu->e[pos] = t.eps;
                        qu->pf[pos] = t.pf;
                        qu->qf[pos] = t.qf;
                        qu->M[pos] = t.M;
                        qu->tag[pos] = (uint32_t)lane | ((uint32_t)k << 8) | (t.fl << 16);
                    }
                    qn += __popc(m);
                }
                __syncwarp();
            }
            const uint32_t n0 = __popc(w0);
            const uint32_t p0 = qh + __popc(w0 & lt), p1 = qh + n0 + __popc(w1 & lt);
            auto take = [&](CSlot& t, uint32_t pos) {
                t.p = qu->p[pos];
                t.q = qu->q[pos];
                t.d = qu->d[pos];
                t.eps = qu->e[pos];
                t.pf = qu->pf[pos];
                t.qf = qu->qf[pos];
                t.M = qu->M[pos];
                const uint32_t tg = qu->tag[pos];
                t.item = (int)(tg & 0xFFFFu);
                t.fl = tg >> 16;
                t.u = 1;
                t.v = 1;
                t.it = 0;
            };
            if (!act0 && p0 < qn) {
                take(s0, p0);
                act0 = true;
            }
            if (!act1 && p1 < qn) {
                take(s1, p1);
                act1 = true;
            }
            qh = min(qh + n0 + __popc(w1), qn);
        }
        if (!__any_sync(0xffffffffu, act0 || act1)) break;
        bool b0, b1, z0 = false, z1 = false;
        float rf0, rf1;
        uint32_t k0, k1;
        cslot_pre(s0, rf0, k0, b0);
        cslot_pre(s1, rf1, k1, b1);
        b0 = b0 && act0;
        b1 = b1 && act1;
        if (__any_sync(0xffffffffu, b0 || b1)) {  // rare: the hardware division
            if (b0) cslot_exact(s0, rf0, k0, z0);
            if (b1) cslot_exact(s1, rf1, k1, z1);
        }
        uint32_t g0, g1;
        const bool e0 = cslot_post<MODE>(s0, rf0, k0, z0, g0);
        const bool e1 = cslot_post<MODE>(s1, rf1, k1, z1, g1);
        if (act0 && e0) {
            if (g0 & CF_FAIL) atomicOr(&qu->fails[s0.item & 31], 1u << (s0.item >> 8));
            its += s0.it;
            act0 = false;
        }
        if (act1 && e1) {
            if (g1 & CF_FAIL) atomicOr(&qu->fails[s1.item & 31], 1u << (s1.item >> 8));
            its += s1.it;
            act1 = false;
        }
    }
    *iters += its;
    __syncwarp();
    return qu->fails[lane];
}

}  // namespace hrb
