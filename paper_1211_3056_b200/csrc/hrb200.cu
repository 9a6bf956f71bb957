// hrb200.cu -- sm_100a kernels + C-ABI of the HR-case search hot path.
//
// Pipeline (reference /root/reference/pkg/src/hardround/pipeline.py:412-463,
// phases 213-293) for one slice of super-domains, entirely on the device:
//
//   prep      per super-domain: warp tiles, max subdomain count, max step
//   phase1    fused tabulated walk (polygen.py:134-158, 255-280) -> degree-1
//             Boolean problem (pipeline.py:141-175) -> search (lowerbound.py)
//             -> verdict bits transposed into a domain bitmap with __ballot_sync
//   compact1  ordered popc-scan compaction of the bitmap -> failing ids
//   phase2    per (failing domain, subdomain): Toeplitz shift + re-test -> bitmap
//   compact2  ordered compaction -> surviving subdomain keys
//   phase3    per (subdomain, chunk): second-order walk mod 2^F, window test,
//             warp-aggregated atomic append (__ballot_sync/__popc, one atomic
//             per warp) + per-thread candidate counts
//   scatter3  scan of the counts turns the unordered append into the
//             reference's argument order (deterministic, no sort)
//
// Data layout: see include/hrb200.h.  All counts between phases stay on the
// device (grid-stride kernels read them), so a slice runs without host
// synchronisation until the caller reads the counts.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <cub/cub.cuh>
#include <cstdlib>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/hrb200.h"
#include "confirm.cuh"
#include "host/polygen.h"
#include "search_core.cuh"
#include "tile_search.cuh"
#include "classic_lockstep.cuh"

using u128 = unsigned __int128;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* msg) {
    g_err = msg;
    return code;
}

int cuda_err(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return HRB_OK;
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return HRB_ERR_RUNTIME;
}

#define CK(x)                                          \
    do {                                               \
        int _rc = cuda_err((x), #x);                   \
        if (_rc) return _rc;                           \
    } while (0)

#ifndef HRB_P1_MINB
#define HRB_P1_MINB 5  // CTAs of 128 per SM for the phase-1 regular kernel
#endif
#ifndef HRB_P2_MINB
#define HRB_P2_MINB 5
#endif
#ifndef HRB_NU
#define HRB_NU 16
#endif
constexpr int NU = HRB_NU;         // domains per lane in phase 1 (stride-32 walk), <= 32
static_assert(NU >= 1 && NU <= 32, "a lane's verdicts live in one 32-bit word");
constexpr int TILE = 32 * NU;      // domains per warp tile
// Phase-3 arguments per thread: chosen on the device per launch (meta[2])
// between CHUNK3_MIN and CHUNK3_MAX (powers of two, multiples of 64): the
// largest chunk that still gives every SM enough threads (fewer per-item
// setups when phase 2 left many subdomains, more parallelism when it left few).
constexpr int CHUNK3_MIN = 128;
#ifndef HRB_CHUNK3_MAX
#define HRB_CHUNK3_MAX 4096  // A/B: 4096 vs 2048 -1.5 to -3.5 % phase 3 at heavy funnels
#endif
constexpr int CHUNK3_MAX = HRB_CHUNK3_MAX;
constexpr int SCAN_BLOCKS = 592;   // 4 CTAs per SM on 148 SMs
constexpr int SCAN_THREADS = 256;

// ---------------------------------------------------------------------------
// slice view on the device
// ---------------------------------------------------------------------------
struct SliceDev {
    int64_t S;
    int CL, F, W, delta;
    const uint32_t* coef;
    const uint64_t* G;
    const uint64_t* s2abs;
    const uint32_t* n_dom;
    const uint32_t* dom_n;
    const uint32_t* last_n;
    const uint64_t* dom_base;
    const uint64_t* m0;
    // streamed upload (hrb_run_slice_host): the coefficient rows, G and
    // s2abs of super-domain t are valid once *ready > t / ready_chunk;
    // nullptr when the slice is resident before the launch
    const uint32_t* ready;
    uint32_t ready_chunk;
};

SliceDev to_dev(const hrb_slice* s) {
    SliceDev d;
    d.S = s->n_super;
    d.CL = s->coef_limbs;
    d.F = s->frac_bits;
    d.W = s->word_bits;
    d.delta = s->delta;
    d.coef = s->coef;
    d.G = s->G;
    d.s2abs = s->s2abs;
    d.n_dom = s->n_dom;
    d.dom_n = s->dom_n;
    d.last_n = s->last_n;
    d.dom_base = s->dom_base;
    d.m0 = s->m0;
    d.ready = nullptr;
    d.ready_chunk = 1;
    return d;
}

// Block the warp until super-domain t's coefficients have landed (streamed
// upload; no-op for a resident slice).  `known` is the warp's last observed
// chunk count: tiles come in increasing order, so a warp polls about once
// per chunk it enters.  Lane 0 polls with backoff.  A counter that never
// gets there (a lost copy, a host-side bug) is given up on after ~60 s of SM
// clock: the warp raises ready[1] (the host turns it into HRB_ERR_RUNTIME)
// and proceeds, so one failed call never kills the CUDA context.
__device__ __forceinline__ void wait_super(const SliceDev& s, int64_t t, uint32_t& known) {
    if (!s.ready) return;
    const uint32_t need = (uint32_t)(t / s.ready_chunk) + 1;
    if (need <= known) return;  // warp-uniform
    uint32_t v = 0;
    if ((threadIdx.x & 31) == 0) {
        const long long t0 = clock64();
        unsigned ns = 128;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(s.ready) : "memory");
        while (v < need) {
            __nanosleep(ns);
            ns = ns < 2048 ? 2 * ns : ns;
            if (clock64() - t0 > 120000000000ll) {
                atomicExch(const_cast<uint32_t*>(s.ready) + 1, 1u);
                v = need;
                break;
            }
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(s.ready) : "memory");
        }
    }
    known = __shfl_sync(0xffffffffu, v, 0);
    // order every lane's later ld.cg after lane 0's acquire (a shuffle
    // carries the value, not the memory ordering; __syncwarp orders memory
    // among the warp's threads)
    __syncwarp();
}

// Loads of data that may be streamed in while the kernel runs go to L2
// (ld.cg): a line cached in L1 before its bytes arrived would be stale.
// Only the regular phase-1 kernel reads streamed data (CG = true).
template <bool CG, class T>
__device__ __forceinline__ T ld_slice(const T* p) {
    if (CG) return __ldcg(p);
    return __ldg(p);
}

__device__ __forceinline__ u128 mask_f(int F) { return F >= 128 ? ~(u128)0 : (((u128)1 << F) - 1); }

// residue mod 2^128 of packed coefficient c of super-domain t: with at least
// four two's-complement limbs it is just the low four limbs (the common case,
// CL = L + 1 = 9; four loads, no shifts); narrower coefficients are
// sign-extended
template <bool CG = false>
__device__ __forceinline__ u128 coef_res(const SliceDev& s, int64_t t, int c) {
    const uint32_t* base = s.coef + (int64_t)c * s.CL * s.S + t;
    if (s.CL >= 4) {
        const uint64_t lo = (uint64_t)ld_slice<CG>(base) | ((uint64_t)ld_slice<CG>(base + s.S) << 32);
        const uint64_t hi = (uint64_t)ld_slice<CG>(base + 2 * s.S) | ((uint64_t)ld_slice<CG>(base + 3 * s.S) << 32);
        return ((u128)hi << 64) | lo;
    }
    u128 r = 0;
    for (int l = 0; l < s.CL; l++) r |= (u128)ld_slice<CG>(base + l * s.S) << (32 * l);
    if (ld_slice<CG>(base + (s.CL - 1) * s.S) & 0x80000000u) r |= ~(u128)0 << (32 * s.CL);  // sign-extend
    return r;
}

// a / b for b < 2^32 through the 32-bit divide when a fits 32 bits (always on
// the pipeline's domain sizes); the 64-bit divide is a CALL to a long routine
__device__ __forceinline__ uint64_t udiv_small(uint64_t a, uint32_t b) {
    return (a >> 32) ? a / b : (uint64_t)((uint32_t)a / b);
}

__device__ __forceinline__ u128 ld128cg(const SliceDev& s, const uint64_t* p, int64_t t) {
    return ((u128)__ldcg(&p[s.S + t]) << 64) | __ldcg(&p[t]);
}

__device__ __forceinline__ u128 ld128(const uint64_t* p, int64_t S, int64_t t) {
    return ((u128)__ldg(&p[S + t]) << 64) | __ldg(&p[t]);
}

// pad of pipeline.py:165-166: ceil((G + |s2| (n-1)^2) / 2^(F-W)) + n + 1
__device__ __forceinline__ uint64_t pad_of(u128 G, u128 s2abs, uint64_t n, int F, int W) {
    uint64_t nm1 = n - 1;
    u128 X = G + s2abs * (u128)(nm1 * nm1);
    int sh = F - W;
    u128 q = sh > 0 ? (X >> sh) + ((X & ((((u128)1) << sh) - 1)) != 0) : X;
    return (uint64_t)q + n + 1;
}

struct Problem {
    uint64_t a, b, eps;
};

// largest t with base[t] <= x, base ascending of length S+1
__device__ __forceinline__ int64_t find_seg(const uint64_t* base, int64_t S, uint64_t x) {
    int64_t lo = 0, hi = S - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (__ldg(&base[mid]) <= x) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// t of a slice-local domain id: interpolation guess (exact when the
// super-domains are uniform) then a short gallop/binary search
__device__ __forceinline__ int64_t locate_super(const uint64_t* base, int64_t S, uint64_t id) {
    const uint64_t total = __ldg(&base[S]);
    int64_t g = total ? (int64_t)((double)id * (double)S / (double)total) : 0;
    if (g >= S) g = S - 1;
    if (__ldg(&base[g]) <= id && id < __ldg(&base[g + 1])) return g;
    return find_seg(base, S, id);
}

__device__ __forceinline__ uint64_t domain_size(const SliceDev& s, int64_t t, uint64_t i) {
    uint32_t nd = __ldg(&s.n_dom[t]);
    return i == (uint64_t)nd - 1 ? __ldg(&s.last_n[t]) : __ldg(&s.dom_n[t]);
}

__device__ __forceinline__ uint64_t binom2(uint64_t i) { return i ? (i * (i - 1)) >> 1 : 0; }

// ---------------------------------------------------------------------------
// prep: tiles per super-domain, max subdomain count J, max subdomain step
// ---------------------------------------------------------------------------
__global__ void prep_kernel(SliceDev s, int split, uint64_t* tiles, unsigned long long* meta) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long J = 0, mstep = 0;
    if (t < s.S) {
        const uint32_t nd = s.n_dom[t];
        tiles[t] = (nd + TILE - 1) / TILE;
        const uint64_t sizes[2] = {s.dom_n[t], s.last_n[t]};
        for (int k = 0; k < 2; k++) {
            const uint64_t n = sizes[k];
            uint64_t step = n / split;
            if (step < 1) step = 1;
            const uint64_t nsub = (n + step - 1) / step;
            J = nsub > J ? nsub : J;
            mstep = step > mstep ? step : mstep;
        }
    } else if (t == s.S) {
        tiles[t] = 0;
    }
    // one atomic per warp (65536 same-address atomics cost ~90 us)
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long j2 = __shfl_xor_sync(0xffffffffu, J, o);
        const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mstep, o);
        J = j2 > J ? j2 : J;
        mstep = m2 > mstep ? m2 : mstep;
    }
    if ((threadIdx.x & 31) == 0 && J) {
        atomicMax(&meta[0], J);
        atomicMax(&meta[1], mstep);
    }
}

// ---------------------------------------------------------------------------
// phases 1 and 2: fused tabulated walk + Boolean test, verdict bitmaps (the
// regular family in tile_search.cuh's throughput form, the classic family
// in classic_lockstep.cuh's)
// ---------------------------------------------------------------------------
struct Walk {  // per-lane stride-32 difference tables, in shared memory
    u128 g0, g1, h0;
};

// top W bits of (x mod 2^F), i.e. (x mod 2^F) >> (F - W), via one funnel
// shift: sh = 128 - F.  SH >= 0 fixes the shift at compile time (the
// pipeline's F = 96: a register pick and one funnel shift instead of a
// variable 128-bit shift).
template <int W, int SH = -1>
__device__ __forceinline__ uint64_t top_bits(u128 x, int sh) {
    const u128 y = SH >= 0 ? x << SH : x << sh;
    return W == 64 ? (uint64_t)(y >> 64) : (uint64_t)(y >> 96);
}

template <int W, int SH = -1>
struct WalkSrc {
    Walk* w;
    const u128* inc;  // per-warp constants in shared memory: {g2, h1}
    uint64_t pad_full, pad_last;
    uint32_t il, nd, nfull, nlast;
    int sh;
    __device__ __forceinline__ bool build(int k, uint64_t& a, uint64_t& b, uint64_t& eps, uint32_t& N) {
        const uint32_t i = il + 32u * (uint32_t)k;
        if (i >= nd) return false;
        const bool last = i == nd - 1;
        const u128 s0 = w->g0, s1 = w->h0, g1 = w->g1;
        const uint64_t pad = last ? pad_last : pad_full;
        const uint64_t wmask = W == 64 ? ~0ull : 0xFFFFFFFFull;
        a = top_bits<W, SH>(0 - s1, sh);
        b = (top_bits<W, SH>(s0, sh) + pad) & wmask;
        eps = 2 * pad;
        N = last ? nlast : nfull;
        // tabulated step: three multi-word additions per domain
        w->g0 = s0 + g1;
        w->g1 = g1 + inc[0];
        w->h0 = s1 + inc[1];
        return true;
    }
    // items k and k + 1 with one load and one store of the walk state (the
    // state stays in registers between the two tabulated steps)
    __device__ __forceinline__ void build2(int k, bool& v0, uint64_t& a0, uint64_t& b0, uint64_t& e0, uint32_t& N0,
                                           bool& v1, uint64_t& a1, uint64_t& b1, uint64_t& e1, uint32_t& N1) {
        const uint32_t i = il + 32u * (uint32_t)k;
        v0 = i < nd;
        v1 = i + 32u < nd;
        if (!v0) return;
        const uint64_t wmask = W == 64 ? ~0ull : 0xFFFFFFFFull;
        u128 s0 = w->g0, s1 = w->h0, g1 = w->g1;
        const u128 g2 = inc[0], h1 = inc[1];
        {
            const bool last = i == nd - 1;
            const uint64_t pad = last ? pad_last : pad_full;
            a0 = top_bits<W, SH>(0 - s1, sh);
            b0 = (top_bits<W, SH>(s0, sh) + pad) & wmask;
            e0 = 2 * pad;
            N0 = last ? nlast : nfull;
        }
        s0 += g1;
        g1 += g2;
        s1 += h1;
        {
            const bool last = i + 32u == nd - 1;
            const uint64_t pad = last ? pad_last : pad_full;
            a1 = top_bits<W, SH>(0 - s1, sh);
            b1 = (top_bits<W, SH>(s0, sh) + pad) & wmask;
            e1 = 2 * pad;
            N1 = last ? nlast : nfull;
        }
        w->g0 = s0 + g1;
        w->g1 = g1 + g2;
        w->h0 = s1 + h1;
    }
    __device__ __forceinline__ void done(int, bool, uint64_t, uint32_t) {}
};

// Tiles are handed out dynamically: a warp starts on tile warp0 and takes
// each further tile from a device counter (tile_ctr, zeroed by ws_prep),
// fetched one tile ahead so the atomic's latency hides behind the search.
// Per-tile times vary with the domains' iteration counts and rare exact
// repairs; a static grid-stride split left ~17 % of the warp slots idle at
// the end of the kernel.  The bitmap and tile_t are indexed by tile, so the
// output does not depend on which warp ran which tile.
// CL: 0 the regular family, 1 + mode the classic family (classic_lockstep.cuh)
template <int W, int SH, int PL, int CL = 0>
__global__ void __launch_bounds__(128, HRB_P1_MINB) phase1_reg_kernel(SliceDev s, int algo, const uint64_t* tile_base,
                                                          uint32_t* bitmap, uint32_t* tile_t,
                                                          unsigned long long* iter_sum,
                                                          unsigned long long* tile_ctr) {
    __shared__ Walk walks[128];
    __shared__ u128 incs[4][2];
    __shared__ hrb::ClQueue clq[CL ? 4 : 1];  // the classic family's per-warp queues
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // work unit: a tile, or a quarter of one (PL = 2) for slices with too
    // few tiles to keep every warp busy to the end
    const uint64_t units = tile_base[s.S] << PL;
    constexpr uint32_t nper = (uint32_t)NU >> PL;
    unsigned long long iters = 0;
    uint32_t known = 0;  // streamed upload: chunks known to have landed
    WalkSrc<W, SH> src;
    src.w = &walks[threadIdx.x];
    src.inc = incs[threadIdx.x >> 5];
    src.sh = 128 - s.F;
    uint64_t u = warp0;
    while (u < units) {
        unsigned long long next = 0;
        if (lane == 0) next = nwarps + atomicAdd(tile_ctr, 1ull);
        const uint64_t gw = u >> PL;
        const uint32_t k0 = (uint32_t)(u & ((1u << PL) - 1)) * nper;  // first item of the part
        const int64_t t = locate_super(tile_base, s.S, gw);
        const uint64_t tile = gw - tile_base[t];
        wait_super(s, t, known);
        const u128 c00 = coef_res<true>(s, t, 0), c01 = coef_res<true>(s, t, 1), c02 = coef_res<true>(s, t, 2);
        const u128 c10 = coef_res<true>(s, t, 3), c11 = coef_res<true>(s, t, 4);
        const u128 G = ld128cg(s, s.G, t);
        const u128 s2a = s.delta >= 2 ? ld128cg(s, s.s2abs, t) : (u128)0;
        src.nd = __ldg(&s.n_dom[t]);
        src.nfull = __ldg(&s.dom_n[t]);
        src.nlast = __ldg(&s.last_n[t]);
        src.pad_full = pad_of(G, s2a, src.nfull, s.F, W);
        src.pad_last = pad_of(G, s2a, src.nlast, s.F, W);
        const uint64_t il = tile * TILE + 32 * k0 + lane;
        src.il = (uint32_t)il;
        __syncwarp();
        src.w->g0 = c00 + c01 * (u128)il + c02 * (u128)binom2(il);
        src.w->g1 = (c01 << 5) + c02 * (u128)(32 * il + 496);
        src.w->h0 = c10 + c11 * (u128)il;
        if (lane == 0) {
            incs[threadIdx.x >> 5][0] = c02 << 10;
            incs[threadIdx.x >> 5][1] = c11 << 5;
        }
        __syncwarp();
        unsigned long long its = 0;
        uint32_t fails;
        if constexpr (CL != 0)
            fails = hrb::lane_items_classic_m<W, NU, CL - 1>(src, &clq[threadIdx.x >> 5], &its, nper);
        else
            fails = hrb::lane_items<W, NU>(src, &its, algo == hrb::ALGO_REGULAR_UNROLLED, nper);
        iters += its;
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < NU; k++) {
            uint32_t wd = __ballot_sync(0xffffffffu, (fails >> k) & 1u);
            if (lane == k) mine = wd;
        }
        if (lane < nper) bitmap[gw * NU + k0 + lane] = mine;
        if (lane == 0) tile_t[gw] = (uint32_t)t;
        u = __shfl_sync(0xffffffffu, next, 0);
    }
    for (int o = 16; o > 0; o >>= 1) iters += __shfl_xor_sync(0xffffffffu, iters, o);
    if (iter_sum && lane == 0 && iters) atomicAdd(iter_sum, iters);
}

// Phase 2, one failing domain per lane: its subdomains j = 0..J-1 are the
// lane's items.  The shifted polynomials (straightforward_shift by j*step,
// polygen.py:143-158) are walked with tabulated differences of stride
// `step`: t0 += dt0, dt0 += s2 step^2, t1 += s2 step (exact mod 2^128).
template <int W, int SH = -1>
struct SubWalkSrc {
    u128 t0, dt0, d2, t1, dt1;
    uint64_t pad_full, pad_last;
    uint32_t nsub, step, last_cnt;
    int sh, base;  // base: first sub index of the current 32-item chunk
    __device__ __forceinline__ bool build(int k, uint64_t& a, uint64_t& b, uint64_t& eps, uint32_t& N) {
        const uint32_t j = (uint32_t)(base + k);
        if (j >= nsub) return false;
        const bool last = j == nsub - 1;
        const uint64_t pad = last ? pad_last : pad_full;
        const uint64_t wmask = W == 64 ? ~0ull : 0xFFFFFFFFull;
        a = top_bits<W, SH>(0 - t1, sh);
        b = (top_bits<W, SH>(t0, sh) + pad) & wmask;
        eps = 2 * pad;
        N = last ? last_cnt : step;
        t0 += dt0;
        dt0 += d2;
        t1 += dt1;
        return true;
    }
    __device__ __forceinline__ void build2(int k, bool& v0, uint64_t& a0, uint64_t& b0, uint64_t& e0, uint32_t& N0,
                                           bool& v1, uint64_t& a1, uint64_t& b1, uint64_t& e1, uint32_t& N1) {
        v0 = build(k, a0, b0, e0, N0);
        v1 = build(k + 1, a1, b1, e1, N1);
    }
    __device__ __forceinline__ void done(int, bool, uint64_t, uint32_t) {}
};

template <int W, int SH, int CL = 0>  // CL as in phase1_reg_kernel
__global__ void __launch_bounds__(128, HRB_P2_MINB) phase2_reg_kernel(SliceDev s, int split, const uint64_t* fail_ids,
                                                          const uint32_t* fail_t, const uint64_t* fail_count,
                                                          uint64_t fail_cap, unsigned long long* meta,
                                                          uint32_t* bitmap) {
    __shared__ hrb::ClQueue clq[CL ? 4 : 1];  // the classic family's per-warp queues
    uint64_t nf = *fail_count;
    if (nf > fail_cap) nf = fail_cap;
    const uint32_t J = (uint32_t)meta[0];
    const uint32_t wpd = (J + 31) >> 5;  // bitmap words per failing domain
    SubWalkSrc<W, SH> src;
    src.sh = 128 - s.F;
    // whole warps iterate together so the lockstep pairs stay converged
    const uint64_t nf_pad = (nf + 31) & ~31ull;
    // a warp takes 32 consecutive failing domains at a time, the first chunk
    // by its id and the rest from a device counter (meta[5], zeroed by
    // ws_prep), fetched one chunk ahead (see phase1_reg_kernel)
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t chunk = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    while (32 * chunk < nf_pad) {
        unsigned long long next = 0;
        if (lane == 0) next = nwarps + atomicAdd(&meta[5], 1ull);
        const uint64_t f = 32 * chunk + lane;
        const bool valid = f < nf;
        src.nsub = 0;
        if (valid) {
            const uint64_t id = fail_ids[f];
            const int64_t t = fail_t[f];
            const uint64_t i = id - __ldg(&s.dom_base[t]);
            const uint64_t n = domain_size(s, t, i);
            uint64_t step = udiv_small(n, (uint32_t)split);
            if (step < 1) step = 1;
            const uint64_t nsub = udiv_small(n + step - 1, (uint32_t)step);
            const u128 c00 = coef_res(s, t, 0), c01 = coef_res(s, t, 1), c02 = coef_res(s, t, 2);
            const u128 c10 = coef_res(s, t, 3), c11 = coef_res(s, t, 4);
            const u128 s2 = s.delta >= 2 ? coef_res(s, t, 5) : (u128)0;
            const u128 s0 = c00 + c01 * (u128)i + c02 * (u128)binom2(i);  // P_{t+i} = r_j(i)
            const u128 s1 = c10 + c11 * (u128)i;
            const u128 G = ld128(s.G, s.S, t);
            const u128 s2a = s.delta >= 2 ? ld128(s.s2abs, s.S, t) : (u128)0;
            src.t0 = s0;
            src.dt0 = s1 * (u128)step + s2 * (u128)binom2(step);
            src.d2 = s2 * (u128)(step * step);
            src.t1 = s1;
            src.dt1 = s2 * (u128)step;
            src.nsub = (uint32_t)nsub;
            src.step = (uint32_t)step;
            src.last_cnt = (uint32_t)(n - (nsub - 1) * step);
            src.pad_full = pad_of(G, s2a, step, s.F, W);
            src.pad_last = pad_of(G, s2a, src.last_cnt, s.F, W);
        }
        for (uint32_t c = 0; c < wpd; c++) {
            src.base = 32 * c;
            unsigned long long its = 0;
            const uint32_t nit = src.nsub > 32 * c ? src.nsub - 32 * c : 0;
            uint32_t fails;
            if constexpr (CL != 0)
                fails = hrb::lane_items_classic_m<W, 32, CL - 1>(src, &clq[threadIdx.x >> 5], &its, nit);
            else
                fails = hrb::lane_items<W, 32>(src, &its, false, nit);
            if (valid) bitmap[f * wpd + c] = fails;
        }
        chunk = __shfl_sync(0xffffffffu, next, 0);
    }
}

// t of each listed slice-local id (standalone ABI calls; the fused path gets
// t from the compaction instead)
__global__ void locate_kernel(const uint64_t* base, int64_t S, const uint64_t* ids, const uint64_t* count,
                              uint64_t cap, int shift, uint32_t* out_t) {
    uint64_t n = *count;
    if (n > cap) n = cap;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        out_t[k] = (uint32_t)locate_super(base, S, ids[k] >> shift);
}

// ---------------------------------------------------------------------------
// phase 3: exhaustive second-order walk of surviving subdomains
// ---------------------------------------------------------------------------
struct Cand {
    uint64_t m, dist, dom, item;
    uint32_t rank;
};

// meta[2] <- the phase-3 chunk for this launch: halve from CHUNK3_MAX while
// the item count (subdomains x chunks per subdomain) stays below min_items.
__global__ void chunk3_kernel(unsigned long long* meta, const uint64_t* sub_count, uint64_t sub_cap,
                              uint64_t min_items) {
    uint64_t ns = *sub_count;
    if (ns > sub_cap) ns = sub_cap;
    const uint64_t maxstep = meta[1];
    uint64_t chunk = CHUNK3_MAX;
    while (chunk > CHUNK3_MIN && ns * ((maxstep + chunk - 1) / chunk) < min_items) chunk >>= 1;
    meta[2] = chunk;
}

// Phase 3 walk, scaled form: with sh = 128 - F the registers hold
// V = (v + window - 1) 2^sh, D1 = d1 2^sh, D2 = d2 2^sh, so the mod-2^F
// walk of pipeline.py:291-292 is plain 128-bit wraparound and the
// two-sided window test of pipeline.py:281 (v < window or v > 2^F - window)
// is the single unsigned compare V < (2 window - 1) 2^sh.  Hits are rare
// (~2 eps' per argument): the hot loop only ORs a conservative test on the
// top 64 bits over 32 arguments; when some lane of the warp flagged, the
// warp re-walks those 32 arguments exactly and appends the candidates with
// __ballot_sync/__popc (one atomic per warp).
#ifndef HRB_P3_MINB
#define HRB_P3_MINB 3
#endif
#ifndef P3BLK
#define P3BLK 64  // phase-3 proxy block: arguments per exact 128-bit advance
#endif
template <bool NARROW>
__global__ void __launch_bounds__(256, HRB_P3_MINB) phase3_kernel(SliceDev s, int split, const uint64_t* sub_keys,
                                                     const uint32_t* sub_t, const uint64_t* sub_count,
                                                     uint64_t sub_cap, const unsigned long long* meta,
                                                     uint32_t* item_counts, Cand* app, unsigned long long* app_count,
                                                     uint64_t app_cap) {
    const int lane = threadIdx.x & 31;
    const uint64_t maxstep = meta[1];
    const uint32_t CHUNK3 = (uint32_t)meta[2];
    const uint64_t CH = (maxstep + CHUNK3 - 1) / CHUNK3;
    uint64_t ns = *sub_count;
    if (ns > sub_cap) ns = sub_cap;
    const uint64_t n_items = ns * CH;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const int F = s.F;
    const int sh = 128 - F;
    for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; base < n_items; base += stride) {
        const uint64_t g = base + lane;
        uint32_t len = 0;
        uint64_t mbase = 0, dom = 0;
        u128 V = 0, D1 = 0, D2 = 0, K = 0, wm1 = 0;
        if (g < n_items) {
            const uint64_t r = udiv_small(g, (uint32_t)CH), c = g - r * CH;
            const uint64_t key = sub_keys[r];
            dom = key >> 8;
            const uint64_t j = key & 255;
            const int64_t t = sub_t[r];
            const uint64_t i = dom - s.dom_base[t];
            const uint64_t n = domain_size(s, t, i);
            uint64_t step = udiv_small(n, (uint32_t)split);
            if (step < 1) step = 1;
            const uint64_t start = j * step;
            const uint64_t cnt = n - start < step ? n - start : step;
            const uint64_t x0 = c * CHUNK3;
            if (x0 < cnt) {
                len = (uint32_t)(cnt - x0 < CHUNK3 ? cnt - x0 : CHUNK3);
                const uint64_t o = start + x0;
                const u128 c00 = coef_res(s, t, 0), c01 = coef_res(s, t, 1), c02 = coef_res(s, t, 2);
                const u128 c10 = coef_res(s, t, 3), c11 = coef_res(s, t, 4);
                const u128 s2 = s.delta >= 2 ? coef_res(s, t, 5) : (u128)0;
                const u128 s0 = c00 + c01 * (u128)i + c02 * (u128)binom2(i);
                const u128 s1 = c10 + c11 * (u128)i;
                const u128 window = ld128(s.G, s.S, t) + 1;  // ceil(eps' 2^F) + 1 (pipeline.py:274)
                wm1 = window - 1;
                V = (s0 + s1 * (u128)o + s2 * (u128)binom2(o) + wm1) << sh;  // P(o), shifted origin
                D1 = (s1 + s2 * (u128)o) << sh;                             // Delta P(o)
                D2 = s2 << sh;
                K = (2 * window - 1) << sh;
                mbase = __ldg(&s.m0[t]) + i * (uint64_t)__ldg(&s.dom_n[t]) + o;
            }
        }
        // Hot loop on a 32-bit proxy of the top word: u = top32(V) + MARGIN,
        // stepped by the top words of D1 and D2.  Floors of sums exceed sums
        // of floors by at most one per term, so after x < 32 steps the true
        // top word T(x) lies in [u - MARGIN, u - MARGIN + x + C(x,2)] (<= 496):
        // V < K  =>  T <= top32(K)  =>  u <= top32(K) + MARGIN (no wrap on
        // either side).  Two instructions per argument; the exact 128-bit
        // state advances once per 32 arguments and a block is re-examined
        // only when some lane's proxy flagged it.
        // blocks of P3BLK arguments (a power of two dividing CHUNK3); the
        // proxy's floor error after x < P3BLK steps is at most x + C(x, 2)
        constexpr uint32_t BLK = P3BLK, LBLK = BLK == 64 ? 6 : 5;
        constexpr uint32_t MARGIN = BLK == 64 ? 4096 : 1024;
        using Mask = typename std::conditional<BLK == 64, unsigned long long, uint32_t>::type;
        const uint32_t Ktop = (uint32_t)(K >> 96);
        const uint32_t KtopM = Ktop > 0xFFFFFFFFu - MARGIN ? 0xFFFFFFFFu : Ktop + MARGIN;
        const uint32_t e32 = (uint32_t)(D2 >> 96), e2x32 = 2 * e32;
        const u128 D2xB = D2 << LBLK, D2xCB = D2 * (u128)(BLK * (BLK - 1) / 2);
        uint32_t rank = 0;
        for (uint32_t x0 = 0; x0 < CHUNK3; x0 += BLK) {
            const u128 V0 = V, D10 = D1;
            uint32_t u = (uint32_t)(V >> 96) + MARGIN, d = (uint32_t)(D1 >> 96);
#ifndef HRB_P3_Q
#define HRB_P3_Q 4  // proxy minima per quarter of the block (A/B: DESIGN.md 9b)
#endif
            constexpr uint32_t NQ = HRB_P3_Q, QL = BLK / NQ;
            uint32_t lq[NQ];
#pragma unroll
            for (uint32_t q = 0; q < NQ; q++) lq[q] = 0xFFFFFFFFu;
            // two arguments per iteration, four instructions: t = u(x+1);
            // a three-input min; u(x+2) = t + d + e as one three-input add
            // (IADD3 -- an ALU-pipe op; two-input adds alone all went to the
            // FMA pipe as IMAD.IADD and throttled it); d(x+2) = d + 2e
#ifndef HRB_P3_ASM
#define HRB_P3_ASM 1
#endif
#pragma unroll
            for (uint32_t x = 0; x < BLK; x += 2) {
#if HRB_P3_ASM
                // as opaque adds: the front end otherwise re-associates the
                // chain into one add per argument for u and one for d (all
                // IMAD.IADD, FMA pipe) and, seeing the replay below compute
                // the same values, keeps them in local memory for it
                uint32_t t;
                asm("add.u32 %0, %1, %2;" : "=r"(t) : "r"(u), "r"(d));
                lq[x / QL] = min(lq[x / QL], min(u, t));
                asm("{\n\t.reg .u32 w;\n\tadd.u32 w, %1, %2;\n\tadd.u32 %0, w, %3;\n\t}"
                    : "=r"(u) : "r"(t), "r"(d), "r"(e32));
                asm("add.u32 %0, %0, %1;" : "+r"(d) : "r"(e2x32));
#else
                const uint32_t t = u + d;
                lq[x / QL] = min(lq[x / QL], min(u, t));
                u = t + d + e32;
                d += e2x32;
#endif
            }
            V += (D1 << LBLK) + D2xCB;  // exact: BLK steps of V += D1, D1 += D2
            D1 += D2xB;
            uint32_t lo_top = lq[0];
#pragma unroll
            for (uint32_t q = 1; q < NQ; q++) lo_top = min(lo_top, lq[q]);
            const bool any = x0 < len && lo_top <= KtopM;
            if (__any_sync(0xffffffffu, any)) {
                // rare: replay the proxy over the block into a per-lane mask
                // of the arguments it flags (the true hits, and near-misses
                // within MARGIN of the window's top word; no votes), then
                // evaluate exactly -- V(x) = V0 + x D1 + C(x,2) D2 -- one
                // flagged argument per lane per round, lowest first, so each
                // lane appends its hits in argument order
                Mask fl = 0;
                if (any) {
                    // only the quarters whose proxy minimum flagged; the proxy
                    // at a quarter's start in closed form (mod 2^32, the same
                    // values the walk stepped through)
                    const uint32_t u0 = (uint32_t)(V0 >> 96) + MARGIN, d0 = (uint32_t)(D10 >> 96);
#pragma unroll
                    for (uint32_t q = 0; q < NQ; q++) {
                        if (lq[q] <= KtopM) {
                            const uint32_t xq = q * QL;
                            uint32_t pu = u0 + xq * d0 + ((xq * (xq - 1)) >> 1) * e32, pd = d0 + xq * e32;
                            using QMask = typename std::conditional<(QL > 32), Mask, uint32_t>::type;
                            QMask m = 0;
#pragma unroll
                            for (uint32_t x = 0; x < QL; x++) {
                                m |= pu <= KtopM ? ((QMask)1 << x) : (QMask)0;
                                pu += pd;
                                pd += e32;
                            }
                            fl |= (Mask)m << xq;
                        }
                    }
                    const uint32_t lim = len - x0;  // > 0 here
                    if (lim < BLK) fl &= ((Mask)1 << lim) - 1;
                }
                while (__any_sync(0xffffffffu, fl != 0)) {
                    bool hit = false;
                    u128 v = 0;
                    uint32_t x = 0;
                    if (fl) {
                        x = BLK == 64 ? (uint32_t)(__ffsll((long long)fl) - 1) : (uint32_t)(__ffs((int)fl) - 1);
                        fl &= fl - 1;
                        v = V0 + D10 * (u128)x + D2 * (u128)((x * (x - 1)) >> 1);
                        hit = v < K;
                    }
                    const uint32_t ball = __ballot_sync(0xffffffffu, hit);
                    if (ball) {
                        const int leader = __ffs(ball) - 1;
                        unsigned long long pos = 0;
                        if (lane == leader) pos = atomicAdd(app_count, (unsigned long long)__popc(ball));
                        pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(ball & ((1u << lane) - 1));
                        if (hit) {
                            if (pos < app_cap) {
                                const u128 vv = ((v >> sh) - wm1) & mask_f(F);
                                const u128 comp = (F >= 128 ? (u128)0 - vv : (((u128)1 << F) - vv)) & mask_f(F);
                                const u128 dist = (vv == 0 || vv < comp) ? vv : comp;
                                Cand cd;
                                cd.m = mbase + x0 + x;
                                cd.dist = F >= 64 ? (uint64_t)(dist >> (F - 64)) : (uint64_t)(dist << (64 - F));
                                cd.dom = dom;
                                cd.item = g;
                                cd.rank = rank;
                                app[pos] = cd;
                            }
                            rank++;
                        }
                    }
                }
            }
        }
        if (g < n_items) item_counts[g] = rank;
    }
}

// ---------------------------------------------------------------------------
// ordered compaction: 3-kernel reduce / scan / scatter with a device-side size
// ---------------------------------------------------------------------------
struct P1Compact {  // bitmap of padded domain indices -> slice-local ids (+ t)
    const uint32_t* bm;
    const uint64_t* tile_base;
    const uint32_t* tile_t;
    const uint64_t* dom_base;
    int64_t S;
    uint64_t* out;
    uint32_t* out_t;
    uint64_t cap;
    __device__ uint64_t size() const { return tile_base[S] * NU; }
    __device__ uint32_t count(uint64_t w) const { return __popc(bm[w]); }
    __device__ void emit(uint64_t w, uint64_t off) const {
        uint32_t x = bm[w];
        const uint64_t gw = w / NU;
        const uint32_t t = tile_t[gw];
        const uint64_t first = dom_base[t] + (gw - tile_base[t]) * TILE + (w - gw * NU) * 32;
        while (x) {
            int b = __ffs(x) - 1;
            x &= x - 1;
            if (off < cap) {
                out[off] = first + b;
                out_t[off] = t;
            }
            off++;
        }
    }
    // the same items into a shared staging area (k = 0.. at sid / st)
    __device__ void stage(uint64_t w, uint64_t* sid, uint32_t* st) const {
        uint32_t x = bm[w];
        const uint64_t gw = w / NU;
        const uint32_t t = tile_t[gw];
        const uint64_t first = dom_base[t] + (gw - tile_base[t]) * TILE + (w - gw * NU) * 32;
        for (int k = 0; x; k++) {
            int b = __ffs(x) - 1;
            x &= x - 1;
            sid[k] = first + b;
            st[k] = t;
        }
    }
};

struct P2Compact {  // bitmap over (f, j) items -> (id << 8 | j) (+ t)
    const uint32_t* bm;
    const uint64_t* fail_ids;
    const uint32_t* fail_t;
    const uint64_t* fail_count;
    uint64_t fail_cap;
    const unsigned long long* meta;
    uint64_t* out;
    uint32_t* out_t;
    uint64_t cap;
    __device__ uint64_t size() const {
        uint64_t nf = *fail_count;
        if (nf > fail_cap) nf = fail_cap;
        return nf * ((meta[0] + 31) >> 5);
    }
    __device__ uint32_t count(uint64_t w) const { return __popc(bm[w]); }
    __device__ void emit(uint64_t w, uint64_t off) const {
        uint32_t x = bm[w];
        const uint64_t wpd = (meta[0] + 31) >> 5;
        const uint64_t f = w / wpd;
        const uint64_t j0 = (w - f * wpd) * 32;
        const uint64_t id = fail_ids[f];
        const uint32_t t = fail_t[f];
        while (x) {
            int b = __ffs(x) - 1;
            x &= x - 1;
            if (off < cap) {
                out[off] = (id << 8) | (j0 + b);
                out_t[off] = t;
            }
            off++;
        }
    }
    __device__ void stage(uint64_t w, uint64_t* sid, uint32_t* st) const {
        uint32_t x = bm[w];
        const uint64_t wpd = (meta[0] + 31) >> 5;
        const uint64_t f = w / wpd;
        const uint64_t j0 = (w - f * wpd) * 32;
        const uint64_t id = fail_ids[f];
        const uint32_t t = fail_t[f];
        for (int k = 0; x; k++) {
            int b = __ffs(x) - 1;
            x &= x - 1;
            sid[k] = (id << 8) | (j0 + b);
            st[k] = t;
        }
    }
};

struct P3Offsets {  // per-item candidate counts -> per-item output offsets
    const uint32_t* counts;
    const uint64_t* sub_count;
    uint64_t sub_cap;
    const unsigned long long* meta;
    uint64_t* offs;
    __device__ uint64_t size() const {
        uint64_t ns = *sub_count;
        if (ns > sub_cap) ns = sub_cap;
        return ns * ((meta[1] + meta[2] - 1) / meta[2]);
    }
    __device__ uint32_t count(uint64_t i) const { return counts[i]; }
    __device__ void emit(uint64_t i, uint64_t off) const { offs[i] = off; }
};

template <class Fn>
__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(Fn fn, uint64_t* block_sums) {
    using BR = cub::BlockReduce<unsigned long long, SCAN_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const uint64_t n = fn.size();
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    unsigned long long acc = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += SCAN_THREADS) acc += fn.count(i);
    unsigned long long tot = BR(tmp).Sum(acc);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_blocks_kernel(uint64_t* block_sums, int nb, uint64_t* total) {
    using BS = cub::BlockScan<unsigned long long, 1024>;
    __shared__ typename BS::TempStorage tmp;
    unsigned long long v = threadIdx.x < nb ? block_sums[threadIdx.x] : 0, excl, agg;
    BS(tmp).ExclusiveSum(v, excl, agg);
    if (threadIdx.x < nb) block_sums[threadIdx.x] = excl;
    if (threadIdx.x == 0) *total = agg;
}

template <class Fn>
__global__ void __launch_bounds__(SCAN_THREADS) scan_scatter_kernel(Fn fn, const uint64_t* block_offs) {
    using BS = cub::BlockScan<unsigned long long, SCAN_THREADS>;
    __shared__ typename BS::TempStorage tmp;
    const uint64_t n = fn.size();
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    unsigned long long run = block_offs[blockIdx.x];
    for (uint64_t base = lo; base < hi; base += SCAN_THREADS) {
        const uint64_t i = base + threadIdx.x;
        unsigned long long c = i < hi ? fn.count(i) : 0, excl, agg;
        BS(tmp).ExclusiveSum(c, excl, agg);
        if (i < hi && c) fn.emit(i, run + excl);
        run += agg;
        __syncthreads();
    }
}

// scan_scatter_kernel for the id lists (P1Compact / P2Compact): a round's
// items are staged in shared memory in output order and then stored by the
// whole block, contiguously (each thread writing its own few ids at its own
// offset gave ~1 TB/s of scattered 8-byte stores); a round with more items
// than the staging area holds emits directly.
constexpr int STAGE_ITEMS = 2048;

template <class Fn>
__global__ void __launch_bounds__(SCAN_THREADS) scan_scatter_staged_kernel(Fn fn, const uint64_t* block_offs) {
    using BS = cub::BlockScan<unsigned long long, SCAN_THREADS>;
    __shared__ typename BS::TempStorage tmp;
    __shared__ uint64_t sid[STAGE_ITEMS];
    __shared__ uint32_t st[STAGE_ITEMS];
    const uint64_t n = fn.size();
    const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    unsigned long long run = block_offs[blockIdx.x];
    for (uint64_t base = lo; base < hi; base += SCAN_THREADS) {
        const uint64_t i = base + threadIdx.x;
        unsigned long long c = i < hi ? fn.count(i) : 0, excl, agg;
        BS(tmp).ExclusiveSum(c, excl, agg);
        if (agg <= STAGE_ITEMS) {
            if (c) fn.stage(i, sid + excl, st + excl);
            __syncthreads();
            for (uint32_t k = threadIdx.x; k < agg; k += SCAN_THREADS) {
                const uint64_t off = run + k;
                if (off < fn.cap) {
                    fn.out[off] = sid[k];
                    fn.out_t[off] = st[k];
                }
            }
        } else if (c) {
            fn.emit(i, run + excl);
        }
        run += agg;
        __syncthreads();
    }
}

__global__ void scatter3_kernel(const Cand* app, const unsigned long long* app_count, uint64_t app_cap,
                                const uint64_t* offs, uint64_t* out_m, uint64_t* out_dist, uint64_t* out_dom,
                                uint64_t cap) {
    uint64_t n = *app_count;
    if (n > app_cap) n = app_cap;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const Cand c = app[k];
        const uint64_t pos = offs[c.item] + c.rank;
        if (pos < cap) {
            out_m[pos] = c.m;
            out_dist[pos] = c.dist;
            out_dom[pos] = c.dom;
        }
    }
}

// ---------------------------------------------------------------------------
// full-width tabulated differences (domain_coefficient_sets parity)
// ---------------------------------------------------------------------------
// x += y over CL limbs with one add-with-carry chain (IADD3 / IADD3.X).
// ONE asm statement per chain: the carry flag does not survive between
// separate asm statements (the compiler may schedule another chain's
// add.cc in between), so every width gets its own single-statement body.
template <int CL>
__device__ __forceinline__ void addc_chain(uint32_t (&x)[CL], const uint32_t (&y)[CL]);

template <>
__device__ __forceinline__ void addc_chain<1>(uint32_t (&x)[1], const uint32_t (&y)[1]) {
    x[0] += y[0];
}

template <>
__device__ __forceinline__ void addc_chain<2>(uint32_t (&x)[2], const uint32_t (&y)[2]) {
    asm("add.cc.u32 %0, %0, %2;\n\t"
        "addc.u32 %1, %1, %3;"
        : "+r"(x[0]), "+r"(x[1])
        : "r"(y[0]), "r"(y[1]));
}

template <>
__device__ __forceinline__ void addc_chain<3>(uint32_t (&x)[3], const uint32_t (&y)[3]) {
    asm("add.cc.u32 %0, %0, %3;\n\t"
        "addc.cc.u32 %1, %1, %4;\n\t"
        "addc.u32 %2, %2, %5;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]));
}

template <>
__device__ __forceinline__ void addc_chain<4>(uint32_t (&x)[4], const uint32_t (&y)[4]) {
    asm("add.cc.u32 %0, %0, %4;\n\t"
        "addc.cc.u32 %1, %1, %5;\n\t"
        "addc.cc.u32 %2, %2, %6;\n\t"
        "addc.u32 %3, %3, %7;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]));
}

template <>
__device__ __forceinline__ void addc_chain<5>(uint32_t (&x)[5], const uint32_t (&y)[5]) {
    asm("add.cc.u32 %0, %0, %5;\n\t"
        "addc.cc.u32 %1, %1, %6;\n\t"
        "addc.cc.u32 %2, %2, %7;\n\t"
        "addc.cc.u32 %3, %3, %8;\n\t"
        "addc.u32 %4, %4, %9;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]));
}

template <>
__device__ __forceinline__ void addc_chain<6>(uint32_t (&x)[6], const uint32_t (&y)[6]) {
    asm("add.cc.u32 %0, %0, %6;\n\t"
        "addc.cc.u32 %1, %1, %7;\n\t"
        "addc.cc.u32 %2, %2, %8;\n\t"
        "addc.cc.u32 %3, %3, %9;\n\t"
        "addc.cc.u32 %4, %4, %10;\n\t"
        "addc.u32 %5, %5, %11;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]));
}

template <>
__device__ __forceinline__ void addc_chain<7>(uint32_t (&x)[7], const uint32_t (&y)[7]) {
    asm("add.cc.u32 %0, %0, %7;\n\t"
        "addc.cc.u32 %1, %1, %8;\n\t"
        "addc.cc.u32 %2, %2, %9;\n\t"
        "addc.cc.u32 %3, %3, %10;\n\t"
        "addc.cc.u32 %4, %4, %11;\n\t"
        "addc.cc.u32 %5, %5, %12;\n\t"
        "addc.u32 %6, %6, %13;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]));
}

template <>
__device__ __forceinline__ void addc_chain<8>(uint32_t (&x)[8], const uint32_t (&y)[8]) {
    asm("add.cc.u32 %0, %0, %8;\n\t"
        "addc.cc.u32 %1, %1, %9;\n\t"
        "addc.cc.u32 %2, %2, %10;\n\t"
        "addc.cc.u32 %3, %3, %11;\n\t"
        "addc.cc.u32 %4, %4, %12;\n\t"
        "addc.cc.u32 %5, %5, %13;\n\t"
        "addc.cc.u32 %6, %6, %14;\n\t"
        "addc.u32 %7, %7, %15;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]));
}

template <>
__device__ __forceinline__ void addc_chain<9>(uint32_t (&x)[9], const uint32_t (&y)[9]) {
    asm("add.cc.u32 %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32 %8, %8, %17;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]));
}

template <>
__device__ __forceinline__ void addc_chain<10>(uint32_t (&x)[10], const uint32_t (&y)[10]) {
    asm("add.cc.u32 %0, %0, %10;\n\t"
        "addc.cc.u32 %1, %1, %11;\n\t"
        "addc.cc.u32 %2, %2, %12;\n\t"
        "addc.cc.u32 %3, %3, %13;\n\t"
        "addc.cc.u32 %4, %4, %14;\n\t"
        "addc.cc.u32 %5, %5, %15;\n\t"
        "addc.cc.u32 %6, %6, %16;\n\t"
        "addc.cc.u32 %7, %7, %17;\n\t"
        "addc.cc.u32 %8, %8, %18;\n\t"
        "addc.u32 %9, %9, %19;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]));
}

template <>
__device__ __forceinline__ void addc_chain<11>(uint32_t (&x)[11], const uint32_t (&y)[11]) {
    asm("add.cc.u32 %0, %0, %11;\n\t"
        "addc.cc.u32 %1, %1, %12;\n\t"
        "addc.cc.u32 %2, %2, %13;\n\t"
        "addc.cc.u32 %3, %3, %14;\n\t"
        "addc.cc.u32 %4, %4, %15;\n\t"
        "addc.cc.u32 %5, %5, %16;\n\t"
        "addc.cc.u32 %6, %6, %17;\n\t"
        "addc.cc.u32 %7, %7, %18;\n\t"
        "addc.cc.u32 %8, %8, %19;\n\t"
        "addc.cc.u32 %9, %9, %20;\n\t"
        "addc.u32 %10, %10, %21;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]));
}

template <>
__device__ __forceinline__ void addc_chain<12>(uint32_t (&x)[12], const uint32_t (&y)[12]) {
    asm("add.cc.u32 %0, %0, %12;\n\t"
        "addc.cc.u32 %1, %1, %13;\n\t"
        "addc.cc.u32 %2, %2, %14;\n\t"
        "addc.cc.u32 %3, %3, %15;\n\t"
        "addc.cc.u32 %4, %4, %16;\n\t"
        "addc.cc.u32 %5, %5, %17;\n\t"
        "addc.cc.u32 %6, %6, %18;\n\t"
        "addc.cc.u32 %7, %7, %19;\n\t"
        "addc.cc.u32 %8, %8, %20;\n\t"
        "addc.cc.u32 %9, %9, %21;\n\t"
        "addc.cc.u32 %10, %10, %22;\n\t"
        "addc.u32 %11, %11, %23;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]));
}

template <>
__device__ __forceinline__ void addc_chain<13>(uint32_t (&x)[13], const uint32_t (&y)[13]) {
    asm("add.cc.u32 %0, %0, %13;\n\t"
        "addc.cc.u32 %1, %1, %14;\n\t"
        "addc.cc.u32 %2, %2, %15;\n\t"
        "addc.cc.u32 %3, %3, %16;\n\t"
        "addc.cc.u32 %4, %4, %17;\n\t"
        "addc.cc.u32 %5, %5, %18;\n\t"
        "addc.cc.u32 %6, %6, %19;\n\t"
        "addc.cc.u32 %7, %7, %20;\n\t"
        "addc.cc.u32 %8, %8, %21;\n\t"
        "addc.cc.u32 %9, %9, %22;\n\t"
        "addc.cc.u32 %10, %10, %23;\n\t"
        "addc.cc.u32 %11, %11, %24;\n\t"
        "addc.u32 %12, %12, %25;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]), "r"(y[12]));
}

template <>
__device__ __forceinline__ void addc_chain<14>(uint32_t (&x)[14], const uint32_t (&y)[14]) {
    asm("add.cc.u32 %0, %0, %14;\n\t"
        "addc.cc.u32 %1, %1, %15;\n\t"
        "addc.cc.u32 %2, %2, %16;\n\t"
        "addc.cc.u32 %3, %3, %17;\n\t"
        "addc.cc.u32 %4, %4, %18;\n\t"
        "addc.cc.u32 %5, %5, %19;\n\t"
        "addc.cc.u32 %6, %6, %20;\n\t"
        "addc.cc.u32 %7, %7, %21;\n\t"
        "addc.cc.u32 %8, %8, %22;\n\t"
        "addc.cc.u32 %9, %9, %23;\n\t"
        "addc.cc.u32 %10, %10, %24;\n\t"
        "addc.cc.u32 %11, %11, %25;\n\t"
        "addc.cc.u32 %12, %12, %26;\n\t"
        "addc.u32 %13, %13, %27;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12]), "+r"(x[13])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]), "r"(y[12]), "r"(y[13]));
}

template <>
__device__ __forceinline__ void addc_chain<15>(uint32_t (&x)[15], const uint32_t (&y)[15]) {
    asm("add.cc.u32 %0, %0, %15;\n\t"
        "addc.cc.u32 %1, %1, %16;\n\t"
        "addc.cc.u32 %2, %2, %17;\n\t"
        "addc.cc.u32 %3, %3, %18;\n\t"
        "addc.cc.u32 %4, %4, %19;\n\t"
        "addc.cc.u32 %5, %5, %20;\n\t"
        "addc.cc.u32 %6, %6, %21;\n\t"
        "addc.cc.u32 %7, %7, %22;\n\t"
        "addc.cc.u32 %8, %8, %23;\n\t"
        "addc.cc.u32 %9, %9, %24;\n\t"
        "addc.cc.u32 %10, %10, %25;\n\t"
        "addc.cc.u32 %11, %11, %26;\n\t"
        "addc.cc.u32 %12, %12, %27;\n\t"
        "addc.cc.u32 %13, %13, %28;\n\t"
        "addc.u32 %14, %14, %29;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12]), "+r"(x[13]), "+r"(x[14])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]), "r"(y[12]), "r"(y[13]), "r"(y[14]));
}

template <>
__device__ __forceinline__ void addc_chain<16>(uint32_t (&x)[16], const uint32_t (&y)[16]) {
    asm("add.cc.u32 %0, %0, %16;\n\t"
        "addc.cc.u32 %1, %1, %17;\n\t"
        "addc.cc.u32 %2, %2, %18;\n\t"
        "addc.cc.u32 %3, %3, %19;\n\t"
        "addc.cc.u32 %4, %4, %20;\n\t"
        "addc.cc.u32 %5, %5, %21;\n\t"
        "addc.cc.u32 %6, %6, %22;\n\t"
        "addc.cc.u32 %7, %7, %23;\n\t"
        "addc.cc.u32 %8, %8, %24;\n\t"
        "addc.cc.u32 %9, %9, %25;\n\t"
        "addc.cc.u32 %10, %10, %26;\n\t"
        "addc.cc.u32 %11, %11, %27;\n\t"
        "addc.cc.u32 %12, %12, %28;\n\t"
        "addc.cc.u32 %13, %13, %29;\n\t"
        "addc.cc.u32 %14, %14, %30;\n\t"
        "addc.u32 %15, %15, %31;"
        : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]), "+r"(x[7]), "+r"(x[8]), "+r"(x[9]), "+r"(x[10]), "+r"(x[11]), "+r"(x[12]), "+r"(x[13]), "+r"(x[14]), "+r"(x[15])
        : "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(y[4]), "r"(y[5]), "r"(y[6]), "r"(y[7]), "r"(y[8]), "r"(y[9]), "r"(y[10]), "r"(y[11]), "r"(y[12]), "r"(y[13]), "r"(y[14]), "r"(y[15]));
}

// r = x * m (mod 2^(32 CL)), two's complement x, unsigned 64-bit m
template <int CL>
__device__ __forceinline__ void mul_u64(uint32_t (&r)[CL], const uint32_t (&x)[CL], uint64_t m) {
    uint32_t acc[CL];
#pragma unroll
    for (int l = 0; l < CL; l++) acc[l] = 0;
    const uint32_t mw[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
#pragma unroll
    for (int h = 0; h < 2; h++) {
        uint64_t carry = 0;
#pragma unroll
        for (int l = 0; l + h < CL; l++) {
            uint64_t p = (uint64_t)x[l] * mw[h] + acc[l + h] + carry;
            acc[l + h] = (uint32_t)p;
            carry = p >> 32;
        }
    }
#pragma unroll
    for (int l = 0; l < CL; l++) r[l] = acc[l];
}

template <int CL>
__device__ __forceinline__ void load_coef_full(const SliceDev& s, int64_t t, int c, uint32_t (&x)[CL]) {
#pragma unroll
    for (int l = 0; l < CL; l++) x[l] = __ldg(&s.coef[((int64_t)c * CL + l) * s.S + t]);
}

template <int CL>
__global__ void __launch_bounds__(128) tabdiff_full_kernel(SliceDev s, const uint64_t* tile_base, int64_t n_total,
                                                          uint32_t* out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total_tiles = tile_base[s.S];
    for (uint64_t gw = warp0; gw < total_tiles; gw += nwarps) {
        const int64_t t = locate_super(tile_base, s.S, gw);
        const uint64_t tile = gw - tile_base[t];
        const uint32_t nd = __ldg(&s.n_dom[t]);
        const uint64_t il = tile * TILE + lane;
        uint32_t c[6][CL];
#pragma unroll
        for (int k = 0; k < 6; k++) load_coef_full<CL>(s, t, k, c[k]);
        // column[j][l]: l-th stride-32 difference of r_j at the lane's domain
        uint32_t g0[CL], g1[CL], g2[CL], h0[CL], h1[CL], z[CL], tmp[CL];
        // g0 = c00 + c01*il + c02*C(il,2)
#pragma unroll
        for (int l = 0; l < CL; l++) g0[l] = c[0][l];
        mul_u64<CL>(tmp, c[1], il);
        addc_chain<CL>(g0, tmp);
        mul_u64<CL>(tmp, c[2], binom2(il));
        addc_chain<CL>(g0, tmp);
        // g1 = 32 c01 + c02 (32 il + 496);  g2 = 1024 c02
        mul_u64<CL>(g1, c[1], 32);
        mul_u64<CL>(tmp, c[2], 32 * il + 496);
        addc_chain<CL>(g1, tmp);
        mul_u64<CL>(g2, c[2], 1024);
        // h0 = c10 + c11 il;  h1 = 32 c11
#pragma unroll
        for (int l = 0; l < CL; l++) h0[l] = c[3][l];
        mul_u64<CL>(tmp, c[4], il);
        addc_chain<CL>(h0, tmp);
        mul_u64<CL>(h1, c[4], 32);
#pragma unroll
        for (int l = 0; l < CL; l++) z[l] = s.delta >= 2 ? c[5][l] : 0u;
        const uint64_t gbase = s.dom_base[t];
        for (int k = 0; k < NU; k++) {
            const uint64_t i = il + 32 * (uint64_t)k;
            if (i < nd) {
                const uint64_t gi = gbase + i;
#pragma unroll
                for (int l = 0; l < CL; l++) {
                    out[((int64_t)0 * CL + l) * n_total + gi] = g0[l];
                    out[((int64_t)1 * CL + l) * n_total + gi] = h0[l];
                    out[((int64_t)2 * CL + l) * n_total + gi] = z[l];
                }
            }
            addc_chain<CL>(g0, g1);
            addc_chain<CL>(g1, g2);
            addc_chain<CL>(h0, h1);
        }
    }
}

// ---------------------------------------------------------------------------
// search batch
// ---------------------------------------------------------------------------
// run one search to completion; REG selects the family at compile time so a
// kernel instantiation carries only one loop body (register pressure)
template <int W, bool REG>
__device__ __forceinline__ hrb::Outcome search_one(int algo, int mode, const Problem& p, uint64_t n) {
    if (REG) {
        hrb::Outcome o = hrb::regular_search<W>(p.a, p.b, p.eps, n);
        if (algo == hrb::ALGO_REGULAR_UNROLLED) o.it = (o.it + 1) >> 1;
        return o;
    }
    return hrb::lefevre_search<W>(p.a, p.b, p.eps, n, mode);
}

template <int W, bool REG>
__global__ void __launch_bounds__(256) search_batch_kernel(int algo, int mode, int64_t n, const uint64_t* a,
                                                           const uint64_t* b, const uint64_t* eps,
                                                           const uint64_t* count, uint8_t* ok, uint64_t* d,
                                                           uint64_t* it, uint64_t* pl, uint8_t* ph) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        Problem p{a[i], b[i], eps[i]};
        hrb::Outcome o = search_one<W, REG>(algo, mode, p, count[i]);
        ok[i] = o.ok;
        d[i] = o.d;
        if (it) it[i] = o.it;
        pl[i] = o.pts_lo;
        ph[i] = (uint8_t)o.pts_hi;
    }
}

// Regular-family verdicts in the throughput form (tile_search.cuh): a warp
// takes 32 * NU consecutive problems, lane l the problems l, l + 32, ...,
// two in flight per lane in lockstep.  Counts >= 2^32 (outside the lockstep
// form's 32-bit counters) run through the general core in place.
template <int W>
struct ArraySrc {
    const uint64_t *a, *b, *eps, *cnt;
    uint8_t* ok;
    uint64_t *d, *it;
    int64_t n, base;
    bool unrolled;
    __device__ __forceinline__ bool build(int k, uint64_t& av, uint64_t& bv, uint64_t& ev, uint32_t& N) {
        const int64_t i = base + 32 * (int64_t)k;
        if (i >= n) return false;
        const uint64_t c = __ldg(&cnt[i]);
        if (c >> 32) {
            hrb::Outcome o = hrb::regular_search<W>(a[i], b[i], eps[i], c);
            ok[i] = o.ok;
            d[i] = o.d;
            if (it) it[i] = unrolled ? (o.it + 1) >> 1 : o.it;
            return false;
        }
        av = __ldg(&a[i]);
        bv = __ldg(&b[i]);
        ev = __ldg(&eps[i]);
        N = (uint32_t)c;
        return true;
    }
    __device__ __forceinline__ void build2(int k, bool& v0, uint64_t& a0, uint64_t& b0, uint64_t& e0, uint32_t& N0,
                                           bool& v1, uint64_t& a1, uint64_t& b1, uint64_t& e1, uint32_t& N1) {
        v0 = build(k, a0, b0, e0, N0);
        v1 = build(k + 1, a1, b1, e1, N1);
    }
    __device__ __forceinline__ void done(int k, bool okv, uint64_t dv, uint32_t itv) {
        const int64_t i = base + 32 * (int64_t)k;
        ok[i] = okv;
        d[i] = dv;
        if (it) it[i] = itv;
    }
};

// NUV problems per lane: the phases' NU for large batches; small batches
// (config 2's 2^17 problems) take 2 per lane so that they still fill the GPU
template <int W, int NUV>
__global__ void __launch_bounds__(128, HRB_P1_MINB) search_verdict_kernel(int algo, int64_t n, const uint64_t* a,
                                                                          const uint64_t* b, const uint64_t* eps,
                                                                          const uint64_t* count, uint8_t* ok,
                                                                          uint64_t* d, uint64_t* it) {
    constexpr int TV = 32 * NUV;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t tiles = (n + TV - 1) / TV;
    ArraySrc<W> src{a, b, eps, count, ok, d, it, n, 0, algo == hrb::ALGO_REGULAR_UNROLLED};
    for (int64_t t = warp0; t < tiles; t += nwarps) {
        src.base = t * TV + lane;
        unsigned long long its = 0;
        hrb::lane_items<W, NUV>(src, &its, src.unrolled);
    }
}

// Same searches with the branch-decision stream of every problem recorded
// (the reference cores' `trace` argument): bits LSB-first in
// trace[i * wpp ...], the full decision count in trace_len[i] (decisions
// past wpp * 64 are counted but not stored).
template <int W>
__global__ void __launch_bounds__(256) search_trace_kernel(int algo, int mode, int64_t n, const uint64_t* a,
                                                           const uint64_t* b, const uint64_t* eps,
                                                           const uint64_t* count, uint8_t* ok, uint64_t* d,
                                                           uint64_t* it, uint64_t* pl, uint8_t* ph, uint64_t* trace,
                                                           int64_t wpp, uint32_t* trace_len) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        hrb::BitTrace tr;
        tr.words = trace + i * wpp;
        tr.cap_bits = (uint32_t)(wpp * 64 < 0xFFFFFFFFll ? wpp * 64 : 0xFFFFFFFFll);
        tr.len = 0;
        hrb::Outcome o;
        if (algo >= hrb::ALGO_REGULAR) {
            const bool unr = algo == hrb::ALGO_REGULAR_UNROLLED;
            o = hrb::regular_search<W, hrb::BitTrace>(a[i], b[i], eps[i], count[i], &tr, unr);
            if (unr) o.it = (o.it + 1) >> 1;
        } else {
            o = hrb::lefevre_search<W, hrb::BitTrace>(a[i], b[i], eps[i], count[i], mode, &tr,
                                                      algo == hrb::ALGO_LEFEVRE_SWAP);
        }
        ok[i] = o.ok;
        d[i] = o.d;
        if (it) it[i] = o.it;
        pl[i] = o.pts_lo;
        ph[i] = (uint8_t)o.pts_hi;
        trace_len[i] = tr.len;
    }
}

// ---------------------------------------------------------------------------
// workspace (per device, grows; guarded by a mutex)
// ---------------------------------------------------------------------------
// bumped on every device (re)allocation: a captured graph is only replayed
// while the workspace pointers it baked in are still the live ones
std::atomic<uint64_t> g_alloc_gen{0};

struct Buf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n) return HRB_OK;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t want = bytes + bytes / 4 + 256;
        CK(cudaMalloc(&p, want));
        n = want;
        g_alloc_gen++;
        return HRB_OK;
    }
};

struct Workspace {
    Buf tiles, tile_base, meta, bm1, bm2, blocks, counts3, offs3, app, appc, cub_tmp, tile_t, fail_t, sub_t;
};

std::mutex g_ws_mu;
Workspace g_ws[64];

int current_ws(Workspace** out) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    *out = &g_ws[dev & 63];
    return HRB_OK;
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!cached[dev & 63]) {
        int v = 148;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev & 63] = v;
    }
    return cached[dev & 63];
}

int check_slice(const hrb_slice* s) {
    if (!s) return set_err(HRB_ERR_CONFIG, "null slice");
    if (s->n_super < 1) return set_err(HRB_ERR_CONFIG, "slice has no super-domains");
    if (s->word_bits != 32 && s->word_bits != 64) return set_err(HRB_ERR_CONFIG, "word_bits must be 32 or 64");
    if (s->frac_bits < s->word_bits || s->frac_bits > 128)
        return set_err(HRB_ERR_CONFIG, "frac_bits must satisfy word_bits <= F <= 128");
    if (s->delta < 1 || s->delta > 2) return set_err(HRB_ERR_CONFIG, "delta must be 1 or 2");
    if (s->coef_limbs < 1 || s->coef_limbs > 16) return set_err(HRB_ERR_CONFIG, "coef_limbs outside [1, 16]");
    return HRB_OK;
}

int ws_prep(Workspace& ws, const SliceDev& sd, int split, cudaStream_t st) {
    const int64_t S = sd.S;
    int rc;
    if ((rc = ws.tiles.ensure(sizeof(uint64_t) * (S + 1)))) return rc;
    if ((rc = ws.tile_base.ensure(sizeof(uint64_t) * (S + 1)))) return rc;
    // meta: [0] J, [1] max subdomain step, [2] phase-3 chunk, [4] phase-1 tile counter,
    // [5] phase-2 chunk counter
    if ((rc = ws.meta.ensure(sizeof(unsigned long long) * 8))) return rc;
    CK(cudaMemsetAsync(ws.meta.p, 0, sizeof(unsigned long long) * 8, st));
    prep_kernel<<<(unsigned)((S + 1 + 255) / 256), 256, 0, st>>>(sd, split, (uint64_t*)ws.tiles.p,
                                                                 (unsigned long long*)ws.meta.p);
    CK(cudaGetLastError());
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (uint64_t*)ws.tiles.p, (uint64_t*)ws.tile_base.p, S + 1, st);
    if ((rc = ws.cub_tmp.ensure(tmp_bytes))) return rc;
    CK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.p, tmp_bytes, (uint64_t*)ws.tiles.p, (uint64_t*)ws.tile_base.p,
                                     S + 1, st));
    return HRB_OK;
}

template <class Fn>
int run_compact(Workspace& ws, const Fn& fn, uint64_t* total, cudaStream_t st) {
    int rc;
    if ((rc = ws.blocks.ensure(sizeof(uint64_t) * SCAN_BLOCKS))) return rc;
    scan_reduce_kernel<Fn><<<SCAN_BLOCKS, SCAN_THREADS, 0, st>>>(fn, (uint64_t*)ws.blocks.p);
    scan_blocks_kernel<<<1, 1024, 0, st>>>((uint64_t*)ws.blocks.p, SCAN_BLOCKS, total);
    if constexpr (std::is_same<Fn, P1Compact>::value || std::is_same<Fn, P2Compact>::value)
        scan_scatter_staged_kernel<Fn><<<SCAN_BLOCKS, SCAN_THREADS, 0, st>>>(fn, (const uint64_t*)ws.blocks.p);
    else
        scan_scatter_kernel<Fn><<<SCAN_BLOCKS, SCAN_THREADS, 0, st>>>(fn, (const uint64_t*)ws.blocks.p);
    CK(cudaGetLastError());
    return HRB_OK;
}

// Streamed upload (hrb_run_slice_host): `ready` / `chunk` let the regular
// phase-1 kernel start before the coefficients have all landed; ev_data is
// recorded on the copy stream once every input is resident, and is waited
// on before anything else reads them.
struct Stream {
    const uint32_t* ready = nullptr;
    uint32_t chunk = 1;
    cudaEvent_t ev_data = nullptr;
};

int phase1_impl(Workspace& ws, const hrb_slice* s, const SliceDev& sd0, int algo, int mode, uint64_t* fail_ids,
                uint64_t* fail_count, uint64_t cap, uint64_t* iter_sum, cudaStream_t st, const Stream& up = Stream()) {
    SliceDev sd = sd0;
    int rc;
    // upper bound of tiles: n_total/TILE + S
    const uint64_t max_tiles = (uint64_t)s->n_total / TILE + (uint64_t)s->n_super + 1;
    if ((rc = ws.bm1.ensure(sizeof(uint32_t) * max_tiles * NU))) return rc;
    if ((rc = ws.tile_t.ensure(sizeof(uint32_t) * max_tiles))) return rc;
    if ((rc = ws.fail_t.ensure(sizeof(uint32_t) * (cap + 1)))) return rc;
    const int grid = sm_count() * 8;
    auto tb = (const uint64_t*)ws.tile_base.p;
    auto bm = (uint32_t*)ws.bm1.p;
    auto tt = (uint32_t*)ws.tile_t.p;
    auto is = (unsigned long long*)iter_sum;
    auto tc = (unsigned long long*)ws.meta.p + 4;
    if (up.ev_data && (algo < hrb::ALGO_REGULAR || !up.ready)) CK(cudaStreamWaitEvent(st, up.ev_data, 0));
    if (algo >= hrb::ALGO_REGULAR && up.ready) {
        sd.ready = up.ready;
        sd.ready_chunk = up.chunk;
    }
    if (algo >= hrb::ALGO_REGULAR) {
        const int g5 = sm_count() * HRB_P1_MINB;  // persistent: one wave at the launch bound
        // quarter tiles when there are fewer than ~8 tiles per resident warp
        // (the last round of 512-domain tiles would idle most of the GPU);
        // the bitmap layout does not change
        const bool quarter = (uint64_t)s->n_total / TILE + 1 < (uint64_t)g5 * 4 * 8;
#define P1(WV, SHV, PLV) phase1_reg_kernel<WV, SHV, PLV><<<g5, 128, 0, st>>>(sd, algo, tb, bm, tt, is, tc)
        if (sd.W == 64 && sd.F == 96) {
            if (quarter) P1(64, 32, 2); else P1(64, 32, 0);
        } else if (sd.W == 64) {
            if (quarter) P1(64, -1, 2); else P1(64, -1, 0);
        } else {
            if (quarter) P1(32, -1, 2); else P1(32, -1, 0);
        }
#undef P1
    } else {  // the classic family: lockstep pairs with refill (classic_lockstep.cuh)
        const int g5 = sm_count() * HRB_P1_MINB;
        const bool quarter = (uint64_t)s->n_total / TILE + 1 < (uint64_t)g5 * 4 * 8;
#define P1C(WV, SHV, PLV)                                                                                  \
    do {                                                                                                   \
        if (mode == 0)                                                                                     \
            phase1_reg_kernel<WV, SHV, PLV, 1><<<g5, 128, 0, st>>>(sd, algo, tb, bm, tt, is, tc);        \
        else if (mode == 1)                                                                                \
            phase1_reg_kernel<WV, SHV, PLV, 2><<<g5, 128, 0, st>>>(sd, algo, tb, bm, tt, is, tc);        \
        else                                                                                               \
            phase1_reg_kernel<WV, SHV, PLV, 3><<<g5, 128, 0, st>>>(sd, algo, tb, bm, tt, is, tc);        \
    } while (0)
        if (sd.W == 64 && sd.F == 96) {
            if (quarter) P1C(64, 32, 2); else P1C(64, 32, 0);
        } else if (sd.W == 64) {
            if (quarter) P1C(64, -1, 2); else P1C(64, -1, 0);
        } else {
            if (quarter) P1C(32, -1, 2); else P1C(32, -1, 0);
        }
#undef P1C
        (void)grid;
    }
    CK(cudaGetLastError());
    if (up.ev_data && algo >= hrb::ALGO_REGULAR && up.ready) CK(cudaStreamWaitEvent(st, up.ev_data, 0));
    P1Compact fn{(const uint32_t*)ws.bm1.p, tb, tt, s->dom_base, sd.S, fail_ids, (uint32_t*)ws.fail_t.p, cap};
    return run_compact(ws, fn, fail_count, st);
}

// fail_t == nullptr: locate the super-domains of caller-provided ids first
int phase2_impl(Workspace& ws, const hrb_slice* s, const SliceDev& sd, int algo, int mode, int split,
                const uint64_t* fail_ids, const uint32_t* fail_t, const uint64_t* fail_count, uint64_t fail_cap,
                uint64_t* sub_keys, uint64_t* sub_count, uint64_t cap, cudaStream_t st) {
    int rc;
    const uint64_t Jmax = 2 * (uint64_t)split;
    if ((rc = ws.bm2.ensure(sizeof(uint32_t) * (fail_cap + 1) * ((Jmax + 31) / 32)))) return rc;
    if ((rc = ws.sub_t.ensure(sizeof(uint32_t) * (cap + 1)))) return rc;
    if (!fail_t) {
        if ((rc = ws.fail_t.ensure(sizeof(uint32_t) * (fail_cap + 1)))) return rc;
        locate_kernel<<<sm_count() * 4, 256, 0, st>>>(s->dom_base, sd.S, fail_ids, fail_count, fail_cap, 0,
                                                      (uint32_t*)ws.fail_t.p);
        fail_t = (const uint32_t*)ws.fail_t.p;
    }
    const int grid = sm_count() * 8;
    auto mt = (unsigned long long*)ws.meta.p;
    auto bm = (uint32_t*)ws.bm2.p;
    if (algo >= hrb::ALGO_REGULAR) {
        const int g4 = sm_count() * HRB_P2_MINB;  // persistent: one wave, chunks from the counter
        if (sd.W == 64 && sd.F == 96)
            phase2_reg_kernel<64, 32><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm);
        else if (sd.W == 64)
            phase2_reg_kernel<64, -1><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm);
        else
            phase2_reg_kernel<32, -1><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm);
    } else {  // the classic family in lockstep form
        const int g4 = sm_count() * HRB_P2_MINB;
#define P2C(WV, SHV)                                                                                         \
    do {                                                                                                     \
        if (mode == 0)                                                                                       \
            phase2_reg_kernel<WV, SHV, 1><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm); \
        else if (mode == 1)                                                                                  \
            phase2_reg_kernel<WV, SHV, 2><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm); \
        else                                                                                                 \
            phase2_reg_kernel<WV, SHV, 3><<<g4, 128, 0, st>>>(sd, split, fail_ids, fail_t, fail_count, fail_cap, mt, bm); \
    } while (0)
        if (sd.W == 64 && sd.F == 96)
            P2C(64, 32);
        else if (sd.W == 64)
            P2C(64, -1);
        else
            P2C(32, -1);
#undef P2C
        (void)grid;
    }
    CK(cudaGetLastError());
    P2Compact fn{(const uint32_t*)ws.bm2.p, fail_ids, fail_t, fail_count, fail_cap, mt, sub_keys,
                 (uint32_t*)ws.sub_t.p, cap};
    return run_compact(ws, fn, sub_count, st);
}

int phase3_impl(Workspace& ws, const hrb_slice* s, const SliceDev& sd, int split, const uint64_t* sub_keys,
                const uint32_t* sub_t, const uint64_t* sub_count, uint64_t sub_cap, uint64_t* cm, uint64_t* cd,
                uint64_t* cdom, uint64_t* cand_count, uint64_t cap, cudaStream_t st) {
    int rc;
    const uint64_t maxstep = s->max_dom_n;  // >= every subdomain step
    // items <= max(2 min_items, sub_cap * chunks of the largest size) by the
    // chunk rule of chunk3_kernel
    const uint64_t min_items = (uint64_t)sm_count() * 2048;
    const uint64_t CH = (maxstep + CHUNK3_MAX - 1) / CHUNK3_MAX;
    const uint64_t ch_min = (maxstep + CHUNK3_MIN - 1) / CHUNK3_MIN;
    uint64_t items = sub_cap * (CH ? CH : 1);
    items = items > 2 * min_items + sub_cap ? items : 2 * min_items + sub_cap;
    if (items > sub_cap * ch_min) items = sub_cap * ch_min;
    if ((rc = ws.counts3.ensure(sizeof(uint32_t) * (items + 1)))) return rc;
    if ((rc = ws.offs3.ensure(sizeof(uint64_t) * (items + 1)))) return rc;
    const uint64_t app_cap = cap;
    if ((rc = ws.app.ensure(sizeof(Cand) * (app_cap + 1)))) return rc;
    if ((rc = ws.appc.ensure(sizeof(unsigned long long)))) return rc;
    if (!sub_t) {
        if ((rc = ws.sub_t.ensure(sizeof(uint32_t) * (sub_cap + 1)))) return rc;
        locate_kernel<<<sm_count() * 4, 256, 0, st>>>(s->dom_base, sd.S, sub_keys, sub_count, sub_cap, 8,
                                                      (uint32_t*)ws.sub_t.p);
        sub_t = (const uint32_t*)ws.sub_t.p;
    }
    CK(cudaMemsetAsync(ws.appc.p, 0, sizeof(unsigned long long), st));
    chunk3_kernel<<<1, 1, 0, st>>>((unsigned long long*)ws.meta.p, sub_count, sub_cap, min_items);
    const int grid = sm_count() * 8;
    if (sd.F <= 96)
        phase3_kernel<true><<<grid, 256, 0, st>>>(sd, split, sub_keys, sub_t, sub_count, sub_cap,
                                                  (const unsigned long long*)ws.meta.p, (uint32_t*)ws.counts3.p,
                                                  (Cand*)ws.app.p, (unsigned long long*)ws.appc.p, app_cap);
    else
        phase3_kernel<false><<<grid, 256, 0, st>>>(sd, split, sub_keys, sub_t, sub_count, sub_cap,
                                                   (const unsigned long long*)ws.meta.p, (uint32_t*)ws.counts3.p,
                                                   (Cand*)ws.app.p, (unsigned long long*)ws.appc.p, app_cap);
    CK(cudaGetLastError());
    P3Offsets fn{(const uint32_t*)ws.counts3.p, sub_count, sub_cap, (const unsigned long long*)ws.meta.p,
                 (uint64_t*)ws.offs3.p};
    if ((rc = run_compact(ws, fn, cand_count, st))) return rc;
    scatter3_kernel<<<sm_count() * 2, 256, 0, st>>>((const Cand*)ws.app.p, (const unsigned long long*)ws.appc.p,
                                                    app_cap, (const uint64_t*)ws.offs3.p, cm, cd, cdom, cap);
    CK(cudaGetLastError());
    return HRB_OK;
}

int check_algo(int algo, int mode) {
    if (algo < 0 || algo > 3) return set_err(HRB_ERR_CONFIG, "unknown algorithm code");
    if (mode < 0 || mode > 2) return set_err(HRB_ERR_CONFIG, "unknown division mode code");
    return HRB_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int hrb_version(void) { return 100; }

const char* hrb_last_error(void) { return g_err.c_str(); }

int hrb_device_info(int device, char* buf, int buflen) {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, device));
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    snprintf(buf, (size_t)buflen, "%s sm_%d%d SMs=%d clock_khz=%d", p.name, p.major, p.minor, p.multiProcessorCount,
             clk);
    return HRB_OK;
}

int hrb_search_batch(int algo, int mode, int word_bits, int64_t n, const uint64_t* a, const uint64_t* b,
                     const uint64_t* eps, const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* iterations,
                     uint64_t* points_lo, uint8_t* points_hi, void* stream) {
    int rc = check_algo(algo, mode);
    if (rc) return rc;
    if (word_bits != 32 && word_bits != 64) return set_err(HRB_ERR_CONFIG, "word_bits must be 32 or 64");
    if (n < 0) return set_err(HRB_ERR_CONFIG, "negative batch size");
    if (n == 0) return HRB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t blocks = (n + 255) / 256;
    int cap = sm_count() * 16;
    int grid = (int)(blocks < cap ? blocks : cap);
    const bool reg = algo >= hrb::ALGO_REGULAR;
#define SB(WV, RV) \
    search_batch_kernel<WV, RV><<<grid, 256, 0, st>>>(algo, mode, n, a, b, eps, count, ok, d, iterations, points_lo, points_hi)
    if (word_bits == 64 && reg) SB(64, true);
    else if (word_bits == 64) SB(64, false);
    else if (reg) SB(32, true);
    else SB(32, false);
#undef SB
    CK(cudaGetLastError());
    return HRB_OK;
}

int hrb_search_verdicts(int algo, int word_bits, int64_t n, const uint64_t* a, const uint64_t* b, const uint64_t* eps,
                        const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* iterations, void* stream) {
    if (algo != hrb::ALGO_REGULAR && algo != hrb::ALGO_REGULAR_UNROLLED)
        return set_err(HRB_ERR_CONFIG, "hrb_search_verdicts serves the regular family only");
    if (word_bits != 32 && word_bits != 64) return set_err(HRB_ERR_CONFIG, "word_bits must be 32 or 64");
    if (n < 0) return set_err(HRB_ERR_CONFIG, "negative batch size");
    if (n == 0) return HRB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t cap = (int64_t)sm_count() * HRB_P1_MINB;
    const bool small = n < cap * 4 * 32 * NU;  // fewer tiles of 32 NU than 4 per resident warp
    const int64_t tv = 32 * (small ? 2 : NU);
    const int64_t blocks = ((n + tv - 1) / tv * 32 + 127) / 128;
    const int grid = (int)(blocks < cap ? blocks : cap);
#define LAUNCH(WV, NV) search_verdict_kernel<WV, NV><<<grid, 128, 0, st>>>(algo, n, a, b, eps, count, ok, d, iterations)
    if (word_bits == 64) {
        if (small) LAUNCH(64, 2); else LAUNCH(64, NU);
    } else {
        if (small) LAUNCH(32, 2); else LAUNCH(32, NU);
    }
#undef LAUNCH
    CK(cudaGetLastError());
    return HRB_OK;
}

int hrb_search_trace(int algo, int mode, int word_bits, int64_t n, const uint64_t* a, const uint64_t* b,
                     const uint64_t* eps, const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* iterations,
                     uint64_t* points_lo, uint8_t* points_hi, uint64_t* trace_words, int64_t words_per_problem,
                     uint32_t* trace_len, void* stream) {
    int rc = check_algo(algo, mode);
    if (rc) return rc;
    if (word_bits != 32 && word_bits != 64) return set_err(HRB_ERR_CONFIG, "word_bits must be 32 or 64");
    if (n < 0 || words_per_problem < 0) return set_err(HRB_ERR_CONFIG, "negative size");
    if (n == 0) return HRB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = (n + 255) / 256;
    const int cap = sm_count() * 16;
    const int grid = (int)(blocks < cap ? blocks : cap);
    if (word_bits == 64)
        search_trace_kernel<64><<<grid, 256, 0, st>>>(algo, mode, n, a, b, eps, count, ok, d, iterations, points_lo,
                                                      points_hi, trace_words, words_per_problem, trace_len);
    else
        search_trace_kernel<32><<<grid, 256, 0, st>>>(algo, mode, n, a, b, eps, count, ok, d, iterations, points_lo,
                                                      points_hi, trace_words, words_per_problem, trace_len);
    CK(cudaGetLastError());
    return HRB_OK;
}

int hrb_domain_coefficients(const hrb_slice* s, uint32_t* out, void* stream) {
    int rc = check_slice(s);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    SliceDev sd = to_dev(s);
    if ((rc = ws_prep(*ws, sd, 2, st))) return rc;
    const int grid = sm_count() * 4;
    const uint64_t* tb = (const uint64_t*)ws->tile_base.p;
    const int64_t nt = s->n_total;
    switch (s->coef_limbs) {
#define CASE(CLV) \
    case CLV: tabdiff_full_kernel<CLV><<<grid, 128, 0, st>>>(sd, tb, nt, out); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12)
        CASE(13) CASE(14) CASE(15) CASE(16)
#undef CASE
        default: return set_err(HRB_ERR_CONFIG, "coef_limbs outside [1, 16]");
    }
    CK(cudaGetLastError());
    return HRB_OK;
}

int hrb_phase1(const hrb_slice* s, int algo, int mode, uint64_t* fail_ids, uint64_t* fail_count, uint64_t cap,
               uint64_t* iter_sum, void* stream) {
    int rc = check_slice(s);
    if (rc || (rc = check_algo(algo, mode))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    SliceDev sd = to_dev(s);
    if ((rc = ws_prep(*ws, sd, 2, st))) return rc;
    return phase1_impl(*ws, s, sd, algo, mode, fail_ids, fail_count, cap, iter_sum, st);
}

int hrb_phase2(const hrb_slice* s, int algo, int mode, int split, const uint64_t* fail_ids,
               const uint64_t* fail_count, uint64_t fail_cap, uint64_t* sub_keys, uint64_t* sub_count, uint64_t cap,
               void* stream) {
    int rc = check_slice(s);
    if (rc || (rc = check_algo(algo, mode))) return rc;
    if (split < 2 || split > 64) return set_err(HRB_ERR_CONFIG, "phase2_split outside {2..64}");
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    SliceDev sd = to_dev(s);
    if ((rc = ws_prep(*ws, sd, split, st))) return rc;
    return phase2_impl(*ws, s, sd, algo, mode, split, fail_ids, nullptr, fail_count, fail_cap, sub_keys, sub_count,
                       cap, st);
}

int hrb_phase3(const hrb_slice* s, int split, const uint64_t* sub_keys, const uint64_t* sub_count, uint64_t sub_cap,
               uint64_t* cand_index, uint64_t* cand_dist, uint64_t* cand_dom, uint64_t* cand_count, uint64_t cap,
               void* stream) {
    int rc = check_slice(s);
    if (rc) return rc;
    if (split < 1 || split > 64) return set_err(HRB_ERR_CONFIG, "split outside {1..64}");
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    SliceDev sd = to_dev(s);
    if ((rc = ws_prep(*ws, sd, split, st))) return rc;
    return phase3_impl(*ws, s, sd, split, sub_keys, nullptr, sub_count, sub_cap, cand_index, cand_dist, cand_dom,
                       cand_count,
                       cap, st);
}

}  // extern "C"

namespace {
// phases 1-3 of a slice on `st`; ev_p1 (may be null) is recorded once the
// phase-1 ids and count are final, so a caller can start copying them out
// while phases 2 and 3 run.  Caller holds g_ws_mu.
// Arguments covered by phases 2 and 3 (PhaseRow.arguments_covered,
// pipeline.py:440-451): sum of the failing domains' sizes and of the
// surviving subdomains' counts, so the host-buffer call returns the
// reference's statistics without shipping the per-domain lists.
__global__ void argsum_kernel(SliceDev s, int split, const uint64_t* fail_ids, const uint32_t* fail_t,
                              const uint64_t* fail_count, uint64_t fail_cap, const uint64_t* sub_keys,
                              const uint32_t* sub_t, const uint64_t* sub_count, uint64_t sub_cap,
                              unsigned long long* out) {
    uint64_t nf = *fail_count, ns = *sub_count;
    if (nf > fail_cap) nf = fail_cap;
    if (ns > sub_cap) ns = sub_cap;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long a2 = 0, a3 = 0;
    for (uint64_t k = g; k < nf; k += stride) {
        const int64_t t = fail_t[k];
        a2 += domain_size(s, t, fail_ids[k] - s.dom_base[t]);
    }
    for (uint64_t k = g; k < ns; k += stride) {
        const int64_t t = sub_t[k];
        const uint64_t key = sub_keys[k];
        const uint64_t n = domain_size(s, t, (key >> 8) - s.dom_base[t]);
        uint64_t step = n / (uint64_t)split;
        if (step < 1) step = 1;
        const uint64_t start = (key & 255) * step;
        a3 += step < n - start ? step : n - start;
    }
    for (int o = 16; o; o >>= 1) {
        a2 += __shfl_down_sync(0xffffffffu, a2, o);
        a3 += __shfl_down_sync(0xffffffffu, a3, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a2) atomicAdd(&out[0], a2);
        if (a3) atomicAdd(&out[1], a3);
    }
}

int run_slice_locked(Workspace& ws, const hrb_slice* s, int algo, int mode, int split, const hrb_run_out* out,
                     cudaStream_t st, cudaEvent_t ev_p1, const Stream& up = Stream(), uint64_t* argsums = nullptr) {
    int rc;
    SliceDev sd = to_dev(s);
    uint64_t* counts = out->counts;
    CK(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * 4, st));
    if ((rc = ws_prep(ws, sd, split, st))) return rc;
    if ((rc = phase1_impl(ws, s, sd, algo, mode, out->fail_ids, counts + 0, out->fail_cap, counts + 3, st, up)))
        return rc;
    if (ev_p1) CK(cudaEventRecord(ev_p1, st));
    if ((rc = phase2_impl(ws, s, sd, algo, mode, split, out->fail_ids, (const uint32_t*)ws.fail_t.p, counts + 0,
                          out->fail_cap, out->sub_keys, counts + 1, out->sub_cap, st)))
        return rc;
    if ((rc = phase3_impl(ws, s, sd, split, out->sub_keys, (const uint32_t*)ws.sub_t.p, counts + 1, out->sub_cap,
                          out->cand_index, out->cand_dist, out->cand_dom, counts + 2, out->cand_cap, st)))
        return rc;
    if (argsums) {
        CK(cudaMemsetAsync(argsums, 0, sizeof(uint64_t) * 2, st));
        argsum_kernel<<<sm_count() * 4, 256, 0, st>>>(sd, split, out->fail_ids, (const uint32_t*)ws.fail_t.p,
                                                      counts + 0, out->fail_cap, out->sub_keys,
                                                      (const uint32_t*)ws.sub_t.p, counts + 1, out->sub_cap,
                                                      (unsigned long long*)argsums);
        CK(cudaGetLastError());
    }
    return HRB_OK;
}

// hrb_run_slice replays its 17 launches as one CUDA graph when called again
// with identical arguments (the bench and every re-run of a resident slice):
// the first call runs eagerly -- sizing the workspace -- and captures the same
// sequence on a private stream; later identical calls launch the graph on the
// caller's stream.  HRB_NO_GRAPH=1 disables it.
struct GraphCache {
    bool valid = false;
    std::vector<uint64_t> key;
    uint64_t gen = 0;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t cap = nullptr;
};
GraphCache g_graph[64];

std::vector<uint64_t> run_key(const hrb_slice* s, int algo, int mode, int split, const hrb_run_out* o) {
    return {(uint64_t)s->n_super, (uint64_t)s->n_total, s->max_dom_n, (uint64_t)s->coef_limbs, (uint64_t)s->frac_bits,
            (uint64_t)s->word_bits, (uint64_t)s->delta, (uint64_t)s->coef, (uint64_t)s->G, (uint64_t)s->s2abs,
            (uint64_t)s->n_dom, (uint64_t)s->dom_n, (uint64_t)s->last_n, (uint64_t)s->dom_base, (uint64_t)s->m0,
            (uint64_t)algo, (uint64_t)mode, (uint64_t)split, (uint64_t)o->fail_ids, o->fail_cap, (uint64_t)o->sub_keys,
            o->sub_cap, (uint64_t)o->cand_index, (uint64_t)o->cand_dist, (uint64_t)o->cand_dom, o->cand_cap,
            (uint64_t)o->counts};
}

int capture_run(GraphCache& G, Workspace& ws, const hrb_slice* s, int algo, int mode, int split, const hrb_run_out* out,
                std::vector<uint64_t>&& key) {
    if (!G.cap) CK(cudaStreamCreateWithFlags(&G.cap, cudaStreamNonBlocking));
    const uint64_t gen0 = g_alloc_gen.load();
    CK(cudaStreamBeginCapture(G.cap, cudaStreamCaptureModeThreadLocal));
    int rc = run_slice_locked(ws, s, algo, mode, split, out, G.cap, nullptr);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(G.cap, &graph);
    G.valid = false;
    if (rc || ec != cudaSuccess || !graph || g_alloc_gen.load() != gen0) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();  // a failed capture is not an error of the run itself
        return HRB_OK;
    }
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G.exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        G.exec = nullptr;
        cudaGetLastError();
        return HRB_OK;
    }
    G.key = std::move(key);
    G.gen = gen0;
    G.valid = true;
    return HRB_OK;
}

#include "wide.cuh"
}  // namespace

extern "C" {

int hrb_run_slice(const hrb_slice* s, int algo, int mode, int split, const hrb_run_out* out, void* stream) {
    int rc = check_slice(s);
    if (rc || (rc = check_algo(algo, mode))) return rc;
    if (split < 2 || split > 64) return set_err(HRB_ERR_CONFIG, "phase2_split outside {2..64}");
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    GraphCache& G = g_graph[dev & 63];
    const bool use_graph = std::getenv("HRB_NO_GRAPH") == nullptr;
    std::vector<uint64_t> key = run_key(s, algo, mode, split, out);
    if (use_graph && G.valid && G.gen == g_alloc_gen.load() && G.key == key) {
        CK(cudaGraphLaunch(G.exec, (cudaStream_t)stream));
        return HRB_OK;
    }
    if ((rc = run_slice_locked(*ws, s, algo, mode, split, out, (cudaStream_t)stream, nullptr))) return rc;
    return use_graph ? capture_run(G, *ws, s, algo, mode, split, out, std::move(key)) : HRB_OK;
}

namespace {
#ifndef HRB_UPLOAD_CHUNKS
#define HRB_UPLOAD_CHUNKS 8
#endif
constexpr int UPLOAD_CHUNKS = HRB_UPLOAD_CHUNKS;  // streamed upload: runs of super-domains

struct HostRunState {
    Buf coef, G, s2, nd, dn, ln, db, m0, fail, sub, cm, cd, cdom, counts, ready;
    cudaStream_t st = nullptr, cs = nullptr;  // compute stream, copy stream (uploads, id copy-out)
    cudaEvent_t e0 = nullptr, e1 = nullptr, ep1 = nullptr, emeta = nullptr, edata = nullptr;
    uint64_t* hcount = nullptr;  // pinned scratch for the phase-1 count
    uint32_t* hseq = nullptr;    // pinned 1 .. UPLOAD_CHUNKS: the chunk counter's values
    uint32_t* hflag = nullptr;   // pinned: wait_super timeout flag read back after a streamed call
};
HostRunState g_host[64];
std::mutex g_host_mu[64];  // one host-buffer call at a time per device (shared buffers, streams)
}  // namespace

}  // extern "C"

namespace {
// hrb_run_slice_host and hrb_run_slice_resident: with `resident` the slice's
// columns are already device pointers (written on stream `after`, e.g. by
// hrb_pack_blocks) and nothing is uploaded.
int run_host_impl(const hrb_slice* hs, bool resident, cudaStream_t after, int algo, int mode, int split,
                  uint64_t* counts, uint64_t* fail_ids, uint64_t fail_cap, uint64_t* cand_index,
                  uint64_t* cand_dist, uint64_t* cand_dom, uint64_t cand_cap, float* device_ms) {
    int rc = check_slice(hs);
    if (rc || (rc = check_algo(algo, mode))) return rc;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> host_lk(g_host_mu[dev & 63]);
    HostRunState& H = g_host[dev & 63];
    if (!H.st) {
        CK(cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&H.cs, cudaStreamNonBlocking));
        CK(cudaEventCreate(&H.e0));
        CK(cudaEventCreate(&H.e1));
        CK(cudaEventCreateWithFlags(&H.ep1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&H.emeta, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&H.edata, cudaEventDisableTiming));
        CK(cudaMallocHost((void**)&H.hcount, sizeof(uint64_t)));
        CK(cudaMallocHost((void**)&H.hseq, sizeof(uint32_t) * UPLOAD_CHUNKS));
        CK(cudaMallocHost((void**)&H.hflag, sizeof(uint32_t)));
        for (int c = 0; c < UPLOAD_CHUNKS; c++) H.hseq[c] = (uint32_t)(c + 1);
    }
    const int64_t S = hs->n_super, CL = hs->coef_limbs, NT = hs->n_total;
    // the phases read coefficients only mod 2^128: with >= 4 two's-complement
    // limbs, only the low four of each coefficient are uploaded
    const int64_t CLd = CL >= 4 ? 4 : CL;
    const size_t b_coef = sizeof(uint32_t) * 6 * CLd * S, b2 = sizeof(uint64_t) * 2 * S, b32 = sizeof(uint32_t) * S;
    if (!resident &&
        ((rc = H.coef.ensure(b_coef)) || (rc = H.G.ensure(b2)) || (rc = H.s2.ensure(b2)) || (rc = H.nd.ensure(b32)) ||
         (rc = H.dn.ensure(b32)) || (rc = H.ln.ensure(b32)) || (rc = H.db.ensure(sizeof(uint64_t) * (S + 1))) ||
         (rc = H.m0.ensure(sizeof(uint64_t) * S))))
        return rc;
    if ((rc = H.counts.ensure(sizeof(uint64_t) * 6)) || (rc = H.ready.ensure(2 * sizeof(uint32_t)))) return rc;
    cudaStream_t st = H.st, cs = H.cs;
    // Upload on the copy stream.  The per-super-domain sizes and offsets go
    // first (prep and phase 1's tile walk need them before the launch).  For
    // the regular family the rest is streamed: coefficients, G, s2abs and m0
    // in runs of super-domains, each followed by a 4-byte write of its
    // sequence number to a chunk counter that phase 1's warps wait on
    // (wait_super), so the upload overlaps the search; phase 1 reads every
    // super-domain, so whatever follows it finds the slice resident.  Every
    // copy is enqueued before the search: a workspace allocation inside the
    // run (cudaFree synchronises the device) must never wait on a kernel that
    // waits on a copy not yet issued.  The classic family (no wait in its
    // kernel) uploads everything before the search starts.
    const bool stream_in = !resident && algo >= hrb::ALGO_REGULAR;
    if (resident) {
        CK(cudaEventRecord(H.edata, after));
        CK(cudaStreamWaitEvent(st, H.edata, 0));
    }
    CK(cudaEventRecord(H.e0, st));
    CK(cudaStreamWaitEvent(cs, H.e0, 0));  // nothing of the previous call still reads the buffers
    CK(cudaMemsetAsync(H.ready.p, 0, 2 * sizeof(uint32_t), cs));  // chunk counter, timeout flag
    if (!resident) {
        CK(cudaMemcpyAsync(H.nd.p, hs->n_dom, b32, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(H.dn.p, hs->dom_n, b32, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(H.ln.p, hs->last_n, b32, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(H.db.p, hs->dom_base, sizeof(uint64_t) * (S + 1), cudaMemcpyHostToDevice, cs));
    }
    const int64_t nchunk = !stream_in ? 1 : (S < UPLOAD_CHUNKS ? S : UPLOAD_CHUNKS);
    const int64_t per = (S + nchunk - 1) / nchunk;
    auto upload_chunk = [&](int64_t c) -> int {
        const int64_t t0 = c * per, n = (t0 + per <= S ? per : S - t0);
        cudaMemcpy3DParms p = {};
        // 6 coefficients x CLd limb rows of n words; host rows have pitch S
        // words and CL rows per coefficient, device rows CLd
        p.srcPtr = make_cudaPitchedPtr((void*)(hs->coef + t0), sizeof(uint32_t) * S, sizeof(uint32_t) * n, CL);
        p.dstPtr = make_cudaPitchedPtr((uint32_t*)H.coef.p + t0, sizeof(uint32_t) * S, sizeof(uint32_t) * n, CLd);
        p.extent = make_cudaExtent(sizeof(uint32_t) * n, CLd, 6);
        p.kind = cudaMemcpyHostToDevice;
        CK(cudaMemcpy3DAsync(&p, cs));
        CK(cudaMemcpy2DAsync((uint64_t*)H.G.p + t0, sizeof(uint64_t) * S, hs->G + t0, sizeof(uint64_t) * S,
                             sizeof(uint64_t) * n, 2, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpy2DAsync((uint64_t*)H.s2.p + t0, sizeof(uint64_t) * S, hs->s2abs + t0, sizeof(uint64_t) * S,
                             sizeof(uint64_t) * n, 2, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync((uint64_t*)H.m0.p + t0, hs->m0 + t0, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, cs));
        if (stream_in)
            CK(cudaMemcpyAsync(H.ready.p, H.hseq + c, sizeof(uint32_t), cudaMemcpyHostToDevice, cs));
        return HRB_OK;
    };
    if (resident) {
        // the columns are on the device already
    } else if (!stream_in) {
        if ((rc = upload_chunk(0))) return rc;
        CK(cudaEventRecord(H.edata, cs));
        CK(cudaStreamWaitEvent(st, H.edata, 0));
    } else {
        CK(cudaEventRecord(H.emeta, cs));
        for (int64_t c = 0; c * per < S; c++)
            if ((rc = upload_chunk(c))) return rc;
        CK(cudaStreamWaitEvent(st, H.emeta, 0));
    }
    Stream up;
    if (stream_in) {
        up.ready = (const uint32_t*)H.ready.p;
        up.chunk = (uint32_t)per;
    }
    hrb_slice ds = *hs;
    if (!resident) {
        ds.coef = (const uint32_t*)H.coef.p;
        ds.coef_limbs = (int32_t)CLd;
        ds.G = (const uint64_t*)H.G.p;
        ds.s2abs = (const uint64_t*)H.s2.p;
        ds.n_dom = (const uint32_t*)H.nd.p;
        ds.dom_n = (const uint32_t*)H.dn.p;
        ds.last_n = (const uint32_t*)H.ln.p;
        ds.dom_base = (const uint64_t*)H.db.p;
        ds.m0 = (const uint64_t*)H.m0.p;
    }
    uint64_t sub_cap = (uint64_t)NT / 8 + 1024;  // grown once from the true count
    const uint64_t fcap = (uint64_t)NT;
    bool fail_copied = false;
    for (int attempt = 0; attempt < 2; attempt++) {
        if ((rc = H.fail.ensure(sizeof(uint64_t) * (fcap + 1))) || (rc = H.sub.ensure(sizeof(uint64_t) * (sub_cap + 1))) ||
            (rc = H.cm.ensure(sizeof(uint64_t) * (cand_cap + 1))) ||
            (rc = H.cd.ensure(sizeof(uint64_t) * (cand_cap + 1))) ||
            (rc = H.cdom.ensure(sizeof(uint64_t) * (cand_cap + 1))))
            return rc;
        hrb_run_out o;
        o.fail_ids = (uint64_t*)H.fail.p;
        o.fail_cap = fcap;
        o.sub_keys = (uint64_t*)H.sub.p;
        o.sub_cap = sub_cap;
        o.cand_index = (uint64_t*)H.cm.p;
        o.cand_dist = (uint64_t*)H.cd.p;
        o.cand_dom = (uint64_t*)H.cdom.p;
        o.cand_cap = cand_cap;
        o.counts = (uint64_t*)H.counts.p;
        {
            std::lock_guard<std::mutex> lk(g_ws_mu);
            Workspace* ws;
            if ((rc = current_ws(&ws))) return rc;
            if ((rc = check_slice(&ds)) || (rc = check_algo(algo, mode))) return rc;
            if (split < 2 || split > 64) return set_err(HRB_ERR_CONFIG, "phase2_split outside {2..64}");
            if ((rc = run_slice_locked(*ws, &ds, algo, mode, split, &o, st, fail_copied ? nullptr : H.ep1,
                                       attempt == 0 ? up : Stream(), (uint64_t*)H.counts.p + 4)))
                return rc;
        }
        if (!fail_copied) {
            // the failing ids are final after phase 1: copy them out on the
            // copy stream while phases 2 and 3 run on the compute stream
            CK(cudaStreamWaitEvent(H.cs, H.ep1, 0));
            CK(cudaMemcpyAsync(H.hcount, H.counts.p, sizeof(uint64_t), cudaMemcpyDeviceToHost, H.cs));
            CK(cudaStreamSynchronize(H.cs));
            const uint64_t nf0 = *H.hcount < fail_cap ? *H.hcount : fail_cap;
            if (fail_ids && nf0)
                CK(cudaMemcpyAsync(fail_ids, H.fail.p, sizeof(uint64_t) * nf0, cudaMemcpyDeviceToHost, H.cs));
            fail_copied = true;
        }
        CK(cudaMemcpyAsync(counts, H.counts.p, sizeof(uint64_t) * 6, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (counts[1] <= sub_cap) break;
        sub_cap = counts[1] + 1024;  // grow once and re-run
        CK(cudaStreamSynchronize(H.cs));  // the copy-out of the ids is done before phase 1 rewrites them
        CK(cudaEventRecord(H.e0, st));
    }
    const uint64_t nc = counts[2] < cand_cap ? counts[2] : cand_cap;
    if (nc) {
        CK(cudaMemcpyAsync(cand_index, H.cm.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(cand_dist, H.cd.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(cand_dom, H.cdom.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(H.cs));
    CK(cudaEventRecord(H.e1, st));
    if (stream_in) CK(cudaMemcpyAsync(H.hflag, (uint32_t*)H.ready.p + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (device_ms) CK(cudaEventElapsedTime(device_ms, H.e0, H.e1));
    if (stream_in && *H.hflag) return set_err(HRB_ERR_RUNTIME, "streamed upload never arrived (wait_super timed out)");
    if (counts[0] > fail_cap && fail_ids) return set_err(HRB_ERR_CAPACITY, "fail_ids buffer too small");
    if (counts[2] > cand_cap) return set_err(HRB_ERR_CAPACITY, "candidate buffer too small");
    return HRB_OK;
}
}  // namespace

extern "C" {

int hrb_run_slice_host(const hrb_slice* hs, int algo, int mode, int split, uint64_t* counts, uint64_t* fail_ids,
                       uint64_t fail_cap, uint64_t* cand_index, uint64_t* cand_dist, uint64_t* cand_dom,
                       uint64_t cand_cap, float* device_ms) {
    return run_host_impl(hs, false, nullptr, algo, mode, split, counts, fail_ids, fail_cap, cand_index, cand_dist,
                         cand_dom, cand_cap, device_ms);
}

int hrb_run_slice_resident(const hrb_slice* s, int algo, int mode, int split, uint64_t* counts,
                           uint64_t* cand_index, uint64_t* cand_dist, uint64_t* cand_dom, uint64_t cand_cap,
                           float* device_ms, void* stream) {
    return run_host_impl(s, true, (cudaStream_t)stream, algo, mode, split, counts, nullptr, 0, cand_index, cand_dist,
                         cand_dom, cand_cap, device_ms);
}

}  // extern "C"

// ===========================================================================
// high-degree (delta_R >= 3) slices: include/hrb200.h hrb_wslice, csrc/wide.cuh
// ===========================================================================
extern "C" {

int hrb_wrun_slice(const hrb_wslice* s, int algo, int split, const hrb_run_out* out, void* stream) {
    int rc = check_wslice(s);
    if (rc) return rc;
    if (algo != hrb::ALGO_REGULAR && algo != hrb::ALGO_REGULAR_UNROLLED)
        return set_err(HRB_ERR_CONFIG, "wide slices run the regular search family");
    if (split < 2 || split > 16) return set_err(HRB_ERR_CONFIG, "wide slices need phase2_split in {2..16}");
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    return run_wslice_locked(*ws, g_wws[dev & 63], s, algo, split, out, (cudaStream_t)stream, nullptr);
}

int hrb_wdomain_coefficients(const hrb_wslice* s, uint32_t* out, void* stream) {
    int rc = check_wslice(s);
    if (rc) return rc;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace* ws;
    if ((rc = current_ws(&ws))) return rc;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    return wtabdiff_impl(*ws, g_wws[dev & 63], s, out, (cudaStream_t)stream);
}

int hrb_wrun_slice_host(const hrb_wslice* hs, int algo, int split, uint64_t* counts, uint64_t* cand_index,
                        uint64_t* cand_dist, uint64_t* cand_dom, uint64_t cand_cap, float* device_ms) {
    int rc = check_wslice(hs);
    if (rc) return rc;
    if (algo != hrb::ALGO_REGULAR && algo != hrb::ALGO_REGULAR_UNROLLED)
        return set_err(HRB_ERR_CONFIG, "wide slices run the regular search family");
    if (split < 2 || split > 16) return set_err(HRB_ERR_CONFIG, "wide slices need phase2_split in {2..16}");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> hl(g_host_mu[dev & 63]);
    HostRunState& H = g_host[dev & 63];
    if (!H.st) {
        CK(cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&H.cs, cudaStreamNonBlocking));
        CK(cudaEventCreate(&H.e0));
        CK(cudaEventCreate(&H.e1));
        CK(cudaEventCreateWithFlags(&H.ep1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&H.emeta, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&H.edata, cudaEventDisableTiming));
        CK(cudaMallocHost((void**)&H.hcount, sizeof(uint64_t)));
        CK(cudaMallocHost((void**)&H.hseq, sizeof(uint32_t) * UPLOAD_CHUNKS));
        CK(cudaMallocHost((void**)&H.hflag, sizeof(uint32_t)));
        for (int c = 0; c < UPLOAD_CHUNKS; c++) H.hseq[c] = (uint32_t)(c + 1);
    }
    const int64_t S = hs->n_super, NT = hs->n_total;
    const int D = hs->degree, NL = hs->frac_limbs, ncoef = (D + 1) * (D + 2) / 2;
    const size_t b_coef = sizeof(uint32_t) * ncoef * NL * S, b2 = sizeof(uint64_t) * 2 * S,
                 b32 = sizeof(uint32_t) * S, b_win = sizeof(uint32_t) * NL * S;
    // the host-state buffers are reused: coef, G <- padg, s2 <- s2b, ready <- win
    if ((rc = H.coef.ensure(b_coef)) || (rc = H.G.ensure(b2)) || (rc = H.s2.ensure(b2)) || (rc = H.ready.ensure(b_win)) ||
        (rc = H.nd.ensure(b32)) || (rc = H.dn.ensure(b32)) || (rc = H.ln.ensure(b32)) ||
        (rc = H.db.ensure(sizeof(uint64_t) * (S + 1))) || (rc = H.m0.ensure(sizeof(uint64_t) * S)) ||
        (rc = H.counts.ensure(sizeof(uint64_t) * 6)))
        return rc;
    cudaStream_t st = H.st;
    CK(cudaEventRecord(H.e0, st));
    CK(cudaMemcpyAsync(H.coef.p, hs->coef, b_coef, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.G.p, hs->padg, b2, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.s2.p, hs->s2b, b2, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.ready.p, hs->win, b_win, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.nd.p, hs->n_dom, b32, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.dn.p, hs->dom_n, b32, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.ln.p, hs->last_n, b32, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.db.p, hs->dom_base, sizeof(uint64_t) * (S + 1), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(H.m0.p, hs->m0, sizeof(uint64_t) * S, cudaMemcpyHostToDevice, st));
    hrb_wslice ds = *hs;
    ds.coef = (const uint32_t*)H.coef.p;
    ds.padg = (const uint64_t*)H.G.p;
    ds.s2b = (const uint64_t*)H.s2.p;
    ds.win = (const uint32_t*)H.ready.p;
    ds.n_dom = (const uint32_t*)H.nd.p;
    ds.dom_n = (const uint32_t*)H.dn.p;
    ds.last_n = (const uint32_t*)H.ln.p;
    ds.dom_base = (const uint64_t*)H.db.p;
    ds.m0 = (const uint64_t*)H.m0.p;
    uint64_t sub_cap = (uint64_t)NT / 8 + 1024;
    const uint64_t fcap = (uint64_t)NT;
    for (int attempt = 0; attempt < 2; attempt++) {
        if ((rc = H.fail.ensure(sizeof(uint64_t) * (fcap + 1))) || (rc = H.sub.ensure(sizeof(uint64_t) * (sub_cap + 1))) ||
            (rc = H.cm.ensure(sizeof(uint64_t) * (cand_cap + 1))) ||
            (rc = H.cd.ensure(sizeof(uint64_t) * (cand_cap + 1))) ||
            (rc = H.cdom.ensure(sizeof(uint64_t) * (cand_cap + 1))))
            return rc;
        hrb_run_out o;
        o.fail_ids = (uint64_t*)H.fail.p;
        o.fail_cap = fcap;
        o.sub_keys = (uint64_t*)H.sub.p;
        o.sub_cap = sub_cap;
        o.cand_index = (uint64_t*)H.cm.p;
        o.cand_dist = (uint64_t*)H.cd.p;
        o.cand_dom = (uint64_t*)H.cdom.p;
        o.cand_cap = cand_cap;
        o.counts = (uint64_t*)H.counts.p;
        {
            std::lock_guard<std::mutex> lk(g_ws_mu);
            Workspace* ws;
            if ((rc = current_ws(&ws))) return rc;
            if ((rc = run_wslice_locked(*ws, g_wws[dev & 63], &ds, algo, split, &o, st, (uint64_t*)H.counts.p + 4)))
                return rc;
        }
        CK(cudaMemcpyAsync(counts, H.counts.p, sizeof(uint64_t) * 6, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (counts[1] <= sub_cap) break;
        sub_cap = counts[1] + 1024;
    }
    const uint64_t nc = counts[2] < cand_cap ? counts[2] : cand_cap;
    if (nc) {
        CK(cudaMemcpyAsync(cand_index, H.cm.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(cand_dist, H.cd.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(cand_dom, H.cdom.p, sizeof(uint64_t) * nc, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaEventRecord(H.e1, st));
    CK(cudaStreamSynchronize(st));
    if (device_ms) CK(cudaEventElapsedTime(device_ms, H.e0, H.e1));
    if (counts[2] > cand_cap) return set_err(HRB_ERR_CAPACITY, "candidate buffer too small");
    return HRB_OK;
}

}  // extern "C"

// ===========================================================================
// rigorous confirmation on the device: csrc/confirm.cuh
// ===========================================================================
extern "C" int hrb_confirm_exp(int precision, int eps_bits, int binade, int64_t n, const uint64_t* index,
                               uint8_t* is_hr, uint64_t* dist_raw, uint8_t* status, void* stream) {
    if (precision < 2 || precision > 64 || eps_bits < 1 || binade > 0 || binade < -1000 || n < 0)
        return set_err(HRB_ERR_CONFIG, "hrb_confirm_exp: exp on binades <= 0, 2 <= p <= 64, eps_bits >= 1");
    if (n == 0) return HRB_OK;
    static std::atomic<bool> inv_ready{false};
    if (!inv_ready.load()) {  // ceil(2^64 / d) for the fast kernel's small divisions
        uint64_t inv[128] = {0, 0};
        for (int d = 2; d < 128; d++) inv[d] = (uint64_t)(((unsigned __int128)1 << 64) / d) + 1;
        CK(cudaMemcpyToSymbol(fw::c_inv, inv, sizeof(inv)));
        inv_ready = true;
    }
    int grid = (int)((n + 127) / 128);
    if (grid > sm_count() * 16) grid = sm_count() * 16;
    // the first precision step's widest value has P + 3 bits (see confirm.cuh)
    const int prec0 = 2 * (precision + eps_bits) + 16;
    int work = prec0 > 64 ? prec0 : 64;
    if (precision - binade + 1 > work) work = precision - binade + 1;
    work += 8;
    const int wp = work + 14;
    int r = 0;
    while ((r + 1) * (r + 1) <= wp) r++;
    const int nl = (wp + r + 3 + 63) / 64;
    cudaStream_t st = (cudaStream_t)stream;
#define FAST(NLV) confirm_exp_fast_kernel<NLV><<<grid, 128, 0, st>>>(precision, eps_bits, binade, prec0, n, index, \
                                                                       is_hr, dist_raw, status)
    if (nl <= 3) FAST(3);
    else if (nl == 4) FAST(4);
    else if (nl == 5) FAST(5);
    else if (nl == 6) FAST(6);
    else confirm_exp_kernel<<<grid, 128, 0, st>>>(precision, eps_bits, binade, n, index, is_hr, dist_raw, status);
#undef FAST
    CK(cudaGetLastError());
    return HRB_OK;
}

// ---------------------------------------------------------------------------
// native generation on the device: one thread per super-domain runs
// csrc/host/polygen.h's one_block -- the SAME source as libhrbhost.so's
// hrbh_pack_blocks -- and writes the packed columns in place
// ---------------------------------------------------------------------------
#ifndef HRB_GEN_MINB
#define HRB_GEN_MINB 8
#endif
__global__ void __launch_bounds__(64, HRB_GEN_MINB) pack_blocks_kernel(hrbh_cfg c, int64_t S, const uint64_t* index_start,
                                                         const uint64_t* count, const uint32_t* n_p,
                                                         const uint32_t* tau, const int32_t* e_out, uint32_t* coef,
                                                         uint64_t* G, uint64_t* s2abs, uint8_t* status,
                                                         uint8_t* shift_ok) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S) return;
    hrbh::BlockOut o;
    if (!hrbh::one_block(c, index_start[t], count[t], n_p[t], tau[t], e_out[t], &o)) {
        status[t] = HRBH_FALLBACK;
        return;
    }
    const int cl = c.limbs + 1;
    status[t] = HRBH_OK;
    shift_ok[t] = o.shift_ok ? 1 : 0;
    for (int k = 0; k < 6; k++) hrbh::put_limbs(o.r[k], cl, coef, k, S, t);
    G[t] = o.G.n > 0 ? o.G.w[0] : 0;
    G[S + t] = o.G.n > 1 ? o.G.w[1] : 0;
    s2abs[t] = o.s2.n > 0 ? o.s2.w[0] : 0;
    s2abs[S + t] = o.s2.n > 1 ? o.s2.w[1] : 0;
}

extern "C" int hrb_pack_blocks(const hrbh_cfg* cfg, int64_t S, const uint64_t* index_start, const uint64_t* count,
                               const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out, uint32_t* coef,
                               uint64_t* G, uint64_t* s2abs, uint8_t* status, uint8_t* shift_ok, void* stream) {
    // the host library's configuration domain, with the device's fixed
    // capacity (1024-bit values, hrbh::NW): limbs <= 12 keeps every product
    // of the checks below 2^1024, frac_bits + guard <= 224 the enclosures'
    // squarings (wp <= 270)
    if (!cfg || cfg->fn != HRBH_FN_EXP || cfg->precision < 2 || cfg->precision > 64 || cfg->eps_bits < 1 ||
        cfg->binade > 0 || cfg->binade <= -1000 || cfg->frac_bits < 8 || cfg->guard < 0 || cfg->limbs < 1 ||
        cfg->limbs > 12 || cfg->frac_bits + cfg->guard > 224 || (cfg->delta != 1 && cfg->delta != 2) ||
        (cfg->word_bits != 32 && cfg->word_bits != 64) || S < 0)
        return set_err(HRB_ERR_CONFIG, "hrb_pack_blocks: exp on binades <= 0, delta <= 2, limbs <= 12, "
                                       "frac_bits + guard <= 224");
    if (S == 0) return HRB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    // The kernel keeps ~15 KB of big integers per thread in local memory;
    // the driver reserves that for every resident thread slot (~4.2 GB of
    // device memory on a B200, kept after the first launch).
    pack_blocks_kernel<<<(unsigned)((S + 63) / 64), 64, 0, st>>>(*cfg, S, index_start, count, n_p, tau, e_out, coef,
                                                                G, s2abs, status, shift_ok);
    CK(cudaGetLastError());
    return HRB_OK;
}
