// wide.cuh -- the high-degree (delta_R = D in 3..8) path: one Taylor
// polynomial per large super-domain, walked on the device with multi-limb
// add-with-carry difference tables (the paper's tabulated-difference kernel,
// words interleaved in global memory, limb count a
// template parameter).  Included by hrb200.cu inside its anonymous
// namespace: it reuses the slice geometry (SliceDev), the lockstep search
// engine (tile_search.cuh), the ordered compactions and the workspace.
//
// Arithmetic is exact mod 2^F with F = 32 NL: a residue is NL 32-bit limbs
// and its top 64 bits are simply the two top limbs.  Layout and semantics:
// include/hrb200.h hrb_wslice; specification: oracle/wide.py.
//
//   wseed    per warp tile (512 domains) and coefficient column (j, l):
//            the unit-step difference columns of r_j at the tile's first
//            domain i0: Delta^l r_j(i0) = sum_m q_{j,m} C(i0, m - l)
//   phase1   per tile: every lane seeds its packet of 16 consecutive domains
//            from the tile column (E^(16 lane), binomials < 2^53) and walks
//            it with D (r_0) and D - 1 (r_1) NL-limb additions per domain,
//            staging (a, b) in shared memory; then the lockstep search of
//            phase1_reg_kernel over the staged problems
//   phase2   per failing domain: s_j(i) from the tile column, shifted to
//            each subdomain start (binomials < 2^128), re-test
//   phase3   per (subdomain, chunk): the exact degree-D walk, D NL-limb
//            additions per argument, a one-limb conservative window test,
//            exact re-walk + ordered append on a hit

constexpr int WMAXD = 8;
constexpr int WMAXNL = 8;

// C(32, k), k <= 8 (all below 2^32)
__host__ __device__ constexpr uint32_t wbinom32(int k) {
    uint64_t b = 1;
    for (int i = 0; i < k; i++) b = b * (uint64_t)(32 - i) / (uint64_t)(i + 1);
    return (uint32_t)b;
}

// Bound on how far the 32-bit top-limb proxy of column 0 of a degree-D
// difference table falls below the true top limb within 32 steps: each
// column's proxy misses at most one carry per step and inherits the next
// column's shortfall, e_l(x + 1) = e_l(x) + e_{l+1}(x) + 1, e_D = 0.
template <int D>
__host__ __device__ constexpr uint32_t wproxy_margin() {
    uint64_t e[WMAXD + 1] = {};
    uint64_t mx = 0;
    for (int x = 0; x <= 32; x++) {
        if (e[0] > mx) mx = e[0];
        for (int l = 0; l < D; l++) e[l] = e[l] + e[l + 1] + 1;
    }
    return (uint32_t)(mx + 1);
}

struct WideDev {
    SliceDev g;  // geometry (S, n_dom, dom_n, last_n, dom_base, m0); coefficient fields unused
    int D, NL, ncoef;
    const uint32_t* coef;   // [ncoef][NL][S]
    const uint64_t* padg;   // [2][S]
    const uint64_t* s2b;    // [2][S]
    const uint32_t* win;    // [NL][S]
    const uint32_t* seeds;  // [tile][ncoef][NL] (workspace, written by wseed_kernel)
};

__host__ __device__ __forceinline__ int wcol(int D, int j, int l) { return j * (2 * D + 3 - j) / 2 + l; }

// acc += x * m mod 2^(32 NL) for an MW-word multiplier m
template <int NL, int MW>
__device__ __forceinline__ void wmad(uint32_t (&acc)[NL], const uint32_t* x, const uint32_t (&m)[MW]) {
#pragma unroll
    for (int h = 0; h < MW; h++) {
        uint32_t carry = 0;
#pragma unroll
        for (int l = 0; l + h < NL; l++) {
            const uint64_t p = (uint64_t)x[l] * m[h] + acc[l + h] + carry;
            acc[l + h] = (uint32_t)p;
            carry = (uint32_t)(p >> 32);
        }
    }
}

template <int NL>
__device__ __forceinline__ void wmad64(uint32_t (&acc)[NL], const uint32_t* x, uint64_t m) {
    const uint32_t mw[2] = {(uint32_t)m, (uint32_t)(m >> 32)};
    if (mw[1] == 0) {
        const uint32_t m1[1] = {mw[0]};
        wmad<NL, 1>(acc, x, m1);
    } else {
        wmad<NL, 2>(acc, x, mw);
    }
}

template <int NL>
__device__ __forceinline__ void wmad128(uint32_t (&acc)[NL], const uint32_t* x, u128 m) {
    const uint32_t mw[4] = {(uint32_t)m, (uint32_t)(m >> 32), (uint32_t)(m >> 64), (uint32_t)(m >> 96)};
    if (!(m >> 64)) {
        const uint32_t m2[2] = {mw[0], mw[1]};
        wmad<NL, 2>(acc, x, m2);
    } else {
        wmad<NL, 4>(acc, x, mw);
    }
}

template <int NL>
__device__ __forceinline__ uint64_t wtop64(const uint32_t (&x)[NL]) {
    return ((uint64_t)x[NL - 1] << 32) | x[NL - 2];
}

// -x mod 2^F (= ~x + 1; one single-statement carry chain, see addc_chain)
template <int NL>
__device__ __forceinline__ void wneg(uint32_t (&y)[NL], const uint32_t (&x)[NL]) {
    uint32_t one[NL];
#pragma unroll
    for (int l = 0; l < NL; l++) {
        y[l] = ~x[l];
        one[l] = l == 0;
    }
    addc_chain<NL>(y, one);
}

template <int NL>
__device__ __forceinline__ uint64_t wtop64_neg(const uint32_t (&x)[NL]) {  // top 64 bits of -x mod 2^F
    uint32_t y[NL];
    wneg<NL>(y, x);
    return ((uint64_t)y[NL - 1] << 32) | y[NL - 2];
}

// x / k for k in 1..8 when k divides x exactly: shift out the power of two,
// multiply by the inverse of the odd part mod 2^128 (no 128-bit division)
__device__ __forceinline__ u128 exact_div_small(u128 x, int k) {
    const u128 INV3 = ((u128)0xAAAAAAAAAAAAAAAAull << 64) | 0xAAAAAAAAAAAAAAABull;
    const u128 INV5 = ((u128)0xCCCCCCCCCCCCCCCCull << 64) | 0xCCCCCCCCCCCCCCCDull;
    const u128 INV7 = ((u128)0xB6DB6DB6DB6DB6DBull << 64) | 0x6DB6DB6DB6DB6DB7ull;
    switch (k) {
        case 2: return x >> 1;
        case 3: return x * INV3;
        case 4: return x >> 2;
        case 5: return x * INV5;
        case 6: return (x >> 1) * INV3;
        case 7: return x * INV7;
        case 8: return x >> 3;
        default: return x;
    }
}

// bn[k] = C(x, k), k = 0..K, for x < 2^16 (every value < 2^128), exactly
template <int K>
__device__ __forceinline__ void binoms_u128(uint64_t x, u128 (&bn)[K + 1]) {
    bn[0] = 1;
#pragma unroll
    for (int k = 1; k <= K; k++)
        bn[k] = x + 1 < (uint64_t)k ? (u128)0 : exact_div_small(bn[k - 1] * (u128)(x + 1 - k), k);
}

__device__ __forceinline__ uint64_t exact_div_small64(uint64_t x, int k) {  // as exact_div_small, mod 2^64
    switch (k) {
        case 2: return x >> 1;
        case 3: return x * 0xAAAAAAAAAAAAAAABull;
        case 4: return x >> 2;
        case 5: return x * 0xCCCCCCCCCCCCCCCDull;
        case 6: return (x >> 1) * 0xAAAAAAAAAAAAAAABull;
        case 7: return x * 0x6DB6DB6DB6DB6DB7ull;
        case 8: return x >> 3;
        default: return x;
    }
}

// bn[k] = C(x, k), k = 0..K, for x < 512 (every value < 2^53)
template <int K>
__device__ __forceinline__ void binoms_u64(uint64_t x, uint64_t (&bn)[K + 1]) {
    bn[0] = 1;
#pragma unroll
    for (int k = 1; k <= K; k++) bn[k] = x + 1 < (uint64_t)k ? 0 : exact_div_small64(bn[k - 1] * (x + 1 - k), k);
}

// C(x, k) mod 2^(32 NL) for x < 2^32, k <= 8, computed exactly in 9 words
// (the divisor of each step is a compile-time constant once unrolled)
template <int NL>
__device__ void binom_big(uint64_t x, int k, uint32_t (&out)[NL]) {
    uint32_t c[9] = {1, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int r = 0; r < 8; r++) {
        if (r < k) {
            if (x < (uint64_t)r + 1) {
#pragma unroll
                for (int l = 0; l < 9; l++) c[l] = 0;
            }
            const uint64_t f = x - (uint64_t)r;
            uint64_t carry = 0;
#pragma unroll
            for (int l = 0; l < 9; l++) {
                const uint64_t p = (uint64_t)c[l] * f + carry;
                c[l] = (uint32_t)p;
                carry = p >> 32;
            }
            uint64_t rem = 0;
#pragma unroll
            for (int l = 8; l >= 0; l--) {
                const uint64_t cur = (rem << 32) | c[l];
                c[l] = (uint32_t)(cur / (uint64_t)(r + 1));
                rem = cur % (uint64_t)(r + 1);
            }
        }
    }
#pragma unroll
    for (int l = 0; l < NL; l++) out[l] = c[l];
}

template <int NL>
__device__ __forceinline__ void wload(uint32_t (&x)[NL], const uint32_t* p, int64_t stride) {
#pragma unroll
    for (int l = 0; l < NL; l++) x[l] = __ldg(p + l * stride);
}

// ---------------------------------------------------------------- seeds
// one 64-thread block per tile (grid-stride): threads 0..D compute
// C(i0, k) exactly once per tile, then thread c < ncoef forms column entry c
template <int NL>
__global__ void __launch_bounds__(64) wseed_kernel(WideDev w, const uint64_t* tile_base, uint32_t* seeds) {
    __shared__ uint32_t bn[WMAXD + 1][NL];
    const uint64_t tiles = tile_base[w.g.S];
    const int c = threadIdx.x;
    int j = 0;
    while (j < w.D && wcol(w.D, j + 1, 0) <= c) j++;
    const int l = c - wcol(w.D, j, 0);
    for (uint64_t gt = blockIdx.x; gt < tiles; gt += gridDim.x) {
        const int64_t t = locate_super(tile_base, w.g.S, gt);
        const uint64_t i0 = (gt - tile_base[t]) * TILE;
        __syncthreads();  // the previous tile's binomials are consumed
        if (c <= w.D) {
            uint32_t b[NL];
            if (i0 < (1ull << 25) && c <= 5) {  // C(i0, c) < 2^125: exact in 128 bits, no divisions
                u128 bb[6];
                binoms_u128<5>(i0, bb);
                const u128 v = bb[c];
#pragma unroll
                for (int q = 0; q < NL; q++) b[q] = q < 4 ? (uint32_t)(v >> (32 * q)) : 0u;
            } else {
                binom_big<NL>(i0, c, b);
            }
#pragma unroll
            for (int q = 0; q < NL; q++) bn[c][q] = b[q];
        }
        __syncthreads();
        if (c < w.ncoef) {
            uint32_t acc[NL];
#pragma unroll
            for (int q = 0; q < NL; q++) acc[q] = 0;
            for (int m = l; m <= w.D - j; m++) {
                uint32_t qv[NL];
                wload<NL>(qv, w.coef + ((int64_t)wcol(w.D, j, m) * NL) * w.g.S + t, w.g.S);
                // acc += qv * C(i0, m - l) mod 2^F
#pragma unroll
                for (int h = 0; h < NL; h++) {
                    const uint32_t bh = bn[m - l][h];
                    uint32_t carry = 0;
#pragma unroll
                    for (int q = 0; q + h < NL; q++) {
                        const uint64_t p = (uint64_t)qv[q] * bh + acc[q + h] + carry;
                        acc[q + h] = (uint32_t)p;
                        carry = (uint32_t)(p >> 32);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < NL; q++) seeds[(gt * w.ncoef + c) * NL + q] = acc[q];
        }
    }
}

// --------------------------------------------------------------- phase 1
constexpr int WPKT = TILE / 32;            // consecutive domains walked per lane (16)
constexpr int WSTAGE = TILE + TILE / WPKT;  // staged problems per warp, one pad word per packet

__device__ __forceinline__ int wstage_idx(int d) { return d + d / WPKT; }

struct ABSrc {  // problems staged in shared memory by the walk
    const uint64_t* A;
    const uint64_t* B;
    uint64_t pad_full, pad_last;
    uint32_t dbase, nd, nfull, nlast;
    int lane;
    __device__ __forceinline__ bool one(int k, uint64_t& a, uint64_t& b, uint64_t& eps, uint32_t& N) {
        const int d = lane + 32 * k;
        const uint32_t i = dbase + (uint32_t)d;
        if (i >= nd) return false;
        const bool last = i == nd - 1;
        const int x = wstage_idx(d);
        a = A[x];
        b = B[x];
        eps = 2 * (last ? pad_last : pad_full);
        N = last ? nlast : nfull;
        return true;
    }
    __device__ __forceinline__ void build2(int k, bool& v0, uint64_t& a0, uint64_t& b0, uint64_t& e0, uint32_t& N0,
                                           bool& v1, uint64_t& a1, uint64_t& b1, uint64_t& e1, uint32_t& N1) {
        v0 = one(k, a0, b0, e0, N0);
        v1 = one(k + 1, a1, b1, e1, N1);
    }
    __device__ __forceinline__ void done(int, bool, uint64_t, uint32_t) {}
};

// walk the lane's packet of WPKT domains for column j (r_0 -> b, r_1 -> a):
// seed from the tile column by E^(16 lane), then tabulated steps
template <int D, int NL, bool IS_B>
__device__ __forceinline__ void wwalk_packet(const uint32_t* tcol, int lane, uint64_t* out, uint32_t dbase,
                                             uint32_t nd, uint64_t pad_full, uint64_t pad_last) {
    constexpr int E = IS_B ? D + 1 : D;  // entries of the column (degree of r_j + 1)
    uint32_t c[E][NL];
    const uint64_t off = (uint64_t)WPKT * lane;
    uint64_t bn[E];
    binoms_u64<E - 1>(off, bn);
#pragma unroll
    for (int l = 0; l < E; l++) {
#pragma unroll
        for (int q = 0; q < NL; q++) c[l][q] = tcol[l * NL + q];
#pragma unroll
        for (int k = 1; l + k < E; k++) wmad64<NL>(c[l], tcol + (l + k) * NL, bn[k]);
    }
#pragma unroll 1
    for (int k = 0; k < WPKT; k++) {
        const uint32_t d = (uint32_t)(WPKT * lane + k);
        if (IS_B) {
            const uint64_t pad = dbase + d == nd - 1 ? pad_last : pad_full;
            out[wstage_idx(d)] = wtop64<NL>(c[0]) + pad;
        } else {
            out[wstage_idx(d)] = wtop64_neg<NL>(c[0]);
        }
#pragma unroll
        for (int l = 0; l + 1 < E; l++) addc_chain<NL>(c[l], c[l + 1]);
    }
}

__device__ __forceinline__ uint64_t wpad(const WideDev& w, int64_t t, uint64_t n) {
    return pad_of(ld128(w.padg, w.g.S, t), ld128(w.s2b, w.g.S, t), n, 128, 64);
}

template <int D, int NL>
__global__ void __launch_bounds__(128, HRB_P1_MINB) phase1_wide_kernel(WideDev w, int algo,
                                                                       const uint64_t* tile_base, uint32_t* bitmap,
                                                                       uint32_t* tile_t,
                                                                       unsigned long long* iter_sum,
                                                                       unsigned long long* tile_ctr) {
    __shared__ uint64_t sA[4][WSTAGE];
    __shared__ uint64_t sB[4][WSTAGE];
    __shared__ uint32_t scol[4][(2 * D + 1) * NL];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t units = tile_base[w.g.S];
    const int ncol = (2 * D + 1) * NL;
    unsigned long long iters = 0;
    uint64_t u = warp0;
    while (u < units) {
        unsigned long long next = 0;
        if (lane == 0) next = nwarps + atomicAdd(tile_ctr, 1ull);
        const int64_t t = locate_super(tile_base, w.g.S, u);
        const uint64_t tile = u - tile_base[t];
        ABSrc src;
        src.A = sA[wq];
        src.B = sB[wq];
        src.lane = lane;
        src.nd = __ldg(&w.g.n_dom[t]);
        src.nfull = __ldg(&w.g.dom_n[t]);
        src.nlast = __ldg(&w.g.last_n[t]);
        src.pad_full = wpad(w, t, src.nfull);
        src.pad_last = wpad(w, t, src.nlast);
        src.dbase = (uint32_t)(tile * TILE);
        // the tile's r_0 and r_1 columns (the first 2D + 1 coefficient columns)
        for (int x = lane; x < ncol; x += 32) scol[wq][x] = __ldg(&w.seeds[u * w.ncoef * NL + x]);
        __syncwarp();
        wwalk_packet<D, NL, true>(scol[wq], lane, sB[wq], src.dbase, src.nd, src.pad_full, src.pad_last);
        wwalk_packet<D, NL, false>(scol[wq] + (D + 1) * NL, lane, sA[wq], src.dbase, src.nd, src.pad_full,
                                   src.pad_last);
        __syncwarp();
        unsigned long long its = 0;
        const uint32_t fails = hrb::lane_items<64, NU>(src, &its, algo == hrb::ALGO_REGULAR_UNROLLED, NU);
        iters += its;
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < NU; k++) {
            uint32_t wd = __ballot_sync(0xffffffffu, (fails >> k) & 1u);
            if (lane == k) mine = wd;
        }
        if (lane < NU) bitmap[u * NU + lane] = mine;
        if (lane == 0) tile_t[u] = (uint32_t)t;
        __syncwarp();  // the staged problems are read before the next tile overwrites them
        u = __shfl_sync(0xffffffffu, next, 0);
    }
    for (int o = 16; o > 0; o >>= 1) iters += __shfl_xor_sync(0xffffffffu, iters, o);
    if (iter_sum && lane == 0 && iters) atomicAdd(iter_sum, iters);
}

// s_j(i) for j = 0..D of domain i (super-domain t) into sc[j][NL], from the
// unit-step columns of its tile (E^(i - i0))
template <int D, int NL>
__device__ __forceinline__ void wdomain_poly(const WideDev& w, const uint64_t* tile_base, int64_t t, uint64_t i,
                                             uint32_t* sc /* [(D+1) NL] */) {
    const uint64_t gt = tile_base[t] + i / TILE;
    const uint64_t di = i % TILE;
    const uint32_t* col = w.seeds + gt * w.ncoef * NL;
    uint64_t bn[D + 1];
    binoms_u64<D>(di, bn);
#pragma unroll
    for (int j = 0; j <= D; j++) {
        uint32_t acc[NL];
        const uint32_t* cj = col + wcol(D, j, 0) * NL;
#pragma unroll
        for (int q = 0; q < NL; q++) acc[q] = __ldg(&cj[q]);
#pragma unroll
        for (int k = 1; k <= D - j; k++) {
            uint32_t x[NL];
#pragma unroll
            for (int q = 0; q < NL; q++) x[q] = __ldg(&cj[k * NL + q]);
            wmad64<NL>(acc, x, bn[k]);
        }
#pragma unroll
        for (int q = 0; q < NL; q++) sc[j * NL + q] = acc[q];
    }
}

// --------------------------------------------------------------- phase 2
template <int D, int NL>
struct WSubSrc {  // the lane's subdomains, shifted from its domain polynomial
    const uint32_t* sc;  // [(D+1) NL] in shared memory
    uint64_t pad_full, pad_last;
    uint32_t nsub, step, last_cnt;
    __device__ __forceinline__ bool one(int k, uint64_t& a, uint64_t& b, uint64_t& eps, uint32_t& N) {
        const uint32_t j = (uint32_t)k;
        if (j >= nsub) return false;
        const bool last = j == nsub - 1;
        const uint64_t start = (uint64_t)j * step;
        uint32_t s0[NL], s1[NL];
#pragma unroll
        for (int q = 0; q < NL; q++) {
            s0[q] = sc[q];
            s1[q] = sc[NL + q];
        }
        u128 bn[D + 1];
        binoms_u128<D>(start, bn);
#pragma unroll
        for (int k2 = 1; k2 <= D; k2++) {
            wmad128<NL>(s0, sc + k2 * NL, bn[k2]);                  // s_k2 C(start, k2)
            if (k2 >= 2) wmad128<NL>(s1, sc + k2 * NL, bn[k2 - 1]);  // s_k2 C(start, k2 - 1)
        }
        const uint64_t pad = last ? pad_last : pad_full;
        a = wtop64_neg<NL>(s1);
        b = wtop64<NL>(s0) + pad;
        eps = 2 * pad;
        N = last ? last_cnt : step;
        return true;
    }
    __device__ __forceinline__ void build2(int k, bool& v0, uint64_t& a0, uint64_t& b0, uint64_t& e0, uint32_t& N0,
                                           bool& v1, uint64_t& a1, uint64_t& b1, uint64_t& e1, uint32_t& N1) {
        v0 = one(k, a0, b0, e0, N0);
        v1 = one(k + 1, a1, b1, e1, N1);
    }
    __device__ __forceinline__ void done(int, bool, uint64_t, uint32_t) {}
};

template <int D, int NL>
__global__ void __launch_bounds__(128, HRB_P2_MINB) phase2_wide_kernel(WideDev w, int split, int algo,
                                                                       const uint64_t* tile_base,
                                                                       const uint64_t* fail_ids,
                                                                       const uint32_t* fail_t,
                                                                       const uint64_t* fail_count, uint64_t fail_cap,
                                                                       unsigned long long* meta, uint32_t* bitmap) {
    __shared__ uint32_t sc[128][(D + 1) * NL];
    uint64_t nf = *fail_count;
    if (nf > fail_cap) nf = fail_cap;
    const uint64_t nf_pad = (nf + 31) & ~31ull;
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t chunk = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    WSubSrc<D, NL> src;
    src.sc = sc[threadIdx.x];
    while (32 * chunk < nf_pad) {
        unsigned long long next = 0;
        if (lane == 0) next = nwarps + atomicAdd(&meta[5], 1ull);
        const uint64_t f = 32 * chunk + lane;
        const bool valid = f < nf;
        src.nsub = 0;
        if (valid) {
            const uint64_t id = fail_ids[f];
            const int64_t t = fail_t[f];
            const uint64_t i = id - __ldg(&w.g.dom_base[t]);
            const uint64_t n = domain_size(w.g, t, i);
            uint64_t step = udiv_small(n, (uint32_t)split);
            if (step < 1) step = 1;
            const uint64_t nsub = udiv_small(n + step - 1, (uint32_t)step);
            wdomain_poly<D, NL>(w, tile_base, t, i, sc[threadIdx.x]);
            src.nsub = (uint32_t)nsub;
            src.step = (uint32_t)step;
            src.last_cnt = (uint32_t)(n - (nsub - 1) * step);
            src.pad_full = wpad(w, t, step);
            src.pad_last = wpad(w, t, src.last_cnt);
        }
        unsigned long long its = 0;
        const uint32_t fails = hrb::lane_items<64, 32>(src, &its, algo == hrb::ALGO_REGULAR_UNROLLED, src.nsub);
        if (valid) bitmap[f] = fails;
        chunk = __shfl_sync(0xffffffffu, next, 0);
    }
}

// --------------------------------------------------------------- phase 3
template <int D, int NL>
__device__ __forceinline__ void wcolumn_at(const uint32_t* sc, uint64_t x0, uint32_t (&c)[D + 1][NL]) {
    // Delta^l P(x0) = sum_{k >= l} s_k C(x0, k - l)
    u128 bn[D + 1];
    binoms_u128<D>(x0, bn);
#pragma unroll
    for (int l = 0; l <= D; l++) {
#pragma unroll
        for (int q = 0; q < NL; q++) c[l][q] = sc[l * NL + q];
#pragma unroll
        for (int k = l + 1; k <= D; k++) wmad128<NL>(c[l], sc + k * NL, bn[k - l]);
    }
}

// x < y (multi-limb, unsigned)
template <int NL>
__device__ __forceinline__ bool wless(const uint32_t (&x)[NL], const uint32_t (&y)[NL]) {
#pragma unroll
    for (int q = NL - 1; q >= 0; q--)
        if (x[q] != y[q]) return x[q] < y[q];
    return false;
}

template <int D, int NL>
__global__ void __launch_bounds__(128) phase3_wide_kernel(WideDev w, int split, const uint64_t* tile_base,
                                                          const uint64_t* sub_keys, const uint32_t* sub_t,
                                                          const uint64_t* sub_count, uint64_t sub_cap,
                                                          const unsigned long long* meta, uint32_t* item_counts,
                                                          Cand* app, unsigned long long* app_count,
                                                          uint64_t app_cap) {
    __shared__ uint32_t sc_all[128][(D + 1) * NL];
    uint32_t* sc = sc_all[threadIdx.x];
    const int lane = threadIdx.x & 31;
    const uint64_t maxstep = meta[1];
    const uint32_t CHUNK3 = (uint32_t)meta[2];
    const uint64_t CH = (maxstep + CHUNK3 - 1) / CHUNK3;
    uint64_t ns = *sub_count;
    if (ns > sub_cap) ns = sub_cap;
    const uint64_t n_items = ns * CH;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; base < n_items; base += stride) {
        const uint64_t g = base + lane;
        uint32_t len = 0;
        uint64_t mbase = 0, dom = 0, o = 0;
        uint32_t K[NL], wm1[NL];
        if (g < n_items) {
            const uint64_t r = udiv_small(g, (uint32_t)CH), ch = g - r * CH;
            const uint64_t key = sub_keys[r];
            dom = key >> 8;
            const uint64_t j = key & 255;
            const int64_t t = sub_t[r];
            const uint64_t i = dom - w.g.dom_base[t];
            const uint64_t n = domain_size(w.g, t, i);
            uint64_t step = udiv_small(n, (uint32_t)split);
            if (step < 1) step = 1;
            const uint64_t start = j * step;
            const uint64_t cnt = n - start < step ? n - start : step;
            const uint64_t x0 = ch * CHUNK3;
            if (x0 < cnt) {
                len = (uint32_t)(cnt - x0 < CHUNK3 ? cnt - x0 : CHUNK3);
                o = start + x0;
                wdomain_poly<D, NL>(w, tile_base, t, i, sc);
                mbase = __ldg(&w.g.m0[t]) + i * (uint64_t)__ldg(&w.g.dom_n[t]) + o;
                // window = ceil(eps' 2^F) + 1 (pipeline.py:274); K = 2 window - 1, wm1 = window - 1
                uint32_t win[NL];
                wload<NL>(win, w.win + t, w.g.S);
#pragma unroll
                for (int q = 0; q < NL; q++) wm1[q] = win[q];
                {
                    uint32_t minus1[NL];
#pragma unroll
                    for (int q = 0; q < NL; q++) minus1[q] = 0xFFFFFFFFu;  // -1 mod 2^F
                    addc_chain<NL>(wm1, minus1);                          // window - 1
                }
#pragma unroll
                for (int q = 0; q < NL; q++) K[q] = wm1[q];
                addc_chain<NL>(K, win);  // 2 window - 1
            }
        }
        uint32_t rank = 0;
        uint32_t c[D + 1][NL];
        if (len) {
            wcolumn_at<D, NL>(sc, o, c);
            addc_chain<NL>(c[0], wm1);  // V = v + window - 1 (mod 2^F)
        } else {
#pragma unroll
            for (int l = 0; l <= D; l++)
#pragma unroll
                for (int q = 0; q < NL; q++) c[l][q] = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < NL; q++) K[q] = 0;
        }
        // Hot loop, D <= 4, on 32-bit proxies of the columns' top limbs, each
        // stepped by the next one's: a top limb misses at most one carry per
        // step, so after x < 32 steps the proxy of column 0 lies below the
        // true top limb by at most e(x) (wproxy_margin).  With u = proxy + M,
        // V < K  =>  top(V) <= top(K)  =>  u <= top(K) + M (no wrap on either
        // side).  D adds and half a min per argument instead of D NL-limb
        // add-with-carry chains; the exact columns advance once per block of
        // 32 (the closed form, sum of C(32, k) multiples), and a flagged block
        // is re-walked exactly as before.  Higher degrees walk exactly: their
        // margins (up to 1.5e7 at D = 8) would flag too many blocks.
        constexpr bool PROXY = D <= 4;
        constexpr uint32_t M = PROXY ? wproxy_margin<D>() : 0u;
        const uint32_t Ktop = K[NL - 1];
        const uint32_t KtopM = Ktop > 0xFFFFFFFFu - M ? 0xFFFFFFFFu : Ktop + M;
        for (uint32_t xb = 0; xb < CHUNK3; xb += 32) {
            uint32_t lo_top = 0xFFFFFFFFu;  // conservative: V < K implies top limb(V) <= top limb(K)
            if constexpr (PROXY) {
                uint32_t pr[D + 1];
#pragma unroll
                for (int l = 0; l <= D; l++) pr[l] = c[l][NL - 1];
                pr[0] += M;
#pragma unroll
                for (uint32_t x = 0; x < 32; x++) {
                    lo_top = min(lo_top, pr[0]);
#pragma unroll
                    for (int l = 0; l < D; l++) pr[l] += pr[l + 1];
                }
                // exact: c_l(x + 32) = sum_k C(32, k) c_{l+k}(x), in
                // increasing l (each row reads only higher rows, not yet
                // advanced)
#pragma unroll
                for (int l = 0; l < D; l++) {
#pragma unroll
                    for (int k = 1; l + k <= D; k++) {
                        const uint32_t m1[1] = {wbinom32(k)};
                        wmad<NL, 1>(c[l], c[l + k], m1);
                    }
                }
            } else {
#pragma unroll 4
                for (uint32_t x = 0; x < 32; x++) {
                    lo_top = min(lo_top, c[0][NL - 1]);
#pragma unroll
                    for (int l = 0; l < D; l++) addc_chain<NL>(c[l], c[l + 1]);
                }
            }
            const bool any = len > xb && lo_top <= KtopM;
            if (__any_sync(0xffffffffu, any)) {  // rare: re-walk the block exactly, append in order
                uint32_t e[D + 1][NL];
                if (len > xb) {
                    wcolumn_at<D, NL>(sc, o + xb, e);
                    addc_chain<NL>(e[0], wm1);
                }
                for (uint32_t x = 0; x < 32; x++) {
                    const bool hit = (xb + x < len) && wless<NL>(e[0], K);
                    const uint32_t ball = __ballot_sync(0xffffffffu, hit);
                    if (ball) {
                        const int leader = __ffs(ball) - 1;
                        unsigned long long pos = 0;
                        if (lane == leader) pos = atomicAdd(app_count, (unsigned long long)__popc(ball));
                        pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(ball & ((1u << lane) - 1));
                        if (hit) {
                            if (pos < app_cap) {
                                // v = V - (window - 1); dist = min(v, 2^F - v), floored to 2^-64
                                uint32_t v[NL], nv[NL], mw[NL];
                                wneg<NL>(mw, wm1);
#pragma unroll
                                for (int q = 0; q < NL; q++) v[q] = e[0][q];
                                addc_chain<NL>(v, mw);
                                wneg<NL>(nv, v);
                                bool vzero = true;
#pragma unroll
                                for (int q = 0; q < NL; q++) vzero = vzero && v[q] == 0;
                                const bool use_v = vzero || wless<NL>(v, nv);
                                Cand cd;
                                cd.m = mbase + xb + x;
                                cd.dist = use_v ? wtop64<NL>(v) : wtop64<NL>(nv);
                                cd.dom = dom;
                                cd.item = g;
                                cd.rank = rank;
                                app[pos] = cd;
                            }
                            rank++;
                        }
                    }
#pragma unroll
                    for (int l = 0; l < D; l++) addc_chain<NL>(e[l], e[l + 1]);
                }
            }
        }
        if (g < n_items) item_counts[g] = rank;
    }
}

// ------------------------------------------------ tabulated values (tests)
// every domain's (s_0..s_D) mod 2^F through the same packet walk as phase 1
// (all D+1 columns): out [D+1][NL][n_total]
template <int D, int NL>
__global__ void __launch_bounds__(128) wtabdiff_kernel(WideDev w, const uint64_t* tile_base, int64_t n_total,
                                                       uint32_t* out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t total_tiles = tile_base[w.g.S];
    for (uint64_t u = warp0; u < total_tiles; u += nwarps) {
        const int64_t t = locate_super(tile_base, w.g.S, u);
        const uint64_t tile = u - tile_base[t];
        const uint32_t nd = __ldg(&w.g.n_dom[t]);
        const uint64_t gbase = w.g.dom_base[t];
        const uint32_t* tcol = w.seeds + u * w.ncoef * NL;
        const uint64_t off = (uint64_t)WPKT * lane;
        for (int j = 0; j <= D; j++) {
            const int E = D - j + 1;
            uint32_t c[WMAXD + 1][NL];
            for (int l = 0; l < E; l++) {
                for (int q = 0; q < NL; q++) c[l][q] = __ldg(&tcol[(wcol(D, j, l)) * NL + q]);
                uint64_t bo[WMAXD + 1];
                binoms_u64<WMAXD>(off, bo);
                for (int k = 1; l + k < E; k++) wmad64<NL>(c[l], tcol + wcol(D, j, l + k) * NL, bo[k]);
            }
            for (int k = 0; k < WPKT; k++) {
                const uint64_t i = tile * TILE + off + k;
                if (i < nd) {
                    for (int q = 0; q < NL; q++) out[((int64_t)j * NL + q) * n_total + gbase + i] = c[0][q];
                }
                for (int l = 0; l + 1 < E; l++) addc_chain<NL>(c[l], c[l + 1]);
            }
        }
    }
}

// ------------------------------------------------------------ host side
int check_wslice(const hrb_wslice* s) {
    if (!s) return set_err(HRB_ERR_CONFIG, "null slice");
    if (s->n_super < 1) return set_err(HRB_ERR_CONFIG, "slice has no super-domains");
    if (s->degree < 3 || s->degree > 8) return set_err(HRB_ERR_CONFIG, "wide slices need degree 3..8");
    if (s->frac_limbs != (s->degree > 4 ? s->degree : 4))
        return set_err(HRB_ERR_CONFIG, "wide slices use frac_limbs = max(4, degree)");
    if (s->word_bits != 64) return set_err(HRB_ERR_CONFIG, "wide slices use word_bits = 64");
    if (s->max_dom_n > 65536) return set_err(HRB_ERR_CONFIG, "wide slices need domains of at most 2^16 arguments");
    return HRB_OK;
}

WideDev to_wdev(const hrb_wslice* s) {
    WideDev w;
    hrb_slice g = {};
    g.n_super = s->n_super;
    g.n_total = s->n_total;
    g.max_dom_n = s->max_dom_n;
    g.coef_limbs = 4;
    g.frac_bits = 128;
    g.word_bits = 64;
    g.delta = 2;
    g.n_dom = s->n_dom;
    g.dom_n = s->dom_n;
    g.last_n = s->last_n;
    g.dom_base = s->dom_base;
    g.m0 = s->m0;
    w.g = to_dev(&g);
    w.D = s->degree;
    w.NL = s->frac_limbs;
    w.ncoef = (w.D + 1) * (w.D + 2) / 2;
    w.coef = s->coef;
    w.padg = s->padg;
    w.s2b = s->s2b;
    w.win = s->win;
    w.seeds = nullptr;
    return w;
}

// dispatch on (D, NL = max(4, D))
#define HRB_WIDE_DISPATCH(D_, MACRO) \
    switch (D_) {                    \
        case 3: MACRO(3, 4); break;  \
        case 4: MACRO(4, 4); break;  \
        case 5: MACRO(5, 5); break;  \
        case 6: MACRO(6, 6); break;  \
        case 7: MACRO(7, 7); break;  \
        case 8: MACRO(8, 8); break;  \
        default: return set_err(HRB_ERR_CONFIG, "degree outside 3..8"); \
    }

struct WideWs {
    Buf seeds;
};
WideWs g_wws[64];

int run_wslice_locked(Workspace& ws, WideWs& wws, const hrb_wslice* s, int algo, int split, const hrb_run_out* out,
                      cudaStream_t st, uint64_t* argsums) {
    int rc;
    WideDev w = to_wdev(s);
    uint64_t* counts = out->counts;
    CK(cudaMemsetAsync(counts, 0, sizeof(uint64_t) * 4, st));
    if ((rc = ws_prep(ws, w.g, split, st))) return rc;
    const uint64_t max_tiles = (uint64_t)s->n_total / TILE + (uint64_t)s->n_super + 1;
    if ((rc = wws.seeds.ensure(sizeof(uint32_t) * max_tiles * w.ncoef * w.NL))) return rc;
    w.seeds = (const uint32_t*)wws.seeds.p;
    auto tb = (const uint64_t*)ws.tile_base.p;
#define SEED(D_, NL_) \
    wseed_kernel<NL_><<<sm_count() * 16, 64, 0, st>>>(w, tb, (uint32_t*)wws.seeds.p)
    HRB_WIDE_DISPATCH(w.D, SEED)
#undef SEED
    CK(cudaGetLastError());
    // phase 1
    if ((rc = ws.bm1.ensure(sizeof(uint32_t) * max_tiles * NU))) return rc;
    if ((rc = ws.tile_t.ensure(sizeof(uint32_t) * max_tiles))) return rc;
    if ((rc = ws.fail_t.ensure(sizeof(uint32_t) * (out->fail_cap + 1)))) return rc;
    auto tc = (unsigned long long*)ws.meta.p + 4;
    const int g1 = sm_count() * HRB_P1_MINB;
#define P1W(D_, NL_)                                                                                            \
    phase1_wide_kernel<D_, NL_><<<g1, 128, 0, st>>>(w, algo, tb, (uint32_t*)ws.bm1.p, (uint32_t*)ws.tile_t.p, \
                                                    (unsigned long long*)(counts + 3), tc)
    HRB_WIDE_DISPATCH(w.D, P1W)
#undef P1W
    CK(cudaGetLastError());
    {
        P1Compact fn{(const uint32_t*)ws.bm1.p, tb, (const uint32_t*)ws.tile_t.p, s->dom_base, w.g.S, out->fail_ids,
                     (uint32_t*)ws.fail_t.p, out->fail_cap};
        if ((rc = run_compact(ws, fn, counts + 0, st))) return rc;
    }
    // phase 2 (one bitmap word per failing domain: J <= 32)
    if ((rc = ws.bm2.ensure(sizeof(uint32_t) * (out->fail_cap + 1)))) return rc;
    if ((rc = ws.sub_t.ensure(sizeof(uint32_t) * (out->sub_cap + 1)))) return rc;
    auto mt = (unsigned long long*)ws.meta.p;
    const int g2 = sm_count() * HRB_P2_MINB;
#define P2W(D_, NL_)                                                                                             \
    phase2_wide_kernel<D_, NL_><<<g2, 128, 0, st>>>(w, split, algo, tb, out->fail_ids, (const uint32_t*)ws.fail_t.p, \
                                                    counts + 0, out->fail_cap, mt, (uint32_t*)ws.bm2.p)
    HRB_WIDE_DISPATCH(w.D, P2W)
#undef P2W
    CK(cudaGetLastError());
    {
        P2Compact fn{(const uint32_t*)ws.bm2.p, out->fail_ids, (const uint32_t*)ws.fail_t.p, counts + 0, out->fail_cap,
                     mt, out->sub_keys, (uint32_t*)ws.sub_t.p, out->sub_cap};
        if ((rc = run_compact(ws, fn, counts + 1, st))) return rc;
    }
    // phase 3
    {
        const uint64_t sub_cap = out->sub_cap;
        const uint64_t maxstep = s->max_dom_n;
        const uint64_t min_items = (uint64_t)sm_count() * 2048;
        const uint64_t CH = (maxstep + CHUNK3_MAX - 1) / CHUNK3_MAX;
        const uint64_t ch_min = (maxstep + CHUNK3_MIN - 1) / CHUNK3_MIN;
        uint64_t items = sub_cap * (CH ? CH : 1);
        items = items > 2 * min_items + sub_cap ? items : 2 * min_items + sub_cap;
        if (items > sub_cap * ch_min) items = sub_cap * ch_min;
        if ((rc = ws.counts3.ensure(sizeof(uint32_t) * (items + 1)))) return rc;
        if ((rc = ws.offs3.ensure(sizeof(uint64_t) * (items + 1)))) return rc;
        if ((rc = ws.app.ensure(sizeof(Cand) * (out->cand_cap + 1)))) return rc;
        if ((rc = ws.appc.ensure(sizeof(unsigned long long)))) return rc;
        CK(cudaMemsetAsync(ws.appc.p, 0, sizeof(unsigned long long), st));
        chunk3_kernel<<<1, 1, 0, st>>>(mt, counts + 1, sub_cap, min_items);
#define P3W(D_, NL_)                                                                                              \
    phase3_wide_kernel<D_, NL_><<<sm_count() * 8, 128, 0, st>>>(                                                 \
        w, split, tb, out->sub_keys, (const uint32_t*)ws.sub_t.p, counts + 1, sub_cap, mt, (uint32_t*)ws.counts3.p, \
        (Cand*)ws.app.p, (unsigned long long*)ws.appc.p, out->cand_cap)
        HRB_WIDE_DISPATCH(w.D, P3W)
#undef P3W
        CK(cudaGetLastError());
        P3Offsets fn{(const uint32_t*)ws.counts3.p, counts + 1, sub_cap, mt, (uint64_t*)ws.offs3.p};
        if ((rc = run_compact(ws, fn, counts + 2, st))) return rc;
        scatter3_kernel<<<sm_count() * 2, 256, 0, st>>>((const Cand*)ws.app.p, (const unsigned long long*)ws.appc.p,
                                                        out->cand_cap, (const uint64_t*)ws.offs3.p, out->cand_index,
                                                        out->cand_dist, out->cand_dom, out->cand_cap);
        CK(cudaGetLastError());
    }
    if (argsums) {
        CK(cudaMemsetAsync(argsums, 0, sizeof(uint64_t) * 2, st));
        argsum_kernel<<<sm_count() * 4, 256, 0, st>>>(w.g, split, out->fail_ids, (const uint32_t*)ws.fail_t.p,
                                                      counts + 0, out->fail_cap, out->sub_keys,
                                                      (const uint32_t*)ws.sub_t.p, counts + 1, out->sub_cap,
                                                      (unsigned long long*)argsums);
        CK(cudaGetLastError());
    }
    return HRB_OK;
}

int wtabdiff_impl(Workspace& ws, WideWs& wws, const hrb_wslice* s, uint32_t* out, cudaStream_t st) {
    int rc;
    WideDev w = to_wdev(s);
    if ((rc = ws_prep(ws, w.g, 8, st))) return rc;
    const uint64_t max_tiles = (uint64_t)s->n_total / TILE + (uint64_t)s->n_super + 1;
    if ((rc = wws.seeds.ensure(sizeof(uint32_t) * max_tiles * w.ncoef * w.NL))) return rc;
    w.seeds = (const uint32_t*)wws.seeds.p;
    auto tb = (const uint64_t*)ws.tile_base.p;
#define SEED(D_, NL_) wseed_kernel<NL_><<<sm_count() * 16, 64, 0, st>>>(w, tb, (uint32_t*)wws.seeds.p)
    HRB_WIDE_DISPATCH(w.D, SEED)
#undef SEED
#define TABW(D_, NL_) wtabdiff_kernel<D_, NL_><<<sm_count() * 4, 128, 0, st>>>(w, tb, s->n_total, out)
    HRB_WIDE_DISPATCH(w.D, TABW)
#undef TABW
    CK(cudaGetLastError());
    return HRB_OK;
}
