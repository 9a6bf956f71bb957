// bign.h -- small exact integers for the host polynomial generator.
//
// Fixed-capacity multi-word integers (64-bit words, little endian), signed
// values as sign + magnitude, and dyadic rationals m * 2^e.  Everything the
// Taylor model, the error budget and the confirmation need is exact integer
// arithmetic on a few hundred bits, so this replaces Python's int / Fraction
// on that path.  A result that would not fit the capacity sets the calling
// thread's overflow flag (the caller then hands the item to the exact Python
// path) instead of wrapping.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>

// The same source compiles for the host (g++, libhrbhost.so) and for the
// device (nvcc, the confirmation kernel in libhrb200.so): one exact
// arithmetic, two targets.
#if defined(__CUDACC__)
#define HRBH_HD __host__ __device__ __forceinline__
#else
#define HRBH_HD inline
#endif

namespace hrbh {

typedef unsigned __int128 u128;
#ifndef HRBH_NW
#define HRBH_NW 16
#endif
constexpr int NW = HRBH_NW;  // 1024 bits on the host: exp_basecase squares ~420-bit values at wp <= 400

HRBH_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

HRBH_HD int ctz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __ffsll((long long)x) - 1;
#else
    return __builtin_ctzll(x);
#endif
}

HRBH_HD int imax(int a, int b) { return a > b ? a : b; }

// Overflow of the fixed capacity: the host path reads it (and hands the
// item to the exact Python path); device callers size their inputs so it
// cannot happen (see confirm.cuh) and never read it.
#if defined(__CUDACC__)
__device__ bool g_hrbh_ovf_sink;
__host__ __device__ inline bool& overflow_flag() {
#if defined(__CUDA_ARCH__)
    return g_hrbh_ovf_sink;
#else
    static thread_local bool f = false;
    return f;
#endif
}
#else
inline bool& overflow_flag() {
    static thread_local bool f = false;
    return f;
}
#endif

struct U {
    uint64_t w[NW];
    int n = 0;  // used words; w[n-1] != 0 unless n == 0

    HRBH_HD U() {}
    HRBH_HD explicit U(uint64_t v) { set(v); }
    HRBH_HD void set(uint64_t v) {
        n = v ? 1 : 0;
        w[0] = v;
    }
    HRBH_HD void trim() {
        while (n > 0 && w[n - 1] == 0) n--;
    }
    HRBH_HD bool zero() const { return n == 0; }
    HRBH_HD int bitlen() const { return n ? 64 * (n - 1) + (64 - clz64(w[n - 1])) : 0; }
    HRBH_HD bool bit(int k) const { return k / 64 < n && ((w[k / 64] >> (k % 64)) & 1); }
    // number of trailing zero bits (0 for zero)
    HRBH_HD int tz() const {
        for (int i = 0; i < n; i++)
            if (w[i]) return 64 * i + ctz64(w[i]);
        return 0;
    }
    // true when the low k bits are all zero
    HRBH_HD bool low_zero(int k) const {
        int q = k / 64, r = k % 64;
        for (int i = 0; i < q && i < n; i++)
            if (w[i]) return false;
        if (r && q < n && (w[q] & ((1ull << r) - 1))) return false;
        return true;
    }
    HRBH_HD uint64_t low64() const { return n ? w[0] : 0; }
};

HRBH_HD int cmp(const U& a, const U& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; i--)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

HRBH_HD U shl(const U& a, int k) {
    U r;
    if (a.zero() || k == 0) return a;
    int q = k / 64, s = k % 64;
    int n = a.n + q + 1;
    if (n > NW) {
        if (a.bitlen() + k > 64 * NW) {
            overflow_flag() = true;
            r.set(0);
            return r;
        }
        n = NW;
    }
    for (int i = 0; i < n; i++) r.w[i] = 0;
    for (int i = 0; i < a.n; i++) {
        r.w[i + q] |= a.w[i] << s;
        if (s && i + q + 1 < n) r.w[i + q + 1] |= a.w[i] >> (64 - s);
    }
    r.n = n;
    r.trim();
    return r;
}

// floor(a / 2^k)
HRBH_HD U shr(const U& a, int k) {
    U r;
    int q = k / 64, s = k % 64;
    if (q >= a.n) return r;
    r.n = a.n - q;
    for (int i = 0; i < r.n; i++) {
        uint64_t lo = a.w[i + q] >> s;
        uint64_t hi = (s && i + q + 1 < a.n) ? a.w[i + q + 1] << (64 - s) : 0;
        r.w[i] = lo | hi;
    }
    r.trim();
    return r;
}

// low k bits of a (a mod 2^k)
HRBH_HD U low_bits(const U& a, int k) {
    U r = a;
    int q = k / 64, s = k % 64;
    if (q >= r.n) return r;
    if (s) {
        r.w[q] &= (1ull << s) - 1;
        r.n = q + 1;
    } else {
        r.n = q;
    }
    r.trim();
    return r;
}

HRBH_HD U add(const U& a, const U& b) {
    const U& x = a.n >= b.n ? a : b;
    const U& y = a.n >= b.n ? b : a;
    U r;
    uint64_t c = 0;
    for (int i = 0; i < x.n; i++) {
        u128 t = (u128)x.w[i] + (i < y.n ? y.w[i] : 0) + c;
        r.w[i] = (uint64_t)t;
        c = (uint64_t)(t >> 64);
    }
    r.n = x.n;
    if (c) {
        if (r.n >= NW) {
            overflow_flag() = true;
            return r;
        }
        r.w[r.n++] = c;
    }
    return r;
}

// a - b, requires a >= b
HRBH_HD U sub(const U& a, const U& b) {
    U r;
    uint64_t br = 0;
    for (int i = 0; i < a.n; i++) {
        uint64_t y = i < b.n ? b.w[i] : 0;
        u128 t = (u128)a.w[i] - y - br;
        r.w[i] = (uint64_t)t;
        br = (uint64_t)(t >> 64) ? 1 : 0;
    }
    r.n = a.n;
    r.trim();
    return r;
}

HRBH_HD U mul(const U& a, const U& b) {
    U r;
    r.set(0);
    if (a.zero() || b.zero()) return r;
    int n = a.n + b.n;
    if (n > NW) {
        if (a.bitlen() + b.bitlen() > 64 * NW) {
            overflow_flag() = true;
            r.set(0);
            return r;
        }
        n = NW;
    }
    for (int i = 0; i < n; i++) r.w[i] = 0;
    for (int i = 0; i < a.n; i++) {
        uint64_t c = 0;
        for (int j = 0; j < b.n && i + j < n; j++) {
            u128 t = (u128)a.w[i] * b.w[j] + r.w[i + j] + c;
            r.w[i + j] = (uint64_t)t;
            c = (uint64_t)(t >> 64);
        }
        if (i + b.n < n) r.w[i + b.n] = c;
    }
    r.n = n;
    r.trim();
    return r;
}

HRBH_HD U mul_u64(const U& a, uint64_t m) { return mul(a, U(m)); }

// floor(a / d), *rem = a mod d
HRBH_HD U divmod_u64(const U& a, uint64_t d, uint64_t* rem = nullptr) {
    U r;
    u128 c = 0;
    r.n = a.n;
    for (int i = a.n - 1; i >= 0; i--) {
        u128 t = (c << 64) | a.w[i];
        r.w[i] = (uint64_t)(t / d);
        c = t % d;
    }
    r.trim();
    if (rem) *rem = (uint64_t)c;
    return r;
}

HRBH_HD U pow2(int k) { return shl(U(1), k); }

// ---------------------------------------------------------------- signed

struct S {
    U m;
    bool neg = false;  // never true for zero
    HRBH_HD S() {}
    HRBH_HD S(const U& u, bool ng = false) : m(u), neg(ng && !u.zero()) {}
    HRBH_HD static S of(int64_t v) { return v < 0 ? S(U((uint64_t)(-(v + 1)) + 1), true) : S(U((uint64_t)v)); }
    HRBH_HD bool zero() const { return m.zero(); }
};

HRBH_HD S neg(const S& a) { return S(a.m, !a.neg); }
HRBH_HD S sadd(const S& a, const S& b) {
    if (a.neg == b.neg) return S(add(a.m, b.m), a.neg);
    int c = cmp(a.m, b.m);
    if (c == 0) return S();
    if (c > 0) return S(sub(a.m, b.m), a.neg);
    return S(sub(b.m, a.m), b.neg);
}
HRBH_HD S ssub(const S& a, const S& b) { return sadd(a, neg(b)); }
HRBH_HD S smul(const S& a, const S& b) { return S(mul(a.m, b.m), a.neg != b.neg); }
HRBH_HD S sshl(const S& a, int k) { return S(shl(a.m, k), a.neg); }
HRBH_HD int scmp(const S& a, const S& b) {
    if (a.neg != b.neg) return a.neg ? -1 : 1;
    int c = cmp(a.m, b.m);
    return a.neg ? -c : c;
}
// floor(a / 2^k)
HRBH_HD S sfloor_shr(const S& a, int k) {
    if (!a.neg) return S(shr(a.m, k));
    // -ceil(|a| / 2^k)
    U q = shr(a.m, k);
    if (!a.m.low_zero(k)) q = add(q, U(1));
    return S(q, true);
}
// Python round(Fraction(a, 2^k)): nearest, ties to even
HRBH_HD S sround_shr(const S& a, int k) {
    if (k <= 0) return sshl(a, -k);
    S fl = sfloor_shr(a, k);
    // rem = a - fl * 2^k in [0, 2^k)
    S rem = ssub(a, sshl(fl, k));
    U half = pow2(k - 1);
    int c = cmp(rem.m, half);
    if (c > 0 || (c == 0 && fl.m.bit(0))) return sadd(fl, S(U(1)));
    return fl;
}

// ---------------------------------------------------------------- dyadic

// value m * 2^e (exact)
struct D {
    S m;
    int e = 0;
    HRBH_HD D() {}
    HRBH_HD D(const S& mm, int ee) : m(mm), e(ee) {}
};

HRBH_HD D dadd(const D& a, const D& b) {
    if (a.m.zero()) return b;
    if (b.m.zero()) return a;
    if (a.e <= b.e) return D(sadd(a.m, sshl(b.m, b.e - a.e)), a.e);
    return D(sadd(sshl(a.m, a.e - b.e), b.m), b.e);
}
HRBH_HD D dsub(const D& a, const D& b) { return dadd(a, D(neg(b.m), b.e)); }
HRBH_HD D dmul(const D& a, const D& b) { return D(smul(a.m, b.m), a.e + b.e); }
HRBH_HD D dabs(const D& a) { return D(S(a.m.m), a.e); }
HRBH_HD D dmul_u(const D& a, const U& k) { return D(S(mul(a.m.m, k), a.m.neg), a.e); }
// integer value * 2^Z, exactly (requires e + Z >= 0; else sets overflow)
HRBH_HD S dscaled(const D& a, int Z) {
    if (a.m.zero()) return S();
    if (a.e + Z < 0) {
        overflow_flag() = true;
        return S();
    }
    return sshl(a.m, a.e + Z);
}

// x^k for small k
HRBH_HD U upow(const U& x, int k) {
    U r(1);
    for (int i = 0; i < k; i++) r = mul(r, x);
    return r;
}

HRBH_HD uint64_t isqrt_u64(uint64_t v) {
    uint64_t r = 0;
    while ((r + 1) * (r + 1) <= v) r++;
    return r;
}

}  // namespace hrbh
