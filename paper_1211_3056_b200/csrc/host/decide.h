// decide.h -- decide_hr for exp (evalf.py:286-327 with the pipeline's start
// precision 2 (p + eps_bits) + 16, pipeline.py:446), on the exact interval
// exp of mpexp.h.  Host (libhrbhost.so, hrbh_confirm) and device
// (libhrb200.so, hrb_confirm_exp) compile this same source.
#pragma once

#include "bign.h"
#include "mpexp.h"

namespace hrbh {

// evalf._dist_range (reference evalf.py:209-232 _dist_interval)
HRBH_HD void dist_range(const U& off, const U& width, const U& grid, U* dlo, U* dhi) {
    U end = add(off, width);
    U half = shr(grid, 1);
    if (cmp(end, grid) >= 0) {
        *dlo = U();
        if (cmp(off, half) <= 0) {
            *dhi = half;
        } else {
            U a = sub(grid, off);
            U eg = sub(end, grid);
            U b = cmp(eg, half) < 0 ? eg : half;
            *dhi = cmp(a, b) > 0 ? a : b;
        }
        return;
    }
    U go = sub(grid, off), ge = sub(grid, end);
    U d0 = cmp(off, go) < 0 ? off : go;
    U d1 = cmp(end, ge) < 0 ? end : ge;
    *dlo = cmp(d0, d1) < 0 ? d0 : d1;
    if (cmp(off, half) <= 0 && cmp(half, end) <= 0)
        *dhi = half;
    else
        *dhi = cmp(d0, d1) > 0 ? d0 : d1;
}

// bit length of the reduced denominator of m 2^e (m > 0)
HRBH_HD int den_bits(const U& m, int e) {
    int ee = e + m.tz();
    return ee >= 0 ? 1 : -ee + 1;
}

// 0 = not HR, 1 = HR (dist set), -1 = fallback
HRBH_HD int decide_exp(int precision, int eps_bits, int binade, uint64_t index, uint64_t* dist) {
    overflow_flag() = false;
    const int p = precision;
    const int xe = binade + 1 - p;
    const uint64_t M = (1ull << (p - 1)) + index;
    int prec = 2 * (p + eps_bits) + 16;
    while (prec <= 4096) {
        Enc en;
        if (!exp_enclose(M, xe, prec, &en)) return -1;
        // lo == hi (exactly representable at this precision): rare; Python
        if (cmp(en.lm, en.hm) == 0) return -1;
        const int sc = imax(imax(den_bits(en.lm, en.le), den_bits(en.hm, en.he)), prec) + 4;
        // nlo = floor(lo 2^sc), nhi = ceil(hi 2^sc)
        U nlo = en.le + sc >= 0 ? shl(en.lm, en.le + sc) : shr(en.lm, -(en.le + sc));
        U nhi;
        if (en.he + sc >= 0) {
            nhi = shl(en.hm, en.he + sc);
        } else {
            int k = -(en.he + sc);
            nhi = shr(en.hm, k);
            if (!en.hm.low_zero(k)) nhi = add(nhi, U(1));
        }
        if (nlo.bitlen() == nhi.bitlen()) {
            const int e = nlo.bitlen() - sc;
            const int gbits = sc + e - p;
            if (gbits > 0) {
                U grid = pow2(gbits);
                U dlo, dhi;
                dist_range(low_bits(nlo, gbits), sub(nhi, nlo), grid, &dlo, &dhi);
                // compare against eps = 2^-eps_bits in grid units
                auto lt_eps = [&](const U& d) -> bool {
                    if (gbits >= eps_bits) return cmp(d, pow2(gbits - eps_bits)) < 0;
                    return d.zero();
                };
                if (overflow_flag()) return -1;
                if (lt_eps(dhi)) {
                    U r = gbits >= 64 ? shr(dlo, gbits - 64) : shl(dlo, 64 - gbits);
                    *dist = r.low64();
                    return 1;
                }
                if (!lt_eps(dlo)) return 0;
            }
        }
        prec *= 2;
    }
    return -1;  // undecided at the cap: the Python path raises UndecidedError
}


// cap of the precision loop; the device stops earlier (confirm.cuh)
}  // namespace hrbh
