/*
 * hrb_host.h -- C-ABI of the native host half of the hybrid CPU-GPU split:
 * Taylor models of the super-domains, their hierarchical split, the exact
 * checks the reference performs on them, packing into the device slice
 * layout of hrb200.h, and the rigorous confirmation of phase-3 candidates.
 *
 * It replaces, for exp on binades <= 0 with delta <= 2 (the north-star
 * workload), the reference's host Python on that path:
 *   taylor_approx           polygen.py:193-252
 *   hierarchical_split      polygen.py:113-131
 *   MPInt limb budget       fixedpoint.py:136-137 (checked, never wrapped)
 *   _boolean_problem pad /
 *   ErrorBudget checks      pipeline.py:141-184, fpmodel.py:220-225
 *   decide_hr               evalf.py:286-327 (pipeline.py:447-461)
 * with results bit-identical to the reference's: the interval exp it reads
 * (mpmath 1.3.0 iv.exp) is restated exactly (csrc/host/mpexp.h).  Items it
 * does not cover -- or where the reference would raise -- come back with
 * status HRBH_FALLBACK, and the Python layer runs its exact path on them
 * (which raises the reference's exception where the reference does).
 *
 * All pointers are HOST pointers; nothing here touches a GPU.
 */
#ifndef HRB_HOST_H
#define HRB_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HRBH_OK 0
#define HRBH_FALLBACK 1 /* per item: not covered here, use the exact Python path */

#define HRBH_FN_EXP 0

typedef struct hrbh_cfg {
    int32_t fn;        /* HRBH_FN_EXP                                        */
    int32_t precision; /* FpFormat.precision p                               */
    int32_t eps_bits;  /* FpFormat.eps_bits: eps = 2^-eps_bits               */
    int32_t binade;    /* arguments X in [2^binade, 2^(binade+1)), binade<=0 */
    int32_t frac_bits; /* PolyGenConfig.frac_bits F (<= 128 for the device)  */
    int32_t guard;     /* PolyGenConfig.guard                                */
    int32_t limbs;     /* PolyGenConfig.limbs L (MPInt budget 2^(32 L))      */
    int32_t delta;     /* PolyGenConfig.delta, 1 or 2                        */
    int32_t word_bits; /* PipelineConfig.word_bits W                         */
} hrbh_cfg;

int hrbh_version(void);

/*
 * One planned block per super-domain (slices.plan_blocks: index_start,
 * count, n_p, tau, e_out).  Outputs, SoA with S columns (include/hrb200.h
 * hrb_slice): coef uint32[6][L+1][S], G uint64[2][S], s2abs uint64[2][S];
 * status[t] HRBH_OK or HRBH_FALLBACK; shift_ok[t] = the phase-2 shift bound
 * of slices.check_super rules limb overflow out.  Columns of fallback items
 * are left untouched.  threads <= 0: all host threads (OpenMP).
 * Returns 0, or 2 for an invalid configuration.
 */
int hrbh_pack_blocks(const hrbh_cfg* cfg, int64_t S, const uint64_t* index_start, const uint64_t* count,
                     const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out, uint32_t* coef, uint64_t* G,
                     uint64_t* s2abs, uint8_t* status, uint8_t* shift_ok, int threads);

/*
 * decide_hr (evalf.py:286-327) with the reference pipeline's start
 * precision 2 (p + eps_bits) + 16 (pipeline.py:446) for n candidates given
 * by their binade argument index.  is_hr[i], and for HR cases dist_raw[i] =
 * floor(distance_lo * 2^64) (UFrac.from_fraction of HrDecision.distance_lo).
 */
int hrbh_confirm(const hrbh_cfg* cfg, int64_t n, const uint64_t* index, uint8_t* is_hr, uint64_t* dist_raw,
                 uint8_t* status, int threads);

/*
 * High-degree super-domains (delta_R = degree in 3..8, F = 32 frac_limbs;
 * the paper's large super-domain generation; the
 * reference rejects delta >= 3, polygen.py:81-82, so this is an extension
 * specified by oracle/wide.py).  Per block: the degree-delta_R Taylor
 * model, its hierarchical split r_j(i) = Delta^j P(i N) in the binomial
 * basis of the domain index, rounded once to 2^-F (the only rounding), the
 * rigorous eps' (Lagrange + enclosure + rounding terms), and the device
 * constants of include/hrb200.h hrb_wslice:
 *   coef  uint32[(D+1)(D+2)/2][NL][S]  q_{j,l} mod 2^F, j-major
 *   padg  uint64[2][S]  ceil((ceil(eps' 2^F) + T3) / 2^(F-128))
 *   s2b   uint64[2][S]  ceil(S2 / 2^(F-128))
 *   win   uint32[NL][S] ceil(eps' 2^F) + 1  (phase-3 window)
 * exp on binades <= 0, W = 64.  status[t] = HRBH_FALLBACK when the block is
 * out of range (budget eps'' >= 1/4, pad too wide, not covered).
 */
int hrbh_wide_blocks(const hrbh_cfg* cfg, int degree, int frac_limbs, int64_t S, const uint64_t* index_start,
                     const uint64_t* count, const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out,
                     uint32_t* coef, uint64_t* padg, uint64_t* s2b, uint32_t* win, uint8_t* status, int threads);

/*
 * The enclosure itself (for tests): exp(M 2^xe) at `prec` as
 * lo = lo_words * 2^lo_exp, hi = hi_words * 2^hi_exp (words little endian,
 * *nwords each, at most 16).  Returns HRBH_FALLBACK when not covered.
 */
int hrbh_exp_enclose(uint64_t M, int xe, int prec, uint64_t* lo_words, int32_t* lo_exp, uint64_t* hi_words,
                     int32_t* hi_exp, int32_t* nwords);

#ifdef __cplusplus
}
#endif

#endif /* HRB_HOST_H */
