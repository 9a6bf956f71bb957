/*
 * hrb200.h -- C-ABI of the B200-native hard-to-round (HR) case search.
 *
 * This is the drop-in boundary between the host (Python `hardround`-shaped
 * package, polynomial generation, error bounds, confirmation) and the
 * sm_100a kernels.  Every function is extern "C", takes plain pointers and
 * sizes, returns an int status and never throws.  Unless stated otherwise
 * pointers are DEVICE pointers owned by the caller and work is enqueued on
 * the caller's cudaStream_t (passed as void*; NULL = legacy default stream).
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/hardround/<file>:<line>).
 */
#ifndef HRB200_H
#define HRB200_H

#include <stdint.h>

#include "hrb_host.h" /* hrbh_cfg (hrb_pack_blocks) */

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes --------------------------------------------------- */
#define HRB_OK 0           /* success                                        */
#define HRB_ERR_RUNTIME 1  /* CUDA error (cli.py:268 exit 1 analogue)         */
#define HRB_ERR_CONFIG 2   /* invalid argument (ValueError, cli.py:264-266)  */
#define HRB_ERR_OVERFLOW 4 /* reserved: limb overflow (MPOverflowError)      */
#define HRB_ERR_CAPACITY 8 /* an output buffer was too small; counts are the
                              true totals so the caller can re-run larger   */

/* ---- enums (values fixed: they cross the ABI) ----------------------- */
/* lowerbound.py:41-45 Algorithm */
#define HRB_ALGO_LEFEVRE 0
#define HRB_ALGO_LEFEVRE_SWAP 1
#define HRB_ALGO_REGULAR 2
#define HRB_ALGO_REGULAR_UNROLLED 3
/* lowerbound.py:80-85 _mode_code (fixedpoint.py:26-33 DivisionMode) */
#define HRB_MODE_SUBTRACTIVE 0
#define HRB_MODE_HYBRID 1
#define HRB_MODE_HARDWARE 2

int hrb_version(void);                  /* 100*major + minor                 */
const char* hrb_last_error(void);       /* thread-local message of last error */
int hrb_device_info(int device, char* buf, int buflen); /* name, SMs, clocks  */

/*
 * Batched lower-bound searches: exactly the SEARCHES registry
 * (lowerbound.py:321-381; raw cores lowerbound.py:88-308) for n independent
 * problems {b - a*x mod 1 : x < count} at word width W in {32, 64}.
 * Inputs a, b, eps are the UFrac raws (< 2^W, eps < 2^(W-1)), count >= 1.
 * Outputs: ok (Verdict.SUCCESS = 1), d raw, iterations (SearchOutcome
 * .iterations, per-mode for the classic family), points_placed as
 * points_lo + 2^64 * points_hi.  iterations may be NULL.
 */
int hrb_search_batch(int algo, int mode, int word_bits, int64_t n, const uint64_t* a,
                     const uint64_t* b, const uint64_t* eps, const uint64_t* count, uint8_t* ok,
                     uint64_t* d, uint64_t* iterations, uint64_t* points_lo, uint8_t* points_hi,
                     void* stream);

/*
 * Regular-family verdicts only (Verdict, d, iterations; no points_placed):
 * the throughput form the phases use (lockstep pairs, warp-uniform control
 * flow), for callers that need what _run_search's callers read
 * (pipeline.py:200-201, 228: `.success`).  algo must be HRB_ALGO_REGULAR or
 * HRB_ALGO_REGULAR_UNROLLED (lowerbound.py:347-373); results equal
 * hrb_search_batch's.  iterations may be NULL.
 */
int hrb_search_verdicts(int algo, int word_bits, int64_t n, const uint64_t* a, const uint64_t* b, const uint64_t* eps,
                        const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* iterations, void* stream);

/*
 * hrb_search_batch plus the branch-decision stream of every problem: the
 * `trace` list the reference cores append to (lowerbound.py:109-110,
 * 126-127, 189-190, 246-259, 299-304), which its warp simulator consumes
 * (divergence.py:243-248).  Decision k of problem i is bit (k mod 64) of
 * trace_words[i * words_per_problem + k / 64]; trace_len[i] is the full
 * decision count (decisions beyond 64 * words_per_problem are counted, not
 * stored, so a caller can size a second call exactly).
 */
int hrb_search_trace(int algo, int mode, int word_bits, int64_t n, const uint64_t* a, const uint64_t* b,
                     const uint64_t* eps, const uint64_t* count, uint8_t* ok, uint64_t* d, uint64_t* iterations,
                     uint64_t* points_lo, uint8_t* points_hi, uint64_t* trace_words, int64_t words_per_problem,
                     uint32_t* trace_len, void* stream);

/*
 * A slice: S consecutive super-domains of one output-exponent piece run,
 * packed by the host after taylor_approx + hierarchical_split
 * (polygen.py:113-131, 193-252).  All arrays are device pointers, SoA.
 *
 *   coef    uint32[6][coef_limbs][S]  two's complement little-endian limbs of
 *           the binomial-basis coefficients of r_0 (3), r_1 (2), r_2 (1) in
 *           the packet variable i (hierarchical_split output), in the order
 *           r0.c0 r0.c1 r0.c2 r1.c0 r1.c1 r2.c0 (unused ones zero for delta=1)
 *   G       uint64[2][S]   ceil(eps' * 2^F) (lo, hi), eps' = eps + eps_approx
 *   s2abs   uint64[2][S]   |r2.c0| saturated to 2^128-1 (delta=2), else 0
 *   n_dom   uint32[S]      domains in the super-domain (tau_t)
 *   dom_n   uint32[S]      domain size N_t
 *   last_n  uint32[S]      size of the last domain (ragged tail)
 *   dom_base uint64[S+1]   exclusive prefix sum of n_dom (slice-local ids)
 *   m0      uint64[S]      binade index of the super-domain's first argument
 *
 * Host guarantees (checked in the Python layer, pipeline.py:178-184 and
 * fpmodel.py:220-225 semantics): W <= F <= 128, 1 <= delta <= 2, and for
 * every count used eps'' < 1/4 and 2*pad < 2^(W-1).
 */
typedef struct hrb_slice {
    int64_t n_super;
    int64_t n_total;    /* sum of n_dom (host scalar: sizes device scratch)   */
    uint32_t max_dom_n; /* max of dom_n and last_n (host scalar)              */
    int32_t coef_limbs;
    int32_t frac_bits;
    int32_t word_bits;
    int32_t delta;
    const uint32_t* coef;
    const uint64_t* G;
    const uint64_t* s2abs;
    const uint32_t* n_dom;
    const uint32_t* dom_n;
    const uint32_t* last_n;
    const uint64_t* dom_base;
    const uint64_t* m0;
} hrb_slice;

/*
 * Tabulated differences (polygen.py:134-158, 255-280 domain_coefficient_sets):
 * per-domain coefficient sets (s0, s1, s2) = (r0(i), r1(i), r2(i)) for every
 * domain of the slice, walked with add-with-carry chains from per-packet
 * seeds.  out: uint32[3][coef_limbs][n_total] two's complement (exact while
 * the values fit coef_limbs limbs; the host checks the MPInt budget).
 */
int hrb_domain_coefficients(const hrb_slice* s, uint32_t* out, void* stream);

/*
 * Phase 1 (pipeline.py:213-231), fused: tabulated walk -> degree-1 Boolean
 * problem (pipeline.py:141-175) -> search -> warp-aggregated compaction of
 * failing slice-local domain ids.  fail_ids receives the ids in ascending
 * order (sorted on the device), *fail_count (device u64) the true count.
 * iter_sum (device u64, may be NULL) accumulates SearchOutcome.iterations.
 */
int hrb_phase1(const hrb_slice* s, int algo, int mode, uint64_t* fail_ids, uint64_t* fail_count,
               uint64_t cap, uint64_t* iter_sum, void* stream);

/*
 * Phase 2 (pipeline.py:234-257): for each failing domain, split `split`
 * ways (2..64), Taylor-shift to each subdomain start, re-test.  Input: the
 * n_fail ids of phase 1 (device count pointer).  Output keys
 * (slice-local id << 8 | sub index), ascending.
 */
int hrb_phase2(const hrb_slice* s, int algo, int mode, int split, const uint64_t* fail_ids,
               const uint64_t* fail_count, uint64_t fail_cap, uint64_t* sub_keys, uint64_t* sub_count,
               uint64_t cap, void* stream);

/*
 * Phase 3 (pipeline.py:260-293): exact second-order walk of each surviving
 * subdomain mod 2^F; arguments inside the eps' window become candidates:
 * binade argument index, distance floored to 2^-64, slice-local domain id,
 * ascending by argument.
 */
int hrb_phase3(const hrb_slice* s, int split, const uint64_t* sub_keys, const uint64_t* sub_count,
               uint64_t sub_cap, uint64_t* cand_index, uint64_t* cand_dist, uint64_t* cand_dom,
               uint64_t* cand_count, uint64_t cap, void* stream);

/*
 * The three phases back to back on the device (the north-star hot path for
 * one slice); no host synchronisation between phases.  A call repeating the
 * previous call's arguments exactly (same slice, outputs, algorithm) replays
 * the captured launch sequence as one CUDA graph (HRB_NO_GRAPH=1 disables).  counts (device
 * uint64[4]): phase-1 fails, phase-2 survivors, phase-3 candidates,
 * phase-1 iteration sum.  Capacities: fail_cap, sub_cap, cand_cap.
 */
typedef struct hrb_run_out {
    uint64_t* fail_ids;
    uint64_t fail_cap;
    uint64_t* sub_keys;
    uint64_t sub_cap;
    uint64_t* cand_index;
    uint64_t* cand_dist;
    uint64_t* cand_dom;
    uint64_t cand_cap;
    uint64_t* counts;
} hrb_run_out;

int hrb_run_slice(const hrb_slice* s, int algo, int mode, int split, const hrb_run_out* out,
                  void* stream);

/*
 * End-to-end variant with HOST buffers (pageable or pinned): copies the
 * slice to the device, runs hrb_run_slice, copies counts and candidates
 * back, synchronises.  Host outputs: counts[6] (hrb_run_slice's four, then
 * the arguments covered by phase 2 and by phase 3 -- PhaseRow
 * .arguments_covered, pipeline.py:440-451), fail_ids (<= fail_cap; NULL or
 * fail_cap 0 skips that copy), cand_* (<= cand_cap).  Device buffers are cached per device and grown on
 * demand (a too-small internal subdomain buffer triggers one re-run).
 * For the regular family the upload is streamed behind the search (phase 1
 * waits per run of super-domains on a device counter) and the failing ids
 * are copied back while phases 2-3 run.  Calls on the same device are
 * serialised (the cached buffers and streams are per device).
 * device_ms (may be NULL) receives the time between the call's first and
 * last event on its compute stream (uploads overlapped, final copies
 * included).
 */
int hrb_run_slice_host(const hrb_slice* host_slice, int algo, int mode, int split,
                       uint64_t* counts, uint64_t* fail_ids, uint64_t fail_cap,
                       uint64_t* cand_index, uint64_t* cand_dist, uint64_t* cand_dom,
                       uint64_t cand_cap, float* device_ms);

/*
 * hrb_run_slice_host for a slice already resident in device memory (every
 * column pointer a device pointer, e.g. hrb_pack_blocks' outputs plus the
 * uploaded size columns): nothing is uploaded; the call's compute stream
 * waits for the work already enqueued on `stream` (the generation), runs
 * the three phases and copies counts[6] and the candidates to the HOST
 * buffers, synchronised.  No failing-id list.  run_range's path when the
 * generation ran on the device (funnel.execute_batch_host).
 */
int hrb_run_slice_resident(const hrb_slice* device_slice, int algo, int mode, int split,
                           uint64_t* counts, uint64_t* cand_index, uint64_t* cand_dist,
                           uint64_t* cand_dom, uint64_t cand_cap, float* device_ms, void* stream);

/*
 * High-degree slices (delta_R = degree in 3..8): one Taylor polynomial per
 * large super-domain (up to 2^25 domains), the paper's large super-domain
 * generation.  The reference rejects delta >= 3
 * (polygen.py:81-82): this is an extension, specified by oracle/wide.py
 * and produced by hrbh_wide_blocks (include/hrb_host.h).  F = 32 frac_limbs
 * with frac_limbs = max(4, degree); residues are frac_limbs 32-bit limbs.
 *
 *   coef  uint32[(D+1)(D+2)/2][NL][S]  q_{j,l} = rho_{j,l} 2^F mod 2^F,
 *         r_j(i) = sum_l q_{j,l} C(i, l) (binomial basis in the domain
 *         index i), columns j-major (r_0's D+1, then r_1's D, ...)
 *   padg  uint64[2][S]  ceil((ceil(eps' 2^F) + T3) / 2^(F-128)): eps' and
 *         the degree >= 3 truncation bound, in 2^-128 units
 *   s2b   uint64[2][S]  ceil(S2 / 2^(F-128)), S2 >= max_i |r_2(i)| 2^F
 *   win   uint32[NL][S] ceil(eps' 2^F) + 1, the phase-3 window
 *   geometry as hrb_slice
 * Phases 1-2 test with pad = ceil((padg + s2b (n-1)^2) / 2^64) + n + 1.
 */
typedef struct hrb_wslice {
    int64_t n_super;
    int64_t n_total;
    uint32_t max_dom_n; /* <= 2^16 */
    int32_t degree;
    int32_t frac_limbs;
    int32_t word_bits; /* 64 */
    const uint32_t* coef;
    const uint64_t* padg;
    const uint64_t* s2b;
    const uint32_t* win;
    const uint32_t* n_dom;
    const uint32_t* dom_n;
    const uint32_t* last_n;
    const uint64_t* dom_base;
    const uint64_t* m0;
} hrb_wslice;

/*
 * Phases 1-3 of a high-degree slice on the device (hrb_run_slice's outputs
 * and ordering): the tile columns of the multi-limb difference tables, the
 * fused packet walk + Boolean test + regular search, phase 2 with the
 * Toeplitz shift to the subdomain starts (split 2..16), the exact
 * degree-delta_R phase-3 walk.  algo: HRB_ALGO_REGULAR or _UNROLLED.
 */
int hrb_wrun_slice(const hrb_wslice* s, int algo, int split, const hrb_run_out* out, void* stream);

/* The same with HOST buffers in and out: counts[6] as hrb_run_slice_host. */
int hrb_wrun_slice_host(const hrb_wslice* host_slice, int algo, int split, uint64_t* counts, uint64_t* cand_index,
                        uint64_t* cand_dist, uint64_t* cand_dom, uint64_t cand_cap, float* device_ms);

/*
 * Tabulated values of a high-degree slice: every domain's (s_0..s_D) mod 2^F
 * through the multi-limb packet walk.  out: uint32[D+1][NL][n_total].
 */
int hrb_wdomain_coefficients(const hrb_wslice* s, uint32_t* out, void* stream);

/*
 * Rigorous confirmation of candidates on the device: decide_hr for exp
 * (evalf.py:286-327) at the pipeline's start precision 2 (p + eps_bits) + 16
 * (pipeline.py:446-461), for n candidates given by their binade argument
 * index (binade <= 0).  is_hr[i]; for HR cases dist_raw[i] =
 * floor(distance_lo 2^64) (UFrac.from_fraction of HrDecision.distance_lo);
 * status[i] = 1 when the device did not settle the candidate (the host's
 * hrbh_confirm / decide_hr does).  The device runs the same exact
 * restatement of mpmath's interval exp as libhrbhost.so (csrc/host/).
 * All pointers are device pointers.
 */
int hrb_confirm_exp(int precision, int eps_bits, int binade, int64_t n, const uint64_t* index, uint8_t* is_hr,
                    uint64_t* dist_raw, uint8_t* status, void* stream);

/*
 * Native generation on the device: hrbh_pack_blocks (include/hrb_host.h --
 * Taylor model, split, checks and packed columns of S super-domains, the
 * reference's polygen.py:193-280 and slices.check_super) with one device
 * thread per super-domain running the same source (csrc/host/polygen.h),
 * bit-identical to the host library.  Outputs as hrbh_pack_blocks: coef
 * uint32[6][limbs + 1][S], G / s2abs uint64[2][S], status[t] (HRBH_OK or
 * HRBH_FALLBACK: the exact Python path takes the item), shift_ok[t].
 * Configuration domain: the host library's, with limbs <= 12 and
 * frac_bits + guard <= 224 (the device's fixed 1024-bit capacity);
 * HRB_ERR_CONFIG otherwise.  All array pointers are device pointers.  The
 * kernel keeps ~15 KB of big integers per thread in local memory, which the
 * driver reserves for every resident thread (~4.2 GB on a B200) from the
 * first call on.
 */
int hrb_pack_blocks(const hrbh_cfg* cfg, int64_t S, const uint64_t* index_start, const uint64_t* count,
                    const uint32_t* n_p, const uint32_t* tau, const int32_t* e_out, uint32_t* coef, uint64_t* G,
                    uint64_t* s2abs, uint8_t* status, uint8_t* shift_ok, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HRB200_H */
