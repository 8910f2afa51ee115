/*
 * gb.h -- C ABI of libgb, the B200 (sm_100a) segmented double-sieve Goldbach
 * verifier.  For every even n in a range it finds the minimal prime p with
 * n - p prime (section 2.1, lines 37-39: "scans primes p from 2 to
 * n/2 and checks whether q = n - p is prime"), using the paper's inverted
 * loop (section 2.3.1: "iterate over candidate primes p and
 * mark all even n for which q = n - p is prime") in the bitwise bulk-marking
 * form the paper names as future work (section 4.3).
 *
 * Conventions for every entry point:
 *   - Every call returns gb_status (GB_OK = 0); nothing throws across the ABI.
 *   - Device pointers (d_*) are caller-owned device memory on the ctx's device;
 *     host pointers (h_*) are caller-owned host memory.  libgb never allocates
 *     device memory: all of it lives in the caller's workspace.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     All device work is enqueued asynchronously on it, except where a function
 *     says it synchronizes.  Use one gb_ctx per stream.
 *   - Integers: n, q and window offsets are uint64_t; primes are uint32_t.
 *
 * Bit layouts (section 2.2, lines 46-51, "Dense prime bitset"):
 *   odd q >= 3  <->  bit index o(q) = (q - 3)/2 ; 64-bit word o/64, bit o%64.
 *   even n >= 4 <->  bit index e(n) = (n - 4)/2 (same word split); with this
 *   choice q = n - p for odd p = 2k + 1 has o(q) = e(n) - k.
 */
#ifndef GB_H
#define GB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GB_OK = 0,
    GB_EINVAL = 1,      /* bad argument: ordering, bounds, NULL / misaligned pointer */
    GB_ERANGE = 2,      /* range needs base primes beyond the ctx's hi_max (SPEC.md:71:
                           insufficient base primes is a hard error, never silent) */
    GB_EWORKSPACE = 3,  /* workspace smaller than gb_ctx_workspace_bytes() */
    GB_ECUDA = 4,       /* a CUDA runtime call or kernel launch failed */
    GB_EINTERNAL = 5
} gb_status;

typedef struct gb_ctx gb_ctx;   /* opaque; host object owned by libgb */

/* ---------------------------------------------------------------------------
 * Result vector (int64 words, device memory, GB_RESULT_WORDS long).
 * Fields are additive over disjoint ranges and ranks (SUM), except
 * FIRST_UNRESOLVED_N (MIN) and MAX_KEY (MAX) -- the reduction rules the
 * multi-GPU layer applies with NCCL ("--gpus distributes work").
 * ------------------------------------------------------------------------- */
#define GB_RESULT_VERSION 0x4742000000000003LL
#define GB_R_VERSION              0   /* GB_RESULT_VERSION                           */
#define GB_R_EVENS                1   /* SUM: even n in the verified ranges          */
#define GB_R_VERIFIED             2   /* SUM: n with a partition found               */
#define GB_R_FASTPATH_UNRESOLVED  3   /* SUM: n sent to the exhaustive fallback
                                         ("Phase 2")          */
#define GB_R_UNRESOLVED           4   /* SUM: n with no partition p <= n/2 (a
                                         counterexample) -- must be 0                */
#define GB_R_SUM_PMIN             5   /* SUM: sum of p_min                           */
/* words 6, 7, 10, 12..15: reserved (0).  No checksum is accumulated on the hot
   path: the exact sum of n * p_min, the position-sensitive check, is taken from the
   per-n dump (d_pmin_dump of gb_verify_range) by the tests. */
#define GB_R_FIRST_UNRESOLVED_N   8   /* MIN: smallest unresolved n, INT64_MAX if none */
#define GB_R_MAX_KEY              9   /* MAX: (min(p_min, 2^14-1) << 49) |
                                         (2^49-1 - (n-origin)/2): largest p_min, ties
                                         to the smallest n (exact while p_min < 2^14;
                                         every p_min below 4e18 is <= 9781)          */
#define GB_R_MAX_PMIN_RAW        11   /* MAX: largest p_min (exact even when the
                                         MAX_KEY field saturates at 2^14-1)         */
#define GB_R_HIST                16   /* SUM: hist[0..GB_NBINS)                       */
#define GB_NBINS               6544   /* hist[0] = unresolved; hist[i] = #n with p_min
                                         = i-th prime (p_1 = 2, p_2 = 3, ...,
                                         p_6542 = 65521); hist[6543] = p_min > 65521 */
#define GB_RESULT_WORDS (GB_R_HIST + GB_NBINS)
#define GB_KEY_SHIFT 49
#define GB_KEY_PMAX 16383              /* 2^14 - 1: p field of MAX_KEY (saturating) */

/* Largest p_max accepted (the fast-path prime bound, PAPER.md:173 P_SMALL = 1e6). */
#define GB_PMAX_LIMIT 1048576u
/* Largest hi accepted: 2^62 (4.61e18, above BASELINE.json's 4e18 window).  Every n
 * stays below 2^63, so GB_R_FIRST_UNRESOLVED_N (an int64 MIN) and the int64 n
 * fields of the result are exact, and 6m + 5, p*k, halos and carries cannot wrap. */
#define GB_HI_LIMIT 4611686018427387904ull   /* 2^62 */

/* Bytes of device workspace a ctx needs for ranges with hi <= hi_max and fast
 * path bound p_max (base-prime bitset + list + per-prime constants + scratch).
 * Returns 0 if the arguments are invalid. */
size_t gb_ctx_workspace_bytes(uint64_t hi_max, uint32_t p_max);

/* Create a context on `device` and run K-BASE: the resident small-prime table
 * (subsystem (b); "permanently resident small-primes bitset")
 * of all primes <= R = max(isqrt(hi_max - 1), p_max), as an odd-only bitset
 * plus an ascending u32 list, built on the GPU inside d_workspace.
 *   origin  : even n origin for GB_R_MAX_KEY; every verified n must satisfy
 *             origin <= n and (n - origin)/2 < 2^49 (one result spans 1.1e15).
 *   hi_max  : exclusive upper bound of every later range.
 *   p_max   : largest fast-path bound later calls may use (3..GB_PMAX_LIMIT).
 * Synchronizes `stream`.  On error *out is NULL. */
gb_status gb_ctx_create(gb_ctx **out, int device, uint64_t origin, uint64_t hi_max,
                        uint32_t p_max, void *d_workspace, size_t ws_bytes, void *stream);

/* Free the host object only; the workspace belongs to the caller. */
void gb_ctx_destroy(gb_ctx *ctx);

/* Number of odd primes in the resident table and its bound R (host values). */
gb_status gb_ctx_info(const gb_ctx *ctx, uint64_t *n_base_primes, uint64_t *R);

/* Device pointers to the resident table: odd-only bitset of [3, R] in the
 * paper's layout (bit o(q)) and the ascending u32 list of odd primes <= R. */
gb_status gb_ctx_tables(const gb_ctx *ctx, const uint64_t **d_bits, const uint32_t **d_primes);

/* K-SIEVE alone (subsystem (a); "segmented Sieve of
 * Eratosthenes to determine the primality of all odd integers in that
 * segment"): writes n_words 64-bit words of the global odd bitset,
 *   bit b of d_words[i]  <->  odd q = 3 + 2*(64*(word_lo + i) + b), 1 = prime.
 * Needs isqrt(largest q) <= R, else GB_ERANGE.  d_words 8-byte aligned.
 * Implementation: the verify kernel's shared-memory wheel sieve (persistent CTAs
 * with carried offsets, K-LARGE mask for primes > 2^21) re-interleaved into this
 * layout.  Uses the ctx's carry rows: do not overlap with another call on the
 * same ctx. */
gb_status gb_sieve_segment(gb_ctx *ctx, uint64_t word_lo, uint64_t n_words,
                           uint64_t *d_words, void *stream);

/* Set d_result (GB_RESULT_WORDS int64) to its initial state on the stream:
 * version word, counters 0, FIRST_UNRESOLVED_N = INT64_MAX, MAX_KEY = 0.  Runs
 * on the device that owns d_result. */
gb_status gb_result_init(int64_t *d_result, void *stream);

/* After a rank's last gb_verify_range, before the cross-rank reduction: a hook for
 * fields that need a final pass.  No field of this result version does (every SUM
 * field stays far below 2^63 on any range the library accepts), so it only checks
 * its arguments and launches nothing. */
gb_status gb_result_finalize(int64_t *d_result, void *stream);

/* Verify every even n with lo <= n < hi (half-open; the paper's "n in [4, N]",
 * PAPER.md:39, is lo = 4, hi = N + 1).  Fast path: odd primes p <= p_max
 * (subsystem (c)); n left unresolved go to the exhaustive on-GPU fallback
 * (subsystem (d); "tests all odd p from 3 to n/2 ... with no
 * upper bound"), which resumes at the first prime > p_max.
 * ACCUMULATES into d_result (initialised once by gb_result_init), so disjoint
 * calls compose.  d_pmin_dump (nullable): one u32 per even n in [lo_e, hi),
 * lo_e = max(4, lo rounded up to even), index (n - lo_e)/2, value p_min, 0 =
 * unresolved.  Launches one kernel (zero for an empty range); when the range
 * needs sieving primes above 2^21 (hi > 4.4e12, e.g. the 4e18 window) it runs in
 * chunks of whole tiles, each a K-LARGE mask fill + marking launch and a verify
 * launch.
 * Errors: GB_EINVAL (p_max < 3 or > the ctx's p_max, hi > GB_HI_LIMIT,
 * n < origin, (hi - origin)/2 >= 2^49, misaligned pointers), GB_ERANGE
 * (hi > ctx hi_max). */
gb_status gb_verify_range(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                          int64_t *d_result, uint32_t *d_pmin_dump, void *stream);

/* Test hook: as gb_verify_range, but the fallback scans p only up to
 * fallback_p_cap, so n with p_min > cap are reported unresolved (makes the
 * counterexample path reproducible; UINT64_MAX = unbounded). */
gb_status gb_verify_range_ex(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                             uint64_t fallback_p_cap, int64_t *d_result,
                             uint32_t *d_pmin_dump, void *stream);

/* End-to-end convenience with HOST buffers: result_init + verify + finalize on
 * the ctx's internal device scratch, then copies the GB_RESULT_WORDS result to
 * h_result (and the dump, if h_pmin_dump != NULL, through the same scratch in
 * chunks).  Synchronizes `stream`. */
gb_status gb_verify_range_host(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                               int64_t *h_result, uint32_t *h_pmin_dump, void *stream);

/* NEXT-1 comparison mode: the paper's own gpu3 Phase-1
 * kernel (section 2.3.2, Fig. 1) -- one thread per even n scans
 * odd primes p <= p_max ascending and tests q = n - p by the three-way oracle:
 * q <= R -> the resident small-prime bitset; q in the current
 * segment -> that segment's odd bitset, sieved by gb_sieve_segment into ctx
 * scratch (segments of 2^28 evens); otherwise deterministic MR64
 * (PAPER.md:89).  Unresolved n go to the same exhaustive fallback.  Same
 * arguments, result semantics and errors as gb_verify_range, and results identical
 * to it field by field; per segment one sieve launch (plus K-LARGE mask launches
 * above 2^21) and one per-n launch.  Not the product path: it
 * exists to measure per-n lookups against the inverted bulk marking on one box. */
gb_status gb_verify_range_pern(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                               int64_t *d_result, uint32_t *d_pmin_dump, void *stream);

/* NEXT-2 comparison mode: the paper's gpu2 (PAPER.md:41-59,
 * section 2.2, "Global GPU-Resident Bitset") -- the odd bitset of the WHOLE range is
 * resident in HBM (d_bits: words [0, n_words) of the global layout, caller-owned,
 * e.g. written by gb_sieve_segment; 62.5 GB at N = 1e12 fits a B200), and one thread
 * per even n scans odd p <= p_max ascending with a direct bitset lookup of q.
 * Requires 3 + 128 * n_words >= hi (GB_EINVAL otherwise).  Same result semantics
 * as gb_verify_range; one launch. */
gb_status gb_verify_range_resident(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                                   const uint64_t *d_bits, uint64_t n_words, int64_t *d_result,
                                   uint32_t *d_pmin_dump, void *stream);

/* NEXT-3: single_check (section 2.4) for ONE even n, 4 <= n <
 * 2^64: writes to *d_out (device u64) the minimal prime p <= p_limit with n - p
 * prime (p tested by the resident bitset or MR64; q = n - p likewise), 0 if none.
 * The paper's tool returns some valid partition; this one returns the minimal one.
 * GB_EINVAL for odd n, n < 4, misaligned d_out. */
gb_status gb_single_check(gb_ctx *ctx, uint64_t n, uint64_t p_limit, uint64_t *d_out, void *stream);

/* NEXT-4: Goldbach partition counts (section 4.5 "large-scale
 * computation of Goldbach partition counts c(n)"; c(n) also at PAPER.md:404).  The
 * paper does not define c(n); read as the Goldbach-comet count (R13)
 *      c(n) = #{ p prime : p <= n/2 and n - p prime },   c(4) = 1 (2 + 2).
 * For every even n in [lo_e, hi), lo_e = max(4, lo rounded up to even):
 * d_counts[(n - lo_e)/2] = c(n) (u64, overwritten).  d_bits: words [0, n_words) of
 * the global odd bitset in the paper's layout (e.g. from gb_sieve_segment), which
 * must hold every odd q < hi (3 + 128 * n_words >= hi), caller-owned.  Work is
 * O(n) bit operations per n (popcount-AND of the bitset against its reversed
 * shifts), so hi is limited to GB_COUNTS_HI_LIMIT.  One init launch and one
 * counting launch.  Errors: GB_EINVAL (bounds, NULL / misaligned pointers, bitset
 * too short). */
#define GB_COUNTS_HI_LIMIT 1099511627776ull   /* 2^40 */
gb_status gb_partition_counts(gb_ctx *ctx, uint64_t lo, uint64_t hi, const uint64_t *d_bits, uint64_t n_words,
                              uint64_t *d_counts, void *stream);

/* Deterministic 64-bit Miller-Rabin (12 prime bases 2..37; PAPER.md:89,
 * SPEC.md:128) as used by the fallback: d_out[i] = 1 iff d_x[i] is prime. */
gb_status gb_is_prime_u64(const uint64_t *d_x, uint8_t *d_out, uint64_t n, void *stream);

/* Number of kernels libgb has launched in this process (instrumentation). */
uint64_t gb_launch_count(void);

const char *gb_status_string(gb_status s);

#ifdef __cplusplus
}
#endif
#endif /* GB_H */
