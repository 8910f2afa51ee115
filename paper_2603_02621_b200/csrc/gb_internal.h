// gb_internal.h -- shared between the C-ABI layer (gb_api.cu) and the kernels
// (gb_kernels.cu).  Product code only; nothing here is visible to oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "gb.h"

namespace gb {

// ---- tiling constants (tuned for sm_100a: 148 SMs, 228 KB smem / SM) ----
constexpr int kThreads = 1024;             // threads per CTA, every kernel (768 / 896: slower)
constexpr int kTileWords = 21376;          // verify tile: 32-bit words per mod-6 class (the largest
                                           // multiple of 128 whose windows fit next to the queues and
                                           // the static shared memory; 20480: +0.3% at 1e12, +1.9% at 4e18)
constexpr int kMarkWarps = kThreads / 32;  // warps of a verify CTA (each sieves, then marks)
constexpr uint32_t kTileM = 32u * kTileWords;  // m-span of a tile (n = 6m + a): 655360 m per class
// verify kernel dynamic shared memory: the two class windows (halo + tile + slack
// words each, <= kVerifyWinSmemMax) + per-warp survivor queues (u32 U + u16 index)
constexpr uint32_t kVerifyWinSmemMax = 171 * 1024;   // + kQueueBytes + 31,840 B static <= 227 KB
constexpr uint32_t kWinSlackWords = 128;      // words past a window phase-1 lanes may read (U = 0)
constexpr uint32_t kQueueEntries = 128;       // per-warp survivor queue
constexpr size_t kQueueBytes = (size_t)kMarkWarps * kQueueEntries * 6;
constexpr size_t kVerifySmemMax = kVerifyWinSmemMax + kQueueBytes;
// sieve_out_kernel: the two class windows of one tile (+ one word) + slack
constexpr size_t kSieveOutSmemMax = 4ull * ((2 * (kTileWords + 1 + kWinSlackWords) + 3) & ~3ull);
constexpr int kSieveTileWords = 16384;     // 32-bit words per gb_sieve_segment CTA
constexpr int kHistSmem = 1024;            // histogram bins kept in shared memory
constexpr uint32_t kWarpPrimeMax = 8192;   // primes <= this: one warp per prime (4096: slower)
constexpr int kTinyPrimes = 10;            // 3..31 sieved by word patterns
constexpr uint64_t kDumpScratch = 1ull << 24;  // u32 entries of host-API dump scratch
constexpr int kScanBlockWords = 2048;      // u64 words per K-BASE compaction block
constexpr uint32_t kCarryPrimeMax = 1u << 21;  // verify CTAs carry sieve offsets of primes below
constexpr int kMaxBlocksPerSm = 4;         // sizing bound for per-CTA carry storage
// Ranges that need sieving primes above kCarryPrimeMax (hi > 2^42, e.g. the 4e18
// window) run in chunks of kLargeTilesPerSm verify tiles per SM; before each
// chunk K-LARGE marks the multiples of those primes into an L2-resident wheel mask.
constexpr int kLargeTilesPerSm = 3;

// Arguments of the window sieve (K-SIEVE) shared by every caller.
struct SievePrimes {
    const uint32_t *primes;   // odd primes ascending (3, 5, 7, ...)
    const uint64_t *magic;    // floor((2^64-1)/p) per prime
    const uint4 *pk;          // (p, kTileM mod p, rA, rB) per prime (see make_pk)
    uint32_t i_med;           // first index with p > 31 (word patterns below)
    uint32_t i_big;           // first index with p > kWarpPrimeMax
    uint32_t n_use;           // primes usable (p^2 beyond the window are skipped)
};

// K-LARGE: multiples of primes [i_begin, i_end) cleared in a wheel-class mask of
// nw words per class (class A at mask[0..nw), class B at mask[stride..stride+nw)),
// word i <-> m in [32(g0+i), 32(g0+i)+32); every other bit stays 1.
struct LargeArgs {
    const uint32_t *primes;
    const uint64_t *magic;
    uint32_t i_begin, i_end;
    int64_t g0;
    uint32_t nw;
    uint64_t stride;
    uint32_t *mask;
};

struct SegmentArgs {
    SievePrimes sp;
    uint64_t g_lo;            // first 32-bit word (o-space) of the output
    uint64_t n_words32;       // 32-bit words to produce
    uint64_t o_limit;         // bits with o >= o_limit are cleared (UINT64_MAX: none)
    uint32_t *out;            // n_words32 words
};

// The fused verify kernel works on the mod-6 wheel (gb_verify.cu): even n = 6m + a
// (classes a = 0, 2, 4) and odd q = 6m + 1 (class A) / 6m + 5 (class B).
struct VerifyArgs {
    SievePrimes sp;
    uint32_t n_cand;          // odd primes p <= p_max used by the fast path
    uint32_t halo;            // words per class below a tile: (max shift >> 5) + 1
    uint64_t m_lo[3], m_hi[3];  // class a = 0, 2, 4: valid m in [m_lo, m_hi)
    uint64_t u_first;         // first 32-bit word (u = m >> 5, same for all classes)
    uint64_t u_end;           // one past the last word
    uint64_t n_tiles;
    uint64_t lo_e;            // dump index = (n - lo_e) / 2
    uint64_t origin;          // MAX_KEY origin
    uint64_t p_fallback;      // first odd candidate after the fast path (p_cand_max + 2)
    uint64_t cap;             // fallback p cap (test hook)
    const uint64_t *base_bits;  // resident odd bitset of [3, R]
    uint64_t R;
    uint32_t n_base;          // odd primes in the resident list
    int64_t *result;
    uint32_t *dump;           // nullable
    uint32_t *carry;          // per-CTA carried sieve offsets, 2 per prime (nullable)
    uint64_t carry_stride;    // u32 entries per class per CTA (row = 2 * carry_stride)
    uint32_t n_carry;         // primes [0, n_carry) carried
    const uint16_t *med_idx;  // LPT schedule of the medium primes over the CTA's warps
    const uint32_t *med_off;  // (kThreads/32 + 1 offsets)
    uint32_t i_b2;            // first prime index with 2p > a full window (<= 2 hits per class)
    uint32_t i_b1;            // first prime index with p > a full window (<= 1 hit per class)
    uint32_t tile_words;      // words per class per tile: kTileWords, smaller when the halo is large
    const uint32_t *lmask;    // K-LARGE mask of this chunk (nullable): ANDed into every window
    int64_t lmask_g0;         // g of mask word 0
    uint64_t lmask_stride;    // class B words start here
};

// gb_sieve_segment: the wheel-class window sieve of the verify kernel (shared memory,
// carried offsets, K-LARGE mask) re-interleaved into the paper's odd layout.
// Output u32 word W <-> odd q in [3 + 64W, 3 + 64W + 64); class word g <-> output
// words 3g, 3g+1, 3g+2.
struct SieveOutArgs {
    SievePrimes sp;
    uint64_t g_first, g_end;  // class words [g_first, g_end) (tiles of tile_words)
    uint64_t n_tiles;
    uint32_t tile_words;
    uint64_t w_lo, w_hi;      // output u32 words [w_lo, w_hi) are written
    uint32_t *out;            // out[W - w_lo]
    uint32_t *carry;
    uint64_t carry_stride;
    uint32_t n_carry;
    const uint16_t *med_idx;
    const uint32_t *med_off;
    uint32_t i_b2, i_b1;
    const uint32_t *lmask;    // K-LARGE mask (nullable), word 0 <-> class word lmask_g0
    int64_t lmask_g0;
    uint64_t lmask_stride;
};

// NEXT-1 (gb_pern.cu): the paper's per-n gpu3 Phase-1 kernel over one segment.
constexpr uint64_t kPerNSegEvens = 1ull << 28;   // evens per segment (paper: SEG_SIZE = 1e7; larger here so
                                                 // gb_sieve_segment fills the GPU, bitset 32 MB in L2)
struct PerNArgs {
    uint64_t n_first, n_evens;     // evens n_first, n_first + 2, ...
    uint32_t n_cand;               // odd primes p <= p_max
    const uint32_t *primes;
    uint32_t n_base;
    const uint64_t *base_bits;     // resident odd bitset of [3, R]
    uint64_t R;
    const uint64_t *seg_bits;      // segment odd bitset, word 0 <-> global word seg_word_lo
    uint64_t seg_word_lo;
    uint64_t seg_q_lo, seg_q_hi;   // odd q in [seg_q_lo, seg_q_hi) are in seg_bits
    uint64_t p_fallback, cap, origin, lo_e;
    int64_t *result;
    uint32_t *dump;
};
cudaError_t launch_pern(const PerNArgs &a, cudaStream_t st);
cudaError_t launch_single_check(uint64_t n, uint64_t p_limit, const uint64_t *bits, uint64_t R, uint64_t *out,
                                cudaStream_t st);

// Launchers (gb_kernels.cu).  Each returns the cudaGetLastError() of its launch.
cudaError_t launch_seed(uint64_t s, uint32_t *primes, uint64_t *magic, uint4 *pk,
                        uint32_t *d_count, cudaStream_t st);
cudaError_t launch_segment(const SegmentArgs &a, cudaStream_t st);
cudaError_t launch_count_bits(const uint64_t *bits, uint64_t n_words, uint64_t *blk,
                              cudaStream_t st);
cudaError_t launch_scan(uint64_t *blk, uint64_t n_blk, cudaStream_t st);
cudaError_t launch_scatter(const uint64_t *bits, uint64_t n_words, const uint64_t *blk,
                           uint32_t *primes, uint64_t *magic, uint4 *pk, cudaStream_t st);
cudaError_t launch_result_init(int64_t *res, cudaStream_t st);
cudaError_t launch_verify(const VerifyArgs &a, int grid, size_t smem, cudaStream_t st);
cudaError_t launch_large(const LargeArgs &a, int num_sms, cudaStream_t st);   // mask fill + marking
cudaError_t launch_is_prime(const uint64_t *x, uint8_t *out, uint64_t n, const uint64_t *bits,
                            uint64_t R, cudaStream_t st);
cudaError_t launch_counts(const uint64_t *bits64, uint64_t n_words64, uint64_t lo_e, uint64_t hi, uint64_t *counts,
                          int num_sms, cudaStream_t st);
cudaError_t configure_verify();
cudaError_t ensure_dyn_smem(const void *kernel, int bytes, std::atomic<uint64_t> &done);
cudaError_t launch_sieve_out(const SieveOutArgs &a, int grid, size_t smem, cudaStream_t st);
int verify_blocks_per_sm(size_t smem);
uint32_t unroll_p_max();       // largest prime of the unrolled class tables

void count_launch();

}  // namespace gb

struct gb_ctx {
    int device;
    int num_sms;
    uint64_t origin, hi_max, R;
    uint32_t p_max;
    cudaStream_t create_stream;
    // workspace carve-out
    uint64_t *bits;        // odd bitset [3, R]
    uint64_t bits_words;
    uint32_t *primes;      // odd primes <= R
    uint64_t *magic;
    uint4 *pk;             // (p, kTileM mod p, rA, rB)
    uint32_t *carry;       // verify-kernel carried offsets: carry_ctas x carry_stride
    uint32_t *lmask;       // K-LARGE chunk mask (null when hi_max needs no primes > kCarryPrimeMax)
    uint64_t lmask_stride; // u32 words per class
    uint64_t carry_stride;
    uint32_t carry_ctas;
    uint16_t *med_idx;     // LPT schedule of medium primes (host-computed, copied once)
    uint32_t *med_off;
    uint64_t *blk;         // K-BASE scratch
    uint32_t *counter;     // K-BASE scratch
    int64_t *res_scratch;  // host API result
    uint32_t *dump_scratch;
    uint64_t *seg_scratch;  // NEXT-1 per-n mode: one segment's odd bitset
    uint64_t n_base;
    std::vector<uint32_t> h_primes;  // host copy for range planning
};
