// gb_counts.cu -- NEXT-4: Goldbach partition counts (section 4.5:
// "large-scale computation of Goldbach partition counts c(n)"), read as the
// Goldbach-comet count c(n) = #{p prime : p <= n/2, n - p prime} (R13).
//
// In the paper's odd layout (bit o <-> q = 3 + 2o) an odd pair
// p = 3 + 2i, q = n - p = 3 + 2j has i + j = K := (n - 6)/2, so for n >= 6
//      c(n) = #{ 0 <= i <= K/2 : O[i] & O[K - i] }            (c(4) = 1: 2 + 2)
// -- the prime bitset ANDed with a bit-REVERSED copy of itself shifted by K and
// popcounted.  A CTA takes 32 consecutive K (one tile of 32 even n) and a chunk
// of i-words: each thread loads its 32-bit word A = O[32w .. 32w+31] once, builds
// the 64 reversed bits around K - 32w once (two loads, a funnel shift, BREV), and
// then, for the 32 K of the tile, does SHF (immediate) + AND + POPC + add: the
// bound is the POPC pipe (16 lanes/clk/SM measured, profiles/peaks_int.json).
// Per-thread counts are transposed-reduced across the warp (lane s ends with
// the warp's total for K0 + s), summed over warps in shared memory, and added to
// the u64 result with one atomic per (K, CTA work item).
#include <stdint.h>

#include <algorithm>

#include "gb_device.cuh"

namespace gb {

constexpr int kCnThreads = 256;
constexpr int kCnTile = 32;           // K per tile (consecutive even n)
constexpr int kCnWpt = 32;            // i-words per thread per work item

// bits [base, base + 32) of the u32-word bitset (0 below bit 0 or at/after n_bits)
__device__ __forceinline__ uint32_t bits32_at(const uint32_t *__restrict__ w, int64_t base, uint64_t n_words)
{
    const int64_t wi = base >> 5;                      // floor division (arithmetic shift)
    const uint32_t sh = (uint32_t)(base & 31);
    const uint32_t a = (wi >= 0 && (uint64_t)wi < n_words) ? __ldg(w + wi) : 0u;
    const uint32_t b = (wi + 1 >= 0 && (uint64_t)(wi + 1) < n_words) ? __ldg(w + wi + 1) : 0u;
    return __funnelshift_r(a, b, sh);
}

__global__ void __launch_bounds__(kCnThreads, 2) counts_kernel(const uint32_t *__restrict__ bits, uint64_t n_words,
                                                            uint64_t K0, uint64_t nK, uint64_t *counts,
                                                            uint64_t words_per_item)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ uint32_t red[kCnThreads / 32][32];
    __shared__ uint32_t bnd[kCnTile];                                // boundary-word counts
    const uint64_t tile = blockIdx.x;
    const uint64_t Kt = K0 + tile * kCnTile;                       // K of s = 0
    const uint64_t kmax = min((uint64_t)kCnTile, nK - tile * kCnTile);
    const uint64_t Klast = Kt + kmax - 1;
    const uint64_t w_end = (Klast / 2) / 32 + 1;                   // words holding some i <= Klast/2
    const uint64_t w_full = Kt / 2 >= 31 ? (Kt / 2 - 31) / 32 + 1 : 0;   // words with every i <= Kt/2
    if (tid < kCnTile) bnd[tid] = 0;
    __syncthreads();
    for (uint64_t item = blockIdx.y; item * words_per_item < w_end; item += gridDim.y) {
        uint32_t cnt[kCnTile];
#pragma unroll
        for (int s = 0; s < kCnTile; ++s) cnt[s] = 0;
        const uint64_t wb = item * words_per_item;
        const uint64_t we = min(w_end, wb + words_per_item);
        const uint64_t wf = min(we, w_full);
        for (uint64_t w = wb + tid; w < wf; w += kCnThreads) {
            const uint32_t A = __ldg(bits + w);
            // reversed bits: B_s bit b = O[Kt + s - 32w - b]; with T = Kt - 32w and
            // W bit t = O[T - 32 + t] (t < 64), V = brev64(W): B_s = V >> (31 - s)
            const int64_t T = (int64_t)Kt - (int64_t)(32 * w);
            const uint32_t wlo = bits32_at(bits, T - 32, n_words), whi = bits32_at(bits, T, n_words);
            const uint32_t vlo = __brev(whi), vhi = __brev(wlo);
#pragma unroll
            for (int s = 0; s < kCnTile; ++s) cnt[s] += __popc(A & __funnelshift_r(vlo, vhi, 31 - s));
        }
        // boundary words (some i > K/2 for some K of the tile): one (word, s) pair per
        // thread, only i <= (Kt + s)/2 counted
        const uint64_t wb2 = max(wb, w_full);
        if (wb2 < we) {
            for (uint64_t x = tid; x < (we - wb2) * kCnTile; x += kCnThreads) {
                const uint64_t w = wb2 + x / kCnTile;
                const uint32_t s = (uint32_t)(x % kCnTile);
                if (s >= kmax) continue;
                const uint32_t A = __ldg(bits + w);
                const int64_t T = (int64_t)Kt - (int64_t)(32 * w);
                const uint32_t wlo = bits32_at(bits, T - 32, n_words), whi = bits32_at(bits, T, n_words);
                const uint32_t B = __funnelshift_r(__brev(whi), __brev(wlo), 31 - s);
                const int64_t lim = (int64_t)((Kt + s) >> 1) - (int64_t)(32 * w);   // last valid bit
                const uint32_t m = lim >= 31 ? 0xFFFFFFFFu : (lim < 0 ? 0u : (0xFFFFFFFFu >> (31 - lim)));
                const uint32_t c = __popc(A & B & m);
                if (c) atomicAdd(&bnd[s], c);
            }
        }
        // transpose-reduce over the warp: lane s ends with the sum of cnt[s]
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const bool upper = lane & off;
#pragma unroll
            for (int k = 0; k < off; ++k) {
                const uint32_t send = upper ? cnt[k] : cnt[k + off];
                const uint32_t keep = upper ? cnt[k + off] : cnt[k];
                cnt[k] = keep + __shfl_xor_sync(FULL, send, off);
            }
        }
        red[warp][lane] = cnt[0];
        __syncthreads();
        if (tid < kCnTile && (uint64_t)tid < kmax) {
            uint64_t t = bnd[tid];
            bnd[tid] = 0;
#pragma unroll
            for (int k = 0; k < kCnThreads / 32; ++k) t += red[k][tid];
            if (t) atomicAdd((unsigned long long *)(counts + tile * kCnTile + tid), (unsigned long long)t);
        }
        __syncthreads();
    }
}

__global__ void counts_init_kernel(uint64_t *counts, uint64_t n, int has4)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        counts[i] = (has4 && i == 0) ? 1 : 0;                     // c(4) = 1 (2 + 2)
}

// counts[(n - lo_e)/2] for even n in [lo_e, hi), lo_e >= 4 even; bits covers o <= (hi - 6)/2
cudaError_t launch_counts(const uint64_t *bits64, uint64_t n_words64, uint64_t lo_e, uint64_t hi, uint64_t *counts,
                          int num_sms, cudaStream_t st)
{
    const uint64_t ne = (hi - lo_e + 1) / 2;
    counts_init_kernel<<<(unsigned)std::min<uint64_t>((ne + 255) / 256, 8ull * num_sms), 256, 0, st>>>(
        counts, ne, lo_e == 4);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint64_t n6 = lo_e < 6 ? 6 : lo_e;                       // first n with an odd pair
    if (hi <= n6) return cudaSuccess;
    const uint64_t K0 = (n6 - 6) / 2, nK = (hi - n6 + 1) / 2;
    uint64_t *c6 = counts + (n6 - lo_e) / 2;
    const uint64_t tiles = (nK + kCnTile - 1) / kCnTile;
    const uint64_t Kmax = K0 + nK - 1;
    const uint64_t words = (Kmax / 2) / 32 + 1;
    const uint64_t wpi = (uint64_t)kCnThreads * kCnWpt;
    const uint64_t items = (words + wpi - 1) / wpi;
    if (tiles > 0x7FFFFFFFull) return cudaErrorInvalidValue;
    const unsigned gy = (unsigned)std::min<uint64_t>(items, 65535);
    counts_kernel<<<dim3((unsigned)tiles, gy), kCnThreads, 0, st>>>((const uint32_t *)bits64, 2 * n_words64, K0, nK,
                                                                    c6, wpi);
    count_launch();
    return cudaGetLastError();
}

}  // namespace gb
