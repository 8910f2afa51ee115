// gb_pern.cu -- NEXT-1: the paper's own gpu3 Phase-1
// verification kernel, for a same-box comparison with the inverted bulk marking of
// gb_verify.cu.  PAPER.md:82-95 (section 2.3.2, Fig. 1): one GPU thread per even n
// of the segment scans candidate primes p ascending and tests q = n - p with the
// three-way primality oracle
//     q <= P_SMALL      -> resident small-prime bitset
//     q in the segment  -> the segment's odd bitset
//     otherwise         -> deterministic 64-bit Miller-Rabin
// stopping at the first prime q.  The paper's batches of primes, atomic counter and
// per-batch 8-byte readback become a per-thread early exit; n left
// unresolved after p_max go to the same on-GPU exhaustive fallback as the product
// path.  Results are accumulated into the same gb_result vector,
// so both modes must agree field by field.
#include <stdint.h>

#include <algorithm>

#include "gb_device.cuh"

namespace gb {

constexpr uint32_t kPerNSmemPrimes = 6542;    // odd primes <= 65521 (the default p_max)

// the MR64 branch (q below the segment and above R) is rare: out of line keeps the
// scan loop's registers and instruction footprint small
static __device__ __noinline__ bool mr64_cold(uint64_t q) { return mr64_odd(q); }

template <bool DUMP>
__global__ void __launch_bounds__(256) pern_kernel(const __grid_constant__ PerNArgs a)
{
    __shared__ uint32_t sh_hist[kHistSmem];
    __shared__ uint32_t sh_p[kPerNSmemPrimes];   // candidate primes, broadcast reads
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < kHistSmem; i += blockDim.x) sh_hist[i] = 0;
    const uint32_t n_sm = min(a.n_cand, kPerNSmemPrimes);
    for (uint32_t i = tid; i < n_sm; i += blockDim.x) sh_p[i] = __ldg(a.primes + i);
    __syncthreads();
    Acc acc;
    // grid-stride over the segment's evens (block-uniform trip count: the fallback
    // below is warp-cooperative)
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < a.n_evens;
         base += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = base + tid;
        const bool valid = idx < a.n_evens;
        const uint64_t n = a.n_first + 2 * idx;
        uint64_t pmin = 0;
        uint32_t bin = 0;
        if (valid) {
            acc.evens += 1;
            if (n == 4) {
                pmin = 2;
                bin = 1;
            } else {
                const uint64_t half = n / 2;
                for (uint32_t j = 0; j < a.n_cand; ++j) {
                    const uint32_t p = j < n_sm ? sh_p[j] : __ldg(a.primes + j);
                    if (p > half) break;                          // no partition below n/2
                    const uint64_t q = n - p;
                    bool prime;
                    if (q <= a.R) {                               // small-prime bitset
                        const uint64_t o = (q - 3) >> 1;
                        prime = (__ldg(a.base_bits + (o >> 6)) >> (o & 63)) & 1;
                    } else if (q >= a.seg_q_lo && q < a.seg_q_hi) {   // segment bitset
                        const uint64_t o = ((q - 3) >> 1) - 64 * a.seg_word_lo;
                        prime = (__ldg(a.seg_bits + (o >> 6)) >> (o & 63)) & 1;
                    } else {                                      // below the segment: MR64
                        prime = mr64_cold(q);
                    }
                    if (prime) {
                        pmin = p;
                        bin = j + 2;                              // primes[0] = 3 is bin 2
                        break;
                    }
                }
            }
        }
        // unresolved after the fast path: warp-cooperative exhaustive fallback, one n
        // at a time (all lanes scan that n's candidates together)
        bool open = valid && pmin == 0;
        if (open) acc.fast_unres += 1;
        while (true) {
            const uint32_t m = __ballot_sync(FULL, open);
            if (!m) break;
            const int L = __ffs(m) - 1;
            const uint64_t nL = __shfl_sync(FULL, n, L);
            const uint64_t p = fallback_scan(nL, a.p_fallback, a.cap, a.base_bits, a.R);
            if (lane == L) {
                open = false;
                if (p) {
                    pmin = p;
                    bin = bin_of_prime(p, a.primes, a.n_base);
                }
            }
        }
        if (valid) {
            if (pmin) {
                acc.verified += 1;
                acc.sum += pmin;
                note_key(acc, pmin, n, a.origin);
                hist_add(sh_hist, a.result, bin, 1);
            } else {
                acc.unres += 1;
                if (n < acc.first_unres) acc.first_unres = n;
                hist_add(sh_hist, a.result, 0, 1);
            }
            if (DUMP) a.dump[(n - a.lo_e) / 2] = (uint32_t)pmin;
        }
    }
    flush_acc(acc, a.result, lane);
    unsigned long long *R = (unsigned long long *)a.result;
    __syncthreads();
    for (int i = tid; i < kHistSmem; i += blockDim.x) {
        const uint32_t v = sh_hist[i];
        if (v) atomicAdd(R + GB_R_HIST + i, (unsigned long long)v);
    }
}

cudaError_t launch_pern(const PerNArgs &a, cudaStream_t st)
{
    if (a.n_evens == 0) return cudaSuccess;
    const uint64_t nb = std::min<uint64_t>((a.n_evens + 255) / 256, 148ull * 8);
    if (a.dump) pern_kernel<true><<<(unsigned)nb, 256, 0, st>>>(a);
    else pern_kernel<false><<<(unsigned)nb, 256, 0, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

}  // namespace gb

namespace gb {

// ---------------------------------------------------------------------------
// NEXT-3: single_check (section 2.4): the minimal prime p with
// n - p prime for ONE even n < 2^64.  One 1024-thread CTA scans odd candidates in
// batches of 1024 ascending (p tested by the resident bitset, or MR64 above R;
// q = n - p likewise) and stops at the first batch with a hit; the block minimum
// of that batch is p_min (the paper's variant returns any valid p; this one is
// minimal).  n = 4 -> 2.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) single_check_kernel(uint64_t n, uint64_t p_limit, const uint64_t *bits,
                                                            uint64_t R, uint64_t *out)
{
    __shared__ unsigned long long best;
    if (threadIdx.x == 0) best = ~0ull;
    __syncthreads();
    if (n == 4) {
        if (threadIdx.x == 0) *out = p_limit >= 2 ? 2 : 0;
        return;
    }
    const uint64_t half = n / 2;
    const uint64_t lim = half < p_limit ? half : p_limit;
    for (uint64_t base = 3; base <= lim; base += 2 * blockDim.x) {
        const uint64_t p = base + 2 * (uint64_t)threadIdx.x;
        if (p <= lim && is_prime_dev(p, bits, R) && is_prime_dev(n - p, bits, R)) atomicMin(&best, p);
        __syncthreads();
        if (best != ~0ull) break;                 // block-uniform: read after the barrier
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = best == ~0ull ? 0 : best;
}

cudaError_t launch_single_check(uint64_t n, uint64_t p_limit, const uint64_t *bits, uint64_t R, uint64_t *out,
                                cudaStream_t st)
{
    single_check_kernel<<<1, 1024, 0, st>>>(n, p_limit, bits, R, out);
    count_launch();
    return cudaGetLastError();
}

}  // namespace gb
