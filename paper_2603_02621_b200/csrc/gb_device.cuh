// gb_device.cuh -- device helpers shared by gb_kernels.cu (K-BASE, K-SIEVE) and
// gb_verify.cu (the fused verify kernel).  Product code only.
#pragma once
#include <stdint.h>

#include "gb_internal.h"
#include "mr64.cuh"

namespace gb {

constexpr uint32_t FULL = 0xffffffffu;

// x mod p with m = floor((2^64-1)/p): the quotient estimate is low by <= 2.
__device__ __forceinline__ uint32_t mod_magic(uint64_t x, uint32_t p, uint64_t m)
{
    uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * p;
    while (r >= p) r -= p;
    return (uint32_t)r;
}

// bits 0, P, 2P, ... < 32 (the repeating hit pattern of a tiny prime in a 32-bit word)
__host__ __device__ constexpr uint32_t tiny_pattern(int P, int i = 0)
{
    return i >= 32 ? 0u : ((1u << i) | tiny_pattern(P, i + P));
}
template <int P>
struct Tiny {
    static constexpr uint32_t value = tiny_pattern(P);
};

// Per-prime constants of the mod-6 wheel sieve (gb_verify.cu): p, kTileM mod p,
// and the residues rA, rB of the m with p | 6m+1 and p | 6m+5.
// 6^-1 mod p is (5p+1)/6 for p == 1 (mod 6) and (p+1)/6 for p == 5 (mod 6).
__host__ __device__ inline uint4 make_pk(uint32_t p)
{
    if (p < 5) return make_uint4(p, 0, 0, 0);
    const uint32_t inv6 = (p % 6 == 1) ? (uint32_t)((5ull * p + 1) / 6) : (p + 1) / 6;
    const uint32_t rA = p - inv6;
    const uint32_t rB = (uint32_t)((5ull * rA) % p);
    return make_uint4(p, kTileM % p, rA, rB);
}

// shared-memory window address (32-bit state-space address) and a no-return AND on it
__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void smem_and(uint32_t saddr, uint32_t mask)
{
    asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(saddr), "r"(mask) : "memory");
}

// ~(1 << (b % 32)) as one funnel-shift rotate
__device__ __forceinline__ uint32_t clear_mask(uint32_t b)
{
    return __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b);
}

// ---------------------------------------------------------------------------
// fallback (subsystem (d)): warp-cooperative exhaustive scan for one n.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool is_prime_dev(uint64_t x, const uint64_t *bits, uint64_t R)
{
    if (x < 3) return x == 2;
    if ((x & 1) == 0) return false;
    if (x <= R) {
        const uint64_t o = (x - 3) >> 1;
        return (__ldg(bits + (o >> 6)) >> (o & 63)) & 1;
    }
    return mr64_odd(x);
}

// Minimal prime p in [p_start, min(n/2, cap)] (p_start odd) with n - p prime, or 0.
// All 32 lanes call it with the same n; lane l tests p_start + 2l + 64i
// ("tests all odd p ... with no upper bound on p").  Cold path:
// kept out of line so the hot loop stays small in the instruction cache.
static __device__ __noinline__ uint64_t fallback_scan(uint64_t n, uint64_t p_start, uint64_t cap,
                                                  const uint64_t *bits, uint64_t R)
{
    const int lane = threadIdx.x & 31;
    const uint64_t half = n / 2;
    const uint64_t lim = half < cap ? half : cap;
    for (uint64_t base = p_start; base <= lim; base += 64) {
        const uint64_t p = base + 2 * (uint64_t)lane;
        bool ok = false;
        if (p <= lim) ok = is_prime_dev(p, bits, R) && is_prime_dev(n - p, bits, R);
        const uint32_t m = __ballot_sync(FULL, ok);
        if (m) return __shfl_sync(FULL, p, __ffs(m) - 1);
    }
    return 0;
}

// histogram bin of an odd prime p: 1 + #primes <= p (bin 1 = the prime 2)
__device__ __forceinline__ uint32_t bin_of_prime(uint64_t p, const uint32_t *primes, uint32_t n_base)
{
    if (p > 65521) return GB_NBINS - 1;
    uint32_t lo = 0, hi = n_base;           // first index with primes[i] >= p
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(primes + mid) < p) lo = mid + 1; else hi = mid;
    }
    return lo + 2;                           // primes[0] = 3 is bin 2
}

struct Acc {
    uint64_t evens = 0, verified = 0, fast_unres = 0, unres = 0, sum = 0;
    uint64_t key = 0, first_unres = UINT64_MAX;
    uint64_t praw = 0;        // largest p_min above GB_KEY_PMAX (the key's p field saturates)
};

// End of a kernel: warp-reduce a thread's accumulators, then one atomic per warp per
// result field (SUM / MAX / MIN as include/gb.h defines them).
__device__ __forceinline__ void flush_acc(const Acc &acc, int64_t *result, int lane)
{
    auto wsum = [](uint64_t v) {
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        return v;
    };
    auto wmax = [](uint64_t v) {
        for (int o = 16; o; o >>= 1) { const uint64_t w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
        return v;
    };
    auto wmin = [](uint64_t v) {
        for (int o = 16; o; o >>= 1) { const uint64_t w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
        return v;
    };
    const uint64_t ev = wsum(acc.evens), vf = wsum(acc.verified), fu = wsum(acc.fast_unres);
    const uint64_t un = wsum(acc.unres), sm = wsum(acc.sum);
    const uint64_t ky = wmax(acc.key), fr = wmin(acc.first_unres), pr = wmax(acc.praw);
    unsigned long long *R = (unsigned long long *)result;
    if (lane == 0) {
        if (ev) atomicAdd(R + GB_R_EVENS, ev);
        if (vf) atomicAdd(R + GB_R_VERIFIED, vf);
        if (fu) atomicAdd(R + GB_R_FASTPATH_UNRESOLVED, fu);
        if (un) atomicAdd(R + GB_R_UNRESOLVED, un);
        if (sm) atomicAdd(R + GB_R_SUM_PMIN, sm);
        if (ky) atomicMax(R + GB_R_MAX_KEY, ky);
        if (pr) atomicMax(R + GB_R_MAX_PMIN_RAW, pr);
        if (fr != UINT64_MAX) atomicMin(R + GB_R_FIRST_UNRESOLVED_N, fr);
    }
}

// GB_R_MAX_KEY encoding: largest p first, then the smallest n
__device__ __forceinline__ uint64_t make_key(uint64_t p, uint64_t n, uint64_t origin)
{
    const uint64_t pk = p < GB_KEY_PMAX ? p : GB_KEY_PMAX;
    const uint64_t idx = (n - origin) >> 1;
    return (pk << GB_KEY_SHIFT) | ((1ull << GB_KEY_SHIFT) - 1 - idx);
}

// fold (p_min, n) into a thread's running max key (and the raw max p_min when the
// key's p field saturates)
__device__ __forceinline__ void note_key(Acc &acc, uint64_t p, uint64_t n, uint64_t origin)
{
    const uint64_t key = make_key(p, n, origin);
    if (key > acc.key) acc.key = key;
    if (p >= GB_KEY_PMAX && p > acc.praw) acc.praw = p;
}

__device__ __forceinline__ void hist_add(uint32_t *sh_hist, int64_t *res, uint32_t bin, uint32_t c)
{
    if (bin >= GB_NBINS) bin = GB_NBINS - 1;
    if (bin < (uint32_t)kHistSmem) atomicAdd(sh_hist + bin, c);
    else atomicAdd((unsigned long long *)(res + GB_R_HIST + bin), (unsigned long long)c);
}

}  // namespace gb
