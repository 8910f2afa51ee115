// mr64.cuh -- deterministic 64-bit Miller-Rabin on the GPU (fallback, subsystem (d)).
//
// PAPER.md:89 (priority 3 of the three-way oracle) and PAPER.md:185: "the
// 12-witness deterministic variant proven correct for all 64-bit integers";
// SPEC.md:128 fixes the witnesses as the first twelve primes 2..37, which is
// deterministic for every n < 3.3e24 > 2^64.  Arithmetic is Montgomery with
// R = 2^64 (__umul64hi for the high halves), so no 128-bit division is needed.
#pragma once
#include <stdint.h>

namespace gb {

__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, uint64_t m, uint64_t ninv)
{
    // REDC(a*b): (a*b + t*m) / 2^64 with t = (a*b mod 2^64) * (-m^-1) mod 2^64.
    uint64_t lo = a * b, hi = __umul64hi(a, b);
    uint64_t t = lo * ninv;
    uint64_t th = __umul64hi(t, m);
    uint64_t r = hi + th;
    bool ov = r < hi;
    uint64_t r2 = r + (lo != 0);          // lo + t*m == 0 mod 2^64: carry iff lo != 0
    ov |= r2 < r;
    if (ov || r2 >= m) r2 -= m;            // true value < 2m
    return r2;
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t m)
{
    // a, b < m
    return (a >= m - b) ? a - (m - b) : a + b;
}

// n odd, n > 37.
__device__ inline bool mr64_odd(uint64_t n)
{
    uint64_t inv = n;                      // n*n == 1 mod 8 for odd n
    for (int i = 0; i < 5; ++i) inv *= 2 - n * inv;
    const uint64_t ninv = 0 - inv;
    const uint64_t one = (0 - n) % n;      // 2^64 mod n
    uint64_t r2 = one;                     // 2^128 mod n by 64 doublings
    for (int i = 0; i < 64; ++i) r2 = add_mod(r2, r2, n);
    const uint64_t minus_one = n - one;
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    const uint32_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int w = 0; w < 12; ++w) {
        uint64_t a = bases[w] % n;
        if (a == 0) continue;
        uint64_t x = one;
        uint64_t b = mont_mul(a, r2, n, ninv);   // a in Montgomery form
        for (uint64_t e = d; e; e >>= 1) {
            if (e & 1) x = mont_mul(x, b, n, ninv);
            b = mont_mul(b, b, n, ninv);
        }
        if (x == one || x == minus_one) continue;
        bool comp = true;
        for (int i = 1; i < s; ++i) {
            x = mont_mul(x, x, n, ninv);
            if (x == minus_one) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

// Primality of any 64-bit value: tiny cases by the witness primes, then MR.
__device__ inline bool is_prime_u64(uint64_t n)
{
    if (n < 2) return false;
    const uint32_t small[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (int i = 0; i < 12; ++i) {
        if (n == small[i]) return true;
        if (n % small[i] == 0) return false;
    }
    if (n < 41 * 41) return true;
    return mr64_odd(n);
}

}  // namespace gb
