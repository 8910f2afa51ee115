// gb_kernels.cu -- sm_100a kernels of the segmented double-sieve Goldbach verifier.
//
//   K-BASE   : seed sieve + segment sieve + compaction of the resident small-prime
//              table ("permanently resident small-primes bitset").
//   K-SIEVE  : odd-only bit-packed window sieve in shared memory (PAPER.md:76-78,
//              moved from the host CPU to the GPU as PAPER.md:421 proposes).
//   K-VERIFY : K-SIEVE fused with the inverted bulk-marking loop (PAPER.md:73-76,
//              406-410) and the on-GPU exhaustive fallback.
//
// Bit layouts: odd q <-> o(q) = (q-3)/2, even n <-> e(n) = (n-4)/2,
// both packed 32 bits per word here (a 64-bit word of the paper's layout is two
// consecutive 32-bit words, little-endian).  For odd p = 2k+1, o(n-p) = e(n) - k,
// so "n - p is prime" over a U word is the O bitset shifted up by k bits.
#include <stdint.h>

#include <atomic>
#include <cstdio>

#include "gb_internal.h"
#include "mr64.cuh"

namespace gb {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace gb

extern "C" uint64_t gb_launch_count(void) { return gb::g_launches.load(); }

namespace gb {

constexpr uint32_t FULL = 0xffffffffu;
#ifdef GB_PROFILE_PHASES
__device__ unsigned long long g_prof[4];
#endif

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mod_magic(uint64_t x, uint32_t p, uint64_t m)
{
    // x mod p with m = floor((2^64-1)/p): the quotient estimate is low by <= 2.
    uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * p;
    while (r >= p) r -= p;
    return (uint32_t)r;
}

// first local bit (relative to o_lo) of an odd multiple of p that is >= p^2 and
// >= o_lo, i.e. o = (p*m - 3)/2 with m odd; in o-space the multiples of p are the
// residue class o == (p-3)/2 (mod p).  Returns UINT64_MAX if p^2 is beyond o_hi.
__device__ __forceinline__ uint64_t first_hit(uint32_t p, uint64_t magic, int64_t o_lo, int64_t o_hi)
{
    const int64_t opp = (int64_t)(((uint64_t)p * p - 3) >> 1);
    if (opp >= o_hi) return UINT64_MAX;
    const uint64_t ostart = (uint64_t)(opp > o_lo ? opp : o_lo);
    const uint32_t r = mod_magic(ostart, p, magic);
    const uint32_t rp = (p - 3) >> 1;
    const uint32_t delta = rp >= r ? rp - r : rp + p - r;
    return ostart + delta - (uint64_t)o_lo;
}

// bits 0, P, 2P, ... < 32
__host__ __device__ constexpr uint32_t tiny_pattern(int P, int i = 0)
{
    return i >= 32 ? 0u : ((1u << i) | tiny_pattern(P, i + P));
}
// Carried sieve state of one persistent CTA: off[i] = first hit of prime i in the
// NEXT window, relative to its start (valid for primes active in this window).
constexpr uint32_t kTileBits = 32u * kTileWords;
constexpr uint32_t kMedMax = 1024;           // medium primes 37..kWarpPrimeMax (1017 of them)
struct Carry {
    uint32_t *off;
    uint32_t n_carry;
    uint32_t n_steady;       // primes [i_med, n_steady): carried, p^2 <= window start
    bool have_prev;
};

// first hit >= kTileBits of the progression off, off + p, ... minus kTileBits
__device__ __forceinline__ uint32_t next_tile_off(uint32_t off, uint32_t p, uint32_t tm)
{
    if (off >= kTileBits) return off - kTileBits;
    uint32_t om = off < p ? off : off % p;       // off >= p only when p^2 fell in this window
    return om >= tm ? om - tm : om + p - tm;
}

template <int P>
struct Tiny {
    static constexpr uint32_t value = tiny_pattern(P);
};

// ---------------------------------------------------------------------------
// K-SIEVE: window of nw 32-bit words, word i <-> o in [32(g0+i), 32(g0+i)+32).
// Words with g0 + i < 0 (q <= 1) are zero.  Bit = 1 iff q = 3 + 2o is prime, for
// every q whose square root is covered by sp (callers guarantee it).
// Ends WITHOUT a barrier; callers __syncthreads() before reading `win`.
// ---------------------------------------------------------------------------
__device__ void sieve_window(uint32_t *win, int64_t g0, uint32_t nw, const SievePrimes &sp,
                             const Carry *cy = nullptr)
{
    const int tid = threadIdx.x, nt = blockDim.x;
    // Phase T: primes 3..31 by shifted word patterns.  For word g the first
    // multiple sits at bit s_p = ((p-3)/2 - 32 g) mod p; mask = pattern_p << s_p.
    {
        // per-thread phases, advanced incrementally by 32*nt words
        int64_t g = g0 + tid;
        uint64_t gg = g < 0 ? 0 : (uint64_t)g;
#define GB_PHASE(P) int s##P = (int)(((uint64_t)(P - 3) / 2 + (uint64_t)P * 32 - (32 * (gg % P)) % P) % P); \
                    const int d##P = (32 * nt) % P;
        GB_PHASE(3) GB_PHASE(5) GB_PHASE(7) GB_PHASE(11) GB_PHASE(13)
        GB_PHASE(17) GB_PHASE(19) GB_PHASE(23) GB_PHASE(29) GB_PHASE(31)
#undef GB_PHASE
        for (int64_t i = tid; i < (int64_t)nw; i += nt, g += nt) {
            uint32_t w = 0;
            if (g >= 0) {
                uint32_t c = (Tiny<3>::value << s3) | (Tiny<5>::value << s5) |
                             (Tiny<7>::value << s7) | (Tiny<11>::value << s11) |
                             (Tiny<13>::value << s13) | (Tiny<17>::value << s17) |
                             (Tiny<19>::value << s19) | (Tiny<23>::value << s23) |
                             (Tiny<29>::value << s29) | (Tiny<31>::value << s31);
                w = ~c;
                if (g == 0) w |= 0x65B7u;   // restore 3,5,7,11,13,17,19,23,29,31 (o = 0,1,2,4,5,7,8,10,13,14)
            }
            win[i] = w;
            if (g >= 0) {
#define GB_ADV(P) s##P -= d##P; if (s##P < 0) s##P += P;
                GB_ADV(3) GB_ADV(5) GB_ADV(7) GB_ADV(11) GB_ADV(13)
                GB_ADV(17) GB_ADV(19) GB_ADV(23) GB_ADV(29) GB_ADV(31)
#undef GB_ADV
            } else if (g + nt >= 0) {
                // crossing from negative to non-negative words: recompute phases at g + nt
                uint64_t g2 = (uint64_t)(g + nt);
#define GB_RE(P) s##P = (int)(((uint64_t)(P - 3) / 2 + (uint64_t)P * 32 - (32 * (g2 % P)) % P) % P);
                GB_RE(3) GB_RE(5) GB_RE(7) GB_RE(11) GB_RE(13)
                GB_RE(17) GB_RE(19) GB_RE(23) GB_RE(29) GB_RE(31)
#undef GB_RE
            }
        }
    }
    const int64_t o_lo = g0 * 32;
    const int64_t o_hi = (g0 + (int64_t)nw) * 32;
    const uint32_t nbits = nw * 32;
    const int lane = tid & 31, warp = tid >> 5;
    // With a carry context (persistent verify CTAs walking consecutive tiles) the
    // first hit of a prime comes from the previous tile instead of a 64-bit modulo:
    // the window of tile t+1 starts kTileBits above that of tile t.  Primes
    // [i_med, n_steady) have p^2 <= the window start and were carried, so their
    // offset is valid and < p: no p^2 check and no modulo at all ("steady").
    const uint32_t ns = cy ? cy->n_steady : 0;
    // Phase M setup (overlaps phase T): the first hit of every medium prime
    // (31 < p <= kWarpPrimeMax) into shared memory, one thread per prime.
    const uint32_t m_end = sp.i_big < sp.n_use ? sp.i_big : sp.n_use;
    __shared__ uint32_t sh_moff[kMedMax];
    __shared__ uint32_t sh_mnext;
    if (tid == 0) sh_mnext = sp.i_med;
    for (uint32_t pi = sp.i_med + tid; pi < m_end; pi += nt) {
        const uint2 pt = __ldg(sp.ptm + pi);
        const uint32_t p = pt.x;
        uint32_t off = 0xFFFFFFFFu;
        if (pi < ns) {
            off = cy->off[pi];
            cy->off[pi] = off >= pt.y ? off - pt.y : off + p - pt.y;
        } else {
            const int64_t opp = (int64_t)(((uint64_t)p * p - 3) >> 1);
            if (opp < o_hi) {
                const bool carried = cy && pi < cy->n_carry;
                uint64_t o64;
                if (carried && cy->have_prev && opp < o_hi - (int64_t)kTileBits) o64 = cy->off[pi];
                else o64 = first_hit(p, __ldg(sp.magic + pi), o_lo, o_hi);
                off = (uint32_t)o64;
                if (carried) cy->off[pi] = next_tile_off(off, p, pt.y);
            }
        }
        sh_moff[pi - sp.i_med] = off;
    }
    __syncthreads();
    // Phase M: one warp per medium prime, primes handed out dynamically in
    // ascending order (largest work first), so the warps finish together.
    while (true) {
        uint32_t pi = 0;
        if (lane == 0) pi = atomicAdd(&sh_mnext, 1u);
        pi = __shfl_sync(FULL, pi, 0);
        if (pi >= m_end) break;
        const uint32_t off = sh_moff[pi - sp.i_med];
        if (off >= nbits) continue;
        const uint32_t p = __ldg(sp.primes + pi);
        const uint32_t stride = 32 * p;
        uint32_t b = off + lane * p;
        for (; b + 3 * stride < nbits; b += 4 * stride) {        // 4 hits per lane per trip
            const uint32_t b1 = b + stride, b2 = b1 + stride, b3 = b2 + stride;
            atomicAnd(win + (b >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b));   // ~(1 << b%32)
            atomicAnd(win + (b1 >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b1));
            atomicAnd(win + (b2 >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b2));
            atomicAnd(win + (b3 >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b3));
        }
        for (; b < nbits; b += stride)
            atomicAnd(win + (b >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b));
    }
    // Phase B: large primes, one thread per prime.  Steady primes first (the next
    // prime's loads issued before this prime's marks), then the rest.
    const uint32_t b_begin = sp.i_big > sp.i_med ? sp.i_big : sp.i_med;
    const uint32_t s_end = ns > b_begin ? (ns < sp.n_use ? ns : sp.n_use) : b_begin;
    // steady: kB primes per thread in flight (their loads issued together) to hide
    // the L2 latency of the per-CTA carry rows
    constexpr int kB = 8;
    // warp-uniform trip count (so __syncwarp below is legal)
    for (uint32_t w0 = b_begin + (tid & ~31u); w0 < s_end; w0 += kB * nt) {
        const uint32_t p0 = w0 + lane;
        uint2 pt[kB];
        uint32_t off[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const uint32_t pi = p0 + k * nt;
            if (pi < s_end) { pt[k] = __ldg(sp.ptm + pi); off[k] = cy->off[pi]; }
            else { pt[k] = make_uint2(1, 0); off[k] = nbits; }
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const uint32_t p = pt[k].x;
            for (uint32_t b = off[k]; b < nbits; b += p)
                atomicAnd(win + (b >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b));
            const uint32_t pi = p0 + k * nt;
            if (pi < s_end) cy->off[pi] = off[k] >= pt[k].y ? off[k] - pt[k].y : off[k] + p - pt[k].y;
        }
        __syncwarp();   // reconverge: the per-lane hit loops diverge
    }
    for (uint32_t pi = s_end + tid; pi < sp.n_use; pi += nt) {
        const uint2 pt = __ldg(sp.ptm + pi);
        const uint32_t p = pt.x;
        const int64_t opp = (int64_t)(((uint64_t)p * p - 3) >> 1);
        if (opp >= o_hi) break;
        const bool carried = cy && pi < cy->n_carry;
        uint64_t off;
        if (carried && cy->have_prev && opp < o_hi - (int64_t)kTileBits) off = cy->off[pi];
        else off = first_hit(p, __ldg(sp.magic + pi), o_lo, o_hi);
        uint32_t b = (uint32_t)min(off, (uint64_t)nbits);
        for (; b < nbits; b += p)
            atomicAnd(win + (b >> 5), __funnelshift_l(0xFFFFFFFEu, 0xFFFFFFFEu, b));
        if (carried) cy->off[pi] = next_tile_off((uint32_t)off, p, pt.y);
    }
}

// ---------------------------------------------------------------------------
// gb_sieve_segment / K-BASE stage 2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) segment_kernel(SegmentArgs a)
{
    extern __shared__ uint32_t win[];          // kSieveTileWords words
    const uint64_t t0 = (uint64_t)blockIdx.x * kSieveTileWords;
    const uint32_t nw = (uint32_t)min((uint64_t)kSieveTileWords, a.n_words32 - t0);
    const int64_t g0 = (int64_t)(a.g_lo + t0);
    sieve_window(win, g0, nw, a.sp);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) {
        uint32_t w = win[i];
        const uint64_t o0 = (uint64_t)(g0 + i) * 32;
        if (o0 + 32 > a.o_limit) {
            w = o0 >= a.o_limit ? 0u : (w & ((1u << (a.o_limit - o0)) - 1u));
        }
        a.out[t0 + i] = w;
    }
}

// ---------------------------------------------------------------------------
// K-BASE stage 1: primes <= s (s <= 65535) in one CTA, byte sieve in smem.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) seed_kernel(uint32_t s, uint32_t *primes, uint64_t *magic,
                                                    uint2 *ptm, uint32_t *d_count)
{
    extern __shared__ uint8_t flag[];
    for (uint32_t i = threadIdx.x; i <= s; i += blockDim.x) flag[i] = (i >= 2);
    __syncthreads();
    for (uint32_t i = 2; i * i <= s; ++i) {
        __syncthreads();
        if (!flag[i]) continue;   // uniform: flag[i] is final once all i' < i are done
        for (uint32_t m = i * i + threadIdx.x * i; m <= s; m += blockDim.x * i) flag[m] = 0;
    }
    __syncthreads();
    __shared__ uint32_t cnt;
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (uint32_t i = 3; i <= s; i += 2)
            if (flag[i]) primes[c++] = i;
        cnt = c;
        *d_count = c;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        magic[i] = ~0ull / primes[i];
        ptm[i] = make_uint2(primes[i], kTileBits % primes[i]);
    }
}

// ---------------------------------------------------------------------------
// K-BASE stage 3: compaction of the bitset into the ascending prime list.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) count_bits_kernel(const uint64_t *bits, uint64_t n_words,
                                                         uint64_t *blk)
{
    const uint64_t w0 = (uint64_t)blockIdx.x * kScanBlockWords;
    uint32_t c = 0;
    for (uint64_t i = w0 + threadIdx.x; i < w0 + kScanBlockWords && i < n_words; i += blockDim.x)
        c += __popcll(bits[i]);
    c = __reduce_add_sync(FULL, c);
    __shared__ uint32_t ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += ws[i];
        blk[blockIdx.x] = t;
    }
}

// exclusive scan of blk[0..n) in place; blk[n] = total.  One CTA.
__global__ void __launch_bounds__(1024) scan_kernel(uint64_t *blk, uint64_t n)
{
    __shared__ uint64_t part[1024];
    const uint64_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint64_t b = threadIdx.x * per, e = min(n, b + per);
    uint64_t s = 0;
    for (uint64_t i = b; i < e; ++i) s += blk[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) { uint64_t v = part[i]; part[i] = run; run += v; }
        blk[n] = run;
    }
    __syncthreads();
    uint64_t run = part[threadIdx.x];
    for (uint64_t i = b; i < e; ++i) { uint64_t v = blk[i]; blk[i] = run; run += v; }
}

__global__ void __launch_bounds__(256) scatter_kernel(const uint64_t *bits, uint64_t n_words,
                                                      const uint64_t *blk, uint32_t *primes,
                                                      uint64_t *magic, uint2 *ptm)
{
    // each thread owns kScanBlockWords/256 = 8 consecutive words of this block
    constexpr int per = kScanBlockWords / 256;
    const uint64_t w0 = (uint64_t)blockIdx.x * kScanBlockWords + (uint64_t)threadIdx.x * per;
    uint32_t c = 0;
    for (int i = 0; i < per; ++i)
        if (w0 + i < n_words) c += __popcll(bits[w0 + i]);
    // block-exclusive scan of c
    __shared__ uint32_t sc[256];
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        uint32_t v = threadIdx.x >= (unsigned)off ? sc[threadIdx.x - off] : 0;
        __syncthreads();
        sc[threadIdx.x] += v;
        __syncthreads();
    }
    uint64_t idx = blk[blockIdx.x] + sc[threadIdx.x] - c;
    for (int i = 0; i < per; ++i) {
        const uint64_t w = w0 + i;
        if (w >= n_words) break;
        uint64_t x = bits[w];
        while (x) {
            const int b = __ffsll((long long)x) - 1;
            x &= x - 1;
            const uint64_t q = 3 + 2 * (64 * w + (uint64_t)b);
            primes[idx] = (uint32_t)q;
            magic[idx] = ~0ull / q;
            ptm[idx] = make_uint2((uint32_t)q, (uint32_t)(kTileBits % q));
            ++idx;
        }
    }
}

// ---------------------------------------------------------------------------
// result vector
// ---------------------------------------------------------------------------
__global__ void result_init_kernel(int64_t *r)
{
    for (int i = threadIdx.x; i < GB_RESULT_WORDS; i += blockDim.x) r[i] = 0;
    if (threadIdx.x == 0) {
        r[GB_R_VERSION] = GB_RESULT_VERSION;
        r[GB_R_FIRST_UNRESOLVED_N] = INT64_MAX;
    }
}

__global__ void result_finalize_kernel(int64_t *r)
{
    const uint64_t c = (uint64_t)r[GB_R_CHK_RAW];
    r[GB_R_CHK_LO32] += (int64_t)(c & 0xffffffffu);
    r[GB_R_CHK_HI32] += (int64_t)(c >> 32);
    r[GB_R_CHK_RAW] = 0;
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
// All 32 lanes call it with the same n; lane l tests p_start + 2l + 64i.
__device__ uint64_t fallback_scan(uint64_t n, uint64_t p_start, uint64_t cap,
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

// histogram bin of an odd prime p found by the fallback: 1 + #primes <= p
__device__ uint32_t bin_of_prime(uint64_t p, const uint32_t *primes, uint32_t n_base)
{
    if (p > 65521) return GB_NBINS - 1;
    uint32_t lo = 0, hi = n_base;           // first index with primes[i] >= p
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(primes + mid) < p) lo = mid + 1; else hi = mid;
    }
    return lo + 2;                           // primes[0] = 3 is bin 2
}

// ---------------------------------------------------------------------------
// K-VERIFY: fused sieve -> inverted bulk marking -> fallback, persistent CTAs.
// ---------------------------------------------------------------------------
struct Acc {
    uint64_t evens = 0, verified = 0, fast_unres = 0, unres = 0, sum = 0, chk = 0;
    uint64_t key = 0, first_unres = UINT64_MAX;
};

__device__ __forceinline__ uint64_t make_key(uint64_t p, uint64_t n, uint64_t origin)
{
    const uint64_t pk = p < (1ull << 23) ? p : (1ull << 23) - 1;
    const uint64_t idx = (n - origin) >> 1;
    return (pk << GB_KEY_SHIFT) | ((1ull << GB_KEY_SHIFT) - 1 - idx);
}

__device__ __forceinline__ void hist_add(uint32_t *sh_hist, int64_t *res, uint32_t bin, uint32_t c)
{
    if (bin >= GB_NBINS) bin = GB_NBINS - 1;
    if (bin < (uint32_t)kHistSmem) atomicAdd(sh_hist + bin, c);
    else atomicAdd((unsigned long long *)(res + GB_R_HIST + bin), (unsigned long long)c);
}

// ---- compile-time table of the first kUnroll odd primes (3, 5, 7, ..., 3673) ----
// The fast path is fully unrolled over these, so every shift k = (p-1)/2, word
// offset k/32 and bit offset k%32 is an immediate ("bitwise
// AND/OR operations across aligned words").
#ifndef GB_UNROLL
#define GB_UNROLL 256
#endif
#ifndef GB_PHASE1
#define GB_PHASE1 64
#endif
constexpr int kUnroll = GB_UNROLL;
struct OddPrimeTable {
    uint32_t p[kUnroll];
};
constexpr OddPrimeTable make_odd_primes()
{
    OddPrimeTable t{};
    int c = 0;
    for (uint32_t x = 3; c < kUnroll; x += 2) {
        bool pr = true;
        for (uint32_t d = 3; d * d <= x; d += 2)
            if (x % d == 0) { pr = false; break; }
        if (pr) t.p[c++] = x;
    }
    return t;
}
constexpr OddPrimeTable kOddPrimes = make_odd_primes();
static_assert(kUnroll + 2 <= kHistSmem, "unrolled bins must live in the shared histogram");
static_assert(kOddPrimes.p[0] == 3 && kOddPrimes.p[kUnroll > 511 ? 511 : 0] == (kUnroll > 511 ? 3673 : 3),
              "odd prime table");

struct Lane {
    const uint32_t *w;   // &win[halo + local word]: O word of this lane's U word
    uint32_t U;          // unresolved evens of the word
    uint32_t word_sum;   // sum of p_min of bits resolved in the unrolled range
    uint32_t lb;         // 1 + index of the last 8-prime block with a hit (0 = none)
    uint32_t lu;         // U at the start of that block
    uint32_t *dump_w;    // dump entry of bit 0 of the word (DUMP only)
};

// one candidate prime P = kOddPrimes.p[J] against one U word: S = O << K (K = (P-1)/2)
template <int J, bool DUMP>
__device__ __forceinline__ uint32_t mark_step(Lane &m)
{
    constexpr uint32_t P = kOddPrimes.p[J];
    constexpr uint32_t K = P >> 1;
    constexpr int A = (int)(K >> 5);
    constexpr uint32_t B = K & 31;
    const uint32_t S = __funnelshift_l(m.w[-(A + 1)], m.w[-A], B);
    const uint32_t nw = m.U & S;          // n resolved now: n - P prime, no smaller p worked
    m.U ^= nw;
    const uint32_t c = __popc(nw);
    m.word_sum += c * P;
    if constexpr (DUMP) {
        uint32_t x = nw;
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            m.dump_w[b] = P;
        }
    }
    return c;
}

// 8 primes, then the warp's per-prime counts go to the CTA histogram: two counts
// per 32-bit register (16-bit fields: per word <= 32, per warp <= 1024), one
// REDUX per pair, then lanes 0..7 add one bin each (bin of odd prime J = J + 2).
template <int J, bool DUMP>
__device__ __forceinline__ void mark_block8(Lane &m, uint32_t *hist, int lane)
{
    const uint32_t Ub = m.U;
    const uint32_t c0 = mark_step<J + 0, DUMP>(m);
    const uint32_t c1 = mark_step<J + 1, DUMP>(m);
    const uint32_t c2 = mark_step<J + 2, DUMP>(m);
    const uint32_t c3 = mark_step<J + 3, DUMP>(m);
    const uint32_t c4 = mark_step<J + 4, DUMP>(m);
    const uint32_t c5 = mark_step<J + 5, DUMP>(m);
    const uint32_t c6 = mark_step<J + 6, DUMP>(m);
    const uint32_t c7 = mark_step<J + 7, DUMP>(m);
    if (m.U != Ub) {
        m.lb = J / 8 + 1;
        m.lu = Ub;
    }
    const uint32_t t0 = __reduce_add_sync(FULL, c0 | (c1 << 16));
    const uint32_t t1 = __reduce_add_sync(FULL, c2 | (c3 << 16));
    const uint32_t t2 = __reduce_add_sync(FULL, c4 | (c5 << 16));
    const uint32_t t3 = __reduce_add_sync(FULL, c6 | (c7 << 16));
    const uint32_t ts = (lane & 4) ? ((lane & 2) ? t3 : t2) : ((lane & 2) ? t1 : t0);
    const uint32_t v = (lane & 1) ? (ts >> 16) : (ts & 0xffffu);
    if (lane < 8 && v) atomicAdd(hist + J + 2 + lane, v);
}

template <int J, bool DUMP>
__device__ __forceinline__ void mark_unrolled(Lane &m, uint32_t *hist, int lane)
{
    if constexpr (J + 8 <= kUnroll) {
        if (!__any_sync(FULL, m.U != 0)) return;   // warp-level early exit, every 8 primes
        mark_block8<J, DUMP>(m, hist, lane);
        mark_unrolled<J + 8, DUMP>(m, hist, lane);
    }
}

// Phase 1 of the mark: the first kPhase1 primes for two words per lane (every word
// needs them: the max p_min index of a 32-even word is rarely below 40), no exit
// checks; the per-prime counts of both words share one REDUX.
constexpr int kPhase1 = GB_PHASE1;
constexpr int kQueue = 128;                  // per-warp survivor queue (entries)

template <int J, bool DUMP>
__device__ __forceinline__ void p1_block8(Lane &m0, Lane &m1, uint32_t *hist, int lane)
{
    const uint32_t U0 = m0.U, U1 = m1.U;
    uint32_t c[8];
    c[0] = mark_step<J + 0, DUMP>(m0); c[0] += mark_step<J + 0, DUMP>(m1);
    c[1] = mark_step<J + 1, DUMP>(m0); c[1] += mark_step<J + 1, DUMP>(m1);
    c[2] = mark_step<J + 2, DUMP>(m0); c[2] += mark_step<J + 2, DUMP>(m1);
    c[3] = mark_step<J + 3, DUMP>(m0); c[3] += mark_step<J + 3, DUMP>(m1);
    c[4] = mark_step<J + 4, DUMP>(m0); c[4] += mark_step<J + 4, DUMP>(m1);
    c[5] = mark_step<J + 5, DUMP>(m0); c[5] += mark_step<J + 5, DUMP>(m1);
    c[6] = mark_step<J + 6, DUMP>(m0); c[6] += mark_step<J + 6, DUMP>(m1);
    c[7] = mark_step<J + 7, DUMP>(m0); c[7] += mark_step<J + 7, DUMP>(m1);
    if (m0.U != U0) { m0.lb = J / 8 + 1; m0.lu = U0; }
    if (m1.U != U1) { m1.lb = J / 8 + 1; m1.lu = U1; }
    // per warp and prime <= 2048 hits: 16-bit fields
    const uint32_t t0 = __reduce_add_sync(FULL, c[0] + (c[1] << 16));
    const uint32_t t1 = __reduce_add_sync(FULL, c[2] + (c[3] << 16));
    const uint32_t t2 = __reduce_add_sync(FULL, c[4] + (c[5] << 16));
    const uint32_t t3 = __reduce_add_sync(FULL, c[6] + (c[7] << 16));
    const uint32_t ts = (lane & 4) ? ((lane & 2) ? t3 : t2) : ((lane & 2) ? t1 : t0);
    const uint32_t v = (lane & 1) ? (ts >> 16) : (ts & 0xffffu);
    if (lane < 8 && v) atomicAdd(hist + J + 2 + lane, v);
}

template <int J, bool DUMP>
__device__ __forceinline__ void p1_blocks(Lane &m0, Lane &m1, uint32_t *hist, int lane)
{
    if constexpr (J < kPhase1) {
        p1_block8<J, DUMP>(m0, m1, hist, lane);
        p1_blocks<J + 8, DUMP>(m0, m1, hist, lane);
    }
}

// max p_min among the hits recorded in m.lb/m.lu: replay that 8-prime block from
// the U saved at its start (only lanes holding the warp's latest block, and only
// when it can raise this warp's running maximum)
__device__ __forceinline__ void replay_key(const Lane &m, uint64_t u, const VerifyArgs &a,
                                           uint32_t &best_block, Acc &acc)
{
    const uint32_t bstar = __reduce_max_sync(FULL, m.lb);
    if (bstar == 0 || bstar < best_block) return;
    best_block = bstar;
    if (m.lb != bstar) return;
    const uint32_t jr = (bstar - 1) * 8;
    uint32_t x = m.lu, lp = 0, lbits = 0;
    for (int i = 0; i < 8; ++i) {
        const uint32_t p = __ldg(a.sp.primes + jr + i);
        const int k = (int)(p >> 1);
        const uint32_t S = __funnelshift_l(m.w[-(k >> 5) - 1], m.w[-(k >> 5)], k);
        const uint32_t nw = x & S;
        x ^= nw;
        if (nw) { lp = p; lbits = nw; }
    }
    const uint64_t n = 4 + 2 * (u * 32 + (uint64_t)(__ffs(lbits) - 1));
    const uint64_t key = make_key(lp, n, a.origin);
    if (key > acc.key) acc.key = key;
}

// Primes past the unrolled range (runtime loop), then the exhaustive on-GPU
// fallback for whatever the fast path left; folds the word into acc.
template <bool DUMP>
__device__ __forceinline__ void finish_word(uint32_t U, uint64_t word_sum, uint32_t j0, uint32_t base,
                                            uint64_t u, const uint32_t *win, uint32_t *sh_hist,
                                            const VerifyArgs &a, Acc &acc, int lane)
{
    const uint64_t e_dump0 = a.e_lo;
    uint32_t lastp = 0, lastb = 0;
    for (uint32_t j = j0; j < a.n_cand; ++j) {
        if (!__any_sync(FULL, U != 0)) break;
        const uint32_t p = __ldg(a.sp.primes + j);
        const uint32_t k = p >> 1;
        const uint32_t wa = k >> 5, bb = k & 31;
        const uint32_t S = __funnelshift_l(win[base - wa - 1], win[base - wa], bb);
        const uint32_t nw = U & S;
        const uint32_t c = __popc(nw);
        if (nw) {
            U ^= nw;
            word_sum += (uint64_t)c * p;
            lastp = p; lastb = nw;
            if (DUMP) {
                uint32_t x = nw;
                while (x) {
                    const int b = __ffs(x) - 1;
                    x &= x - 1;
                    a.dump[u * 32 + b - e_dump0] = p;
                }
            }
        }
        const uint32_t tot = __reduce_add_sync(FULL, c);
        if (lane == 0 && tot) hist_add(sh_hist, a.result, j + 2, tot);
    }
    if (lastp) {
        const uint64_t n = 4 + 2 * (u * 32 + (uint64_t)(__ffs(lastb) - 1));
        const uint64_t key = make_key(lastp, n, a.origin);
        if (key > acc.key) acc.key = key;
    }
    acc.fast_unres += __popc(U);
    while (true) {
        const uint32_t m = __ballot_sync(FULL, U != 0);
        if (!m) break;
        const int L = __ffs(m) - 1;
        const uint32_t lw = __shfl_sync(FULL, U, L);
        const uint64_t uL = __shfl_sync(FULL, u, L);
        const int bit = __ffs(lw) - 1;
        const uint64_t n = 4 + 2 * (uL * 32 + (uint64_t)bit);
        const uint64_t p = fallback_scan(n, a.p_fallback, a.cap, a.base_bits, a.R);
        if (lane == L) {
            U &= ~(1u << bit);
            if (p) {
                word_sum += p;
                hist_add(sh_hist, a.result, bin_of_prime(p, a.sp.primes, a.n_base), 1);
                const uint64_t key = make_key(p, n, a.origin);
                if (key > acc.key) acc.key = key;
            } else {
                acc.unres += 1;
                hist_add(sh_hist, a.result, 0, 1);
                if (n < acc.first_unres) acc.first_unres = n;
            }
            if (DUMP) a.dump[uL * 32 + bit - e_dump0] = (uint32_t)p;
        }
    }
    acc.sum += word_sum;
    acc.chk += word_sum * u;                 // sum p_min * floor((n-4)/64): u = e >> 5
}

__device__ __forceinline__ uint32_t valid_mask(uint64_t u, const VerifyArgs &a)
{
    const uint64_t eb = u * 32;
    uint32_t U = FULL;
    if (eb < a.e_lo) U = (a.e_lo - eb >= 32) ? 0u : (U << (a.e_lo - eb));
    if (eb + 32 > a.e_hi) U &= (a.e_hi <= eb) ? 0u : (FULL >> (eb + 32 - a.e_hi));
    return U;
}

// n = 4 (bit 0 of word 0): p_min = 2, the only even p (reading R2)
template <bool DUMP>
__device__ __forceinline__ uint32_t take_n4(uint32_t U, uint64_t u, uint32_t *sh_hist,
                                            const VerifyArgs &a, Acc &acc)
{
    if ((U & 1u) && u == 0) {
        U &= ~1u;
        acc.sum += 2;
        atomicAdd(sh_hist + 1, 1u);
        const uint64_t key = make_key(2, 4, a.origin);
        if (key > acc.key) acc.key = key;
        if (DUMP) a.dump[0 - a.e_lo] = 2;
    }
    return U;
}

// UNROLL: n_cand >= kUnroll, so the whole unrolled table is inside the fast path.
template <bool DUMP, bool UNROLL>
__global__ void __launch_bounds__(kThreads) verify_kernel(VerifyArgs a)
{
    extern __shared__ uint32_t win[];          // halo + kTileWords words
    __shared__ uint32_t sh_hist[kHistSmem];
    __shared__ uint32_t q_li[kThreads / 32][kQueue];
    __shared__ uint32_t q_U[kThreads / 32][kQueue];
    __shared__ uint32_t sh_next;               // next phase-1 round of the tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int i = tid; i < kHistSmem; i += blockDim.x) sh_hist[i] = 0;
    Acc acc;
    uint32_t best_block = 0;                   // per warp: replay only rounds that can raise the max
    const uint64_t e_dump0 = a.e_lo;
    // contiguous run of tiles per CTA, so the sieve can carry its offsets
    const uint64_t t_begin = (uint64_t)blockIdx.x * a.n_tiles / gridDim.x;
    const uint64_t t_end = (uint64_t)(blockIdx.x + 1) * a.n_tiles / gridDim.x;
    Carry cy;
    cy.off = a.carry ? a.carry + (uint64_t)blockIdx.x * a.carry_stride : nullptr;
    cy.n_carry = a.carry ? a.n_carry : 0;
    cy.have_prev = false;
    cy.n_steady = 0;
    __shared__ uint32_t sh_ns;
    uint32_t ns_run = 0;                       // thread 0: running count (monotone in the tile)

    for (uint64_t tile = t_begin; tile < t_end; ++tile) {
        const uint64_t u0 = a.u_first + tile * kTileWords;
        const uint32_t tw = (uint32_t)min((uint64_t)kTileWords, a.u_end - u0);
        __syncthreads();                      // previous tile fully consumed
#ifdef GB_PROFILE_PHASES
        long long t_start = clock64();
#endif
        if (tid == 0) {
            sh_next = 0;
            // steady primes of this window: carried (previous tile done by this CTA)
            // and p^2 <= 2*o_lo + 3, i.e. (p^2 - 3)/2 <= o_lo
            uint32_t ns = 0;
            const int64_t o_lo = ((int64_t)u0 - (int64_t)a.halo) * 32;
            if (cy.have_prev && o_lo > 0) {
                const uint64_t lim = 2 * (uint64_t)o_lo + 3;
                const uint32_t top = min(cy.n_carry, a.sp.n_use);
                ns = max(ns_run, a.sp.i_med);
                if (ns == a.sp.i_med) {              // first use: binary search
                    uint32_t lo = a.sp.i_med, hi = top;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        const uint64_t pm = __ldg(a.sp.primes + mid);
                        if (pm * pm <= lim) lo = mid + 1; else hi = mid;
                    }
                    ns = lo;
                } else {
                    while (ns < top) {
                        const uint64_t pm = __ldg(a.sp.primes + ns);
                        if (pm * pm > lim) break;
                        ++ns;
                    }
                }
                ns_run = ns;
            }
            sh_ns = ns;
        }
        __syncthreads();
        cy.n_steady = sh_ns;
        sieve_window(win, (int64_t)u0 - a.halo, a.halo + tw, a.sp, a.carry ? &cy : nullptr);
        cy.have_prev = true;
        __syncthreads();
#ifdef GB_PROFILE_PHASES
        long long t_sieved = clock64();
#endif

        if constexpr (UNROLL) {
            // phase 1: rounds of 64 words (2 per lane) through the first kPhase1 primes,
            // handed out dynamically; survivors queue per warp; batches of 32 go
            // through phase 2 (the rest of the unrolled table with warp exits)
            uint32_t qn = 0;
            const uint32_t n_rounds = (tw + 63) >> 6;
            auto phase2 = [&](uint32_t take) {
                const uint32_t e = qn - take;
                uint32_t li = 0, U = 0;
                if ((uint32_t)lane < take) { li = q_li[warp][e + lane]; U = q_U[warp][e + lane]; }
                __syncwarp();
                qn = e;
                const uint64_t u = u0 + li;
                Lane m;
                m.w = win + a.halo + li;
                m.U = U;
                m.word_sum = 0;
                m.lb = 0; m.lu = 0;
                m.dump_w = DUMP ? a.dump + ((int64_t)(u * 32) - (int64_t)e_dump0) : nullptr;
                mark_unrolled<kPhase1, DUMP>(m, sh_hist, lane);
                replay_key(m, u, a, best_block, acc);
                finish_word<DUMP>(m.U, m.word_sum, kUnroll, a.halo + li, u, win, sh_hist, a, acc, lane);
            };
            while (true) {
                uint32_t r = 0;
                if (lane == 0) r = atomicAdd(&sh_next, 1u);
                r = __shfl_sync(FULL, r, 0);
                if (r >= n_rounds) break;
                const uint32_t li0 = r * 64 + lane, li1 = li0 + 32;
                const uint64_t ua = u0 + li0, ub = u0 + li1;
                uint32_t Ua = li0 < tw ? valid_mask(ua, a) : 0u;
                uint32_t Ub = li1 < tw ? valid_mask(ub, a) : 0u;
                acc.evens += __popc(Ua) + __popc(Ub);
                Ua = take_n4<DUMP>(Ua, ua, sh_hist, a, acc);
                Lane m0, m1;
                m0.w = win + a.halo + (li0 < tw ? li0 : tw - 1);
                m1.w = win + a.halo + (li1 < tw ? li1 : tw - 1);
                m0.U = Ua; m1.U = Ub;
                m0.word_sum = m1.word_sum = 0;
                m0.lb = m1.lb = 0; m0.lu = m1.lu = 0;
                m0.dump_w = DUMP ? a.dump + ((int64_t)(ua * 32) - (int64_t)e_dump0) : nullptr;
                m1.dump_w = DUMP ? a.dump + ((int64_t)(ub * 32) - (int64_t)e_dump0) : nullptr;
                p1_blocks<0, DUMP>(m0, m1, sh_hist, lane);
                acc.sum += (uint64_t)m0.word_sum + m1.word_sum;
                acc.chk += (uint64_t)m0.word_sum * ua + (uint64_t)m1.word_sum * ub;
                // max key of the phase-1 hits of this round (both words may hold it)
                replay_key(m0, ua, a, best_block, acc);
                replay_key(m1, ub, a, best_block, acc);
                // enqueue survivors
                uint32_t bal = __ballot_sync(FULL, m0.U != 0);
                if (m0.U) {
                    const uint32_t pos = qn + __popc(bal & ((1u << lane) - 1));
                    q_li[warp][pos] = li0;
                    q_U[warp][pos] = m0.U;
                }
                qn += __popc(bal);
                bal = __ballot_sync(FULL, m1.U != 0);
                if (m1.U) {
                    const uint32_t pos = qn + __popc(bal & ((1u << lane) - 1));
                    q_li[warp][pos] = li1;
                    q_U[warp][pos] = m1.U;
                }
                qn += __popc(bal);
                __syncwarp();
                while (qn >= 32) phase2(32);
            }
            if (qn > 0) phase2(qn);
        } else {
            // p_max below the unrolled table: runtime loop for every word (tests)
            const uint32_t n_rounds = (tw + 31) >> 5;
            for (uint32_t r = warp; r < n_rounds; r += nwarps) {
                const uint32_t li = r * 32 + lane;
                const uint64_t u = u0 + li;
                uint32_t U = li < tw ? valid_mask(u, a) : 0u;
                acc.evens += __popc(U);
                U = take_n4<DUMP>(U, u, sh_hist, a, acc);
                finish_word<DUMP>(U, 0, 0, a.halo + (li < tw ? li : tw - 1), u, win, sh_hist, a, acc,
                                  lane);
            }
        }
        // per-tile flush of the shared histogram keeps its 32-bit bins exact
#ifdef GB_PROFILE_PHASES
        long long t_marked = clock64();
#endif
        __syncthreads();
#ifdef GB_PROFILE_PHASES
        long long t_synced = clock64();
        if (lane == 0) {
            atomicAdd(&g_prof[0], (unsigned long long)(t_sieved - t_start));
            atomicAdd(&g_prof[1], (unsigned long long)(t_marked - t_sieved));
            atomicAdd(&g_prof[2], (unsigned long long)(t_synced - t_marked));
            atomicAdd(&g_prof[3], 1ull);
        }
        if (blockIdx.x == 0 && tid == 0 && tile + 1 == t_end)
            printf("GBPROF sieve=%llu mark=%llu markwait=%llu warp-tiles=%llu (cycles summed over warps, all CTAs so far)\n",
                   g_prof[0], g_prof[1], g_prof[2], g_prof[3]);
#endif
        {
            unsigned long long *R = (unsigned long long *)a.result;
            for (int i = tid; i < kHistSmem; i += blockDim.x) {
                const uint32_t v = sh_hist[i];
                if (v) {
                    atomicAdd(R + GB_R_HIST + i, (unsigned long long)v);
                    sh_hist[i] = 0;
                }
            }
        }
    }
    acc.verified = acc.evens - acc.unres;

    // flush: warp-reduce then one atomic per warp per field
    auto wsum = [&](uint64_t v) {
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        return v;
    };
    auto wmax = [&](uint64_t v) {
        for (int o = 16; o; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
        return v;
    };
    auto wmin = [&](uint64_t v) {
        for (int o = 16; o; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
        return v;
    };
    const uint64_t ev = wsum(acc.evens), vf = wsum(acc.verified), fu = wsum(acc.fast_unres);
    const uint64_t un = wsum(acc.unres), sm = wsum(acc.sum), ck = wsum(acc.chk);
    const uint64_t ky = wmax(acc.key), fr = wmin(acc.first_unres);
    unsigned long long *R = (unsigned long long *)a.result;
    if (lane == 0) {
        if (ev) atomicAdd(R + GB_R_EVENS, ev);
        if (vf) atomicAdd(R + GB_R_VERIFIED, vf);
        if (fu) atomicAdd(R + GB_R_FASTPATH_UNRESOLVED, fu);
        if (un) atomicAdd(R + GB_R_UNRESOLVED, un);
        if (sm) atomicAdd(R + GB_R_SUM_PMIN, sm);
        if (ck) atomicAdd(R + GB_R_CHK_RAW, ck);
        if (ky) atomicMax(R + GB_R_MAX_KEY, ky);
        if (fr != UINT64_MAX) atomicMin(R + GB_R_FIRST_UNRESOLVED_N, fr);
    }
}

__global__ void is_prime_kernel(const uint64_t *x, uint8_t *out, uint64_t n)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = is_prime_u64(x[i]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_seed(uint64_t s, uint32_t *primes, uint64_t *magic, uint2 *ptm,
                        uint32_t *d_count, cudaStream_t st)
{
    static const cudaError_t attr = cudaFuncSetAttribute(
        seed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 16);
    if (attr != cudaSuccess) return attr;
    seed_kernel<<<1, 1024, (size_t)s + 1, st>>>((uint32_t)s, primes, magic, ptm, d_count);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_segment(const SegmentArgs &a, cudaStream_t st)
{
    const uint64_t nb = (a.n_words32 + kSieveTileWords - 1) / kSieveTileWords;
    if (nb == 0) return cudaSuccess;
    static const cudaError_t attr = cudaFuncSetAttribute(
        segment_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSieveTileWords * 4);
    if (attr != cudaSuccess) return attr;
    segment_kernel<<<(unsigned)nb, kThreads, kSieveTileWords * 4, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_count_bits(const uint64_t *bits, uint64_t n_words, uint64_t *blk, cudaStream_t st)
{
    const uint64_t nb = (n_words + kScanBlockWords - 1) / kScanBlockWords;
    count_bits_kernel<<<(unsigned)nb, 256, 0, st>>>(bits, n_words, blk);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_scan(uint64_t *blk, uint64_t n_blk, cudaStream_t st)
{
    scan_kernel<<<1, 1024, 0, st>>>(blk, n_blk);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_scatter(const uint64_t *bits, uint64_t n_words, const uint64_t *blk,
                           uint32_t *primes, uint64_t *magic, uint2 *ptm, cudaStream_t st)
{
    const uint64_t nb = (n_words + kScanBlockWords - 1) / kScanBlockWords;
    scatter_kernel<<<(unsigned)nb, 256, 0, st>>>(bits, n_words, blk, primes, magic, ptm);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_result_init(int64_t *res, cudaStream_t st)
{
    result_init_kernel<<<1, 256, 0, st>>>(res);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_result_finalize(int64_t *res, cudaStream_t st)
{
    result_finalize_kernel<<<1, 1, 0, st>>>(res);
    count_launch();
    return cudaGetLastError();
}

cudaError_t configure_verify(size_t smem_max)
{
    const int sm = (int)smem_max;
    cudaError_t e = cudaFuncSetAttribute(verify_kernel<false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(verify_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(verify_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(verify_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    return e;
}

int verify_blocks_per_sm(size_t smem)
{
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, verify_kernel<false, true>, kThreads, smem) !=
        cudaSuccess)
        return 1;
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_verify(const VerifyArgs &a, int grid, size_t smem, cudaStream_t st)
{
    const bool unroll = a.n_cand >= (uint32_t)kUnroll;
    if (a.dump) {
        if (unroll) verify_kernel<true, true><<<grid, kThreads, smem, st>>>(a);
        else verify_kernel<true, false><<<grid, kThreads, smem, st>>>(a);
    } else {
        if (unroll) verify_kernel<false, true><<<grid, kThreads, smem, st>>>(a);
        else verify_kernel<false, false><<<grid, kThreads, smem, st>>>(a);
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_is_prime(const uint64_t *x, uint8_t *out, uint64_t n, const uint64_t *,
                            uint64_t, cudaStream_t st)
{
    if (n == 0) return cudaSuccess;
    is_prime_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, out, n);
    count_launch();
    return cudaGetLastError();
}

}  // namespace gb
