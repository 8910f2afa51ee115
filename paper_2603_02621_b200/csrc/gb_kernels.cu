// gb_kernels.cu -- K-BASE (resident small-prime table) and K-SIEVE in the paper's
// odd-only layout (gb_sieve_segment), plus the result-vector and MR64 entry kernels.
//
//   K-BASE   : seed sieve + segment sieve + compaction of the resident small-prime
//              table ("permanently resident small-primes bitset").
//   K-SIEVE  : odd-only bit-packed window sieve in shared memory (PAPER.md:76-78,
//              moved from the host CPU to the GPU as PAPER.md:421 proposes).
// The fused verify kernel (gb_verify.cu) sieves the same windows in a mod-6 wheel
// layout; both sieves are checked against the oracle.
//
// Odd layout: odd q <-> o(q) = (q-3)/2, 32 bits per word here (a
// 64-bit word of the paper's layout is two consecutive 32-bit words, little-endian).
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdio>

#include "gb_device.cuh"

namespace gb {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// cudaFuncSetAttribute applies to the current device's context only: opt each
// kernel in once per device (bit d of `done`), always to the largest size it is
// ever launched with, so no later call can lower it under another context's feet.
cudaError_t ensure_dyn_smem(const void *kernel, int bytes, std::atomic<uint64_t> &done)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}
}  // namespace gb

extern "C" uint64_t gb_launch_count(void) { return gb::g_launches.load(); }

namespace gb {

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

constexpr uint32_t kMedMax = 1024;           // medium primes 37..kWarpPrimeMax (1017 of them)

// ---------------------------------------------------------------------------
// K-SIEVE (odd layout): window of nw 32-bit words, word i <-> o in
// [32(g0+i), 32(g0+i)+32).  Words with g0 + i < 0 (q <= 1) are zero.  Bit = 1 iff
// q = 3 + 2o is prime, for every q whose square root is covered by sp.
// Ends WITHOUT a barrier; callers __syncthreads() before reading `win`.
// ---------------------------------------------------------------------------
__device__ void sieve_window(uint32_t *win, int64_t g0, uint32_t nw, const SievePrimes &sp)
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
    const int lane = tid & 31;
    // medium primes (31 < p <= kWarpPrimeMax): first hits into shared memory, one
    // thread per prime (overlaps phase T), then one warp per prime handed out
    // dynamically (ascending: largest work first).
    const uint32_t m_end = sp.i_big < sp.n_use ? sp.i_big : sp.n_use;
    __shared__ uint32_t sh_moff[kMedMax];
    __shared__ uint32_t sh_mnext;
    if (tid == 0) sh_mnext = sp.i_med;
    for (uint32_t pi = sp.i_med + tid; pi < m_end; pi += nt) {
        const uint32_t p = __ldg(sp.primes + pi);
        const uint64_t off = first_hit(p, __ldg(sp.magic + pi), o_lo, o_hi);
        sh_moff[pi - sp.i_med] = off == UINT64_MAX ? 0xFFFFFFFFu : (uint32_t)off;
    }
    __syncthreads();
    while (true) {
        uint32_t pi = 0;
        if (lane == 0) pi = atomicAdd(&sh_mnext, 1u);
        pi = __shfl_sync(FULL, pi, 0);
        if (pi >= m_end) break;
        const uint32_t off = sh_moff[pi - sp.i_med];
        if (off >= nbits) continue;
        const uint32_t p = __ldg(sp.primes + pi);
        const uint32_t stride = 32 * p;
        for (uint32_t b = off + lane * p; b < nbits; b += stride) atomicAnd(win + (b >> 5), clear_mask(b));
    }
    // large primes: one thread per prime
    const uint32_t b_begin = sp.i_big > sp.i_med ? sp.i_big : sp.i_med;
    for (uint32_t pi = b_begin + tid; pi < sp.n_use; pi += nt) {
        const uint32_t p = __ldg(sp.primes + pi);
        const uint64_t off = first_hit(p, __ldg(sp.magic + pi), o_lo, o_hi);
        if (off == UINT64_MAX) break;
        for (uint32_t b = (uint32_t)min(off, (uint64_t)nbits); b < nbits; b += p)
            atomicAnd(win + (b >> 5), clear_mask(b));
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
                                                    uint4 *pk, uint32_t *d_count)
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
        pk[i] = make_pk(primes[i]);
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
                                                      uint64_t *magic, uint4 *pk)
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
            pk[idx] = make_pk((uint32_t)q);
            ++idx;
        }
    }
}

// ---------------------------------------------------------------------------
// K-LARGE: sieving primes too large for the per-tile shared-memory sieve (p >
// kCarryPrimeMax: at most a few hits per verify window, most windows none).  Their
// multiples in class A (6m+1) and class B (6m+5) are cleared, one thread per prime,
// by no-return L2 atomics into a chunk mask that stays resident in L2; the verify
// kernel ANDs the mask into its windows.  The prime table is streamed with
// evict-first loads so it does not push the mask out of L2.
// ---------------------------------------------------------------------------
// L2 policy for the chunk mask: keep it resident (evict_last) while the prime table
// streams through with evict-first loads
__device__ __forceinline__ uint64_t l2_keep_policy()
{
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__global__ void __launch_bounds__(256) large_fill_kernel(uint32_t *mask, uint64_t stride, uint32_t nw)
{
    const uint64_t n = stride + nw;             // class A [0, nw) .. class B [stride, stride + nw)
    const uint64_t pol = l2_keep_policy();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(mask + i), "r"(0xFFFFFFFFu), "l"(pol)
                     : "memory");
}

__device__ __forceinline__ void gmem_and(uint32_t *p, uint32_t v, uint64_t pol)
{
    asm volatile("red.global.and.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

constexpr int kLargeBlock = 256;
constexpr int kLargeGridPerSm = 64;         // (8: one resident wave, 89.6 vs 83.3 ms on the C5 span)

// K-LARGE with a cofactor wheel.  A bit q = p k of the mask needs
// clearing only if no other sieve clears it: the window's shared-memory sieve
// clears every q with a prime factor <= 2^21 (q >= f^2 always holds here), so a
// multiple whose cofactor k has a factor 5, 7, 11, 13, 17 or 19 is cleared anyway
// (k even or divisible by 3 puts q outside classes A/B).  Each thread walks its
// prime's cofactors k >= max(p, q_lo / p) over the residues coprime to 210 and skips
// k divisible by 11..19 (a bitmap of k mod 11*13*17*19 in shared memory): 17% of the
// multiples instead of 33%, i.e. about half the L2 atomics of a plain walk.  The
// kernel is bound by those atomics: red.global.and runs at ~0.92 per clock per SM
// and saturates the L2 at ~1.8e11/s from ~100 SMs (64 MB buffer; 1.3e11/s at 96 MB,
// profiles/r02b_red_sms.json), against 1.15e8 REDs per 3-tile-per-SM chunk at 4e18.
struct Wheel210 {
    uint8_t res[48];                      // residues mod 210 coprime to 210, ascending
    uint8_t gap[48];                      // gap to the next residue (wrapping)
};
constexpr Wheel210 make_wheel210()
{
    Wheel210 w{};
    int c = 0;
    for (int r = 0; r < 210; ++r)
        if (r % 2 && r % 3 && r % 5 && r % 7) w.res[c++] = (uint8_t)r;
    for (int i = 0; i < 48; ++i) w.gap[i] = (uint8_t)(i + 1 < 48 ? w.res[i + 1] - w.res[i] : 210 + w.res[0] - w.res[i]);
    return w;
}
constexpr Wheel210 kW210 = make_wheel210();
static_assert(kW210.res[0] == 1 && kW210.res[47] == 209 && kW210.gap[47] == 2, "wheel 210");
__constant__ Wheel210 c_w210 = make_wheel210();

// k coprime to 11 * 13 * 17 * 19 = 46189, as a bitmap of k mod 46189 (5.8 KB):
// one residue register, one shared load and a bit test per cofactor step instead of
// four incremental residues and their tests
constexpr uint32_t kM4 = 11u * 13 * 17 * 19;
constexpr uint32_t kM4Words = (kM4 + 31) / 32;
struct CopBits {
    uint32_t w[kM4Words];
};
constexpr CopBits make_cop_bits()
{
    CopBits b{};
    for (uint32_t r = 0; r < kM4; ++r)
        if (r % 11 && r % 13 && r % 17 && r % 19) b.w[r >> 5] |= 1u << (r & 31);
    return b;
}
__device__ const CopBits g_cop = make_cop_bits();

__global__ void __launch_bounds__(kLargeBlock) large_mark_wheel_kernel(LargeArgs a)
{
    __shared__ uint8_t s_next[210];       // index of the first wheel residue >= r
    __shared__ uint8_t s_res[48], s_gap[48];
    __shared__ uint32_t s_cop[kM4Words];
    for (uint32_t i = threadIdx.x; i < kM4Words; i += blockDim.x) s_cop[i] = g_cop.w[i];
    for (int i = threadIdx.x; i < 48; i += blockDim.x) {
        s_res[i] = c_w210.res[i];
        s_gap[i] = c_w210.gap[i];
    }
    for (int r = threadIdx.x; r < 210; r += blockDim.x) {
        int j = 0;
        while (c_w210.res[j] < r) ++j;                    // 209 is a residue: j < 48
        s_next[r] = (uint8_t)j;
    }
    __syncthreads();
    const int64_t m_lo = a.g0 * 32;
    const uint32_t nbits = 32 * a.nw;
    // offsets off = q - q_base, m = off / 6; q_base = 6 m_lo wraps mod 2^64 when
    // m_lo < 0 (ranges starting below the halo), and exceeds INT64_MAX near 2^64
    const uint64_t q_base = 6 * (uint64_t)m_lo;
    const uint64_t lim_off = 6ull * nbits;                 // < 2^32 (launch_large checks 192 nw < 2^32)
    const uint64_t q_first = m_lo > 0 ? q_base : 0;
    const uint64_t n = a.i_end - a.i_begin;
    const uint64_t total = (uint64_t)gridDim.x * blockDim.x;
    uint32_t *__restrict__ mA = a.mask;
    uint32_t *__restrict__ mB = a.mask + a.stride;
    const uint64_t pol = l2_keep_policy();
    // the (p, reciprocal) pairs of the next prime(s) are loaded before this one is
    // walked: independent DRAM loads in flight per thread instead of two dependent
    // ones per prime (C5 span 84.8 -> 83.5 ms; two primes ahead: 83.6)
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t p_nx = 0;
    uint64_t mg_nx = 0;
    if (t < n) { p_nx = __ldcs(a.primes + a.i_begin + t); mg_nx = __ldcs(a.magic + a.i_begin + t); }
    for (; t < n; t += total) {
        const uint64_t p = p_nx;
        const uint64_t mg = mg_nx;
        if (t + total < n) {
            p_nx = __ldcs(a.primes + a.i_begin + (t + total));
            mg_nx = __ldcs(a.magic + a.i_begin + (t + total));
        }
        // first cofactor: k >= p (q >= p^2) and p k >= q_first
        uint64_t k = p;
        if (q_first > p * p) {
            const uint64_t x = q_first + p - 1;            // ceil(q_first / p)
            uint64_t quo = __umul64hi(x, mg);
            uint64_t rem = x - quo * p;
            while (rem >= p) { ++quo; rem -= p; }
            k = quo;
        }
        // one 64-bit reduction, then 32-bit residues (210 * 11 * 13 * 17 * 19 < 2^24)
        constexpr uint32_t kM = 210u * 11 * 13 * 17 * 19;
        const uint32_t km = (uint32_t)(k % kM);
        const uint32_t kr = km % 210;
        const uint32_t idx0 = s_next[kr];
        const uint32_t adv = s_res[idx0] - kr;
        k += adv;
        uint32_t idx = idx0;
        uint64_t off = p * k - q_base;
        if (off >= lim_off) continue;
        const uint32_t kk = km + adv;                     // k mod kM, possibly + up to 10
        uint32_t r = kk % kM4;
        while (off < lim_off) {
            const uint32_t o = (uint32_t)off;
            const uint32_t m = __umulhi(o, 0xAAAAAAABu) >> 2;     // o / 6
            if ((s_cop[r >> 5] >> (r & 31)) & 1u) {
                uint32_t *w = (o - 6 * m == 1 ? mA : mB) + (m >> 5);
                gmem_and(w, clear_mask(m), pol);
            }
            const uint32_t g = s_gap[idx];
            idx = idx == 47 ? 0 : idx + 1;
            off += p * g;
            r += g; if (r >= kM4) r -= kM4;
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

__global__ void is_prime_kernel(const uint64_t *x, uint8_t *out, uint64_t n)
{
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = is_prime_u64(x[i]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_seed(uint64_t s, uint32_t *primes, uint64_t *magic, uint4 *pk,
                        uint32_t *d_count, cudaStream_t st)
{
    static std::atomic<uint64_t> done{0};
    const cudaError_t attr = ensure_dyn_smem((const void *)seed_kernel, 65536 + 16, done);
    if (attr != cudaSuccess) return attr;
    seed_kernel<<<1, 1024, (size_t)s + 1, st>>>((uint32_t)s, primes, magic, pk, d_count);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_segment(const SegmentArgs &a, cudaStream_t st)
{
    const uint64_t nb = (a.n_words32 + kSieveTileWords - 1) / kSieveTileWords;
    if (nb == 0) return cudaSuccess;
    static std::atomic<uint64_t> done{0};
    const cudaError_t attr = ensure_dyn_smem((const void *)segment_kernel, kSieveTileWords * 4, done);
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
                           uint32_t *primes, uint64_t *magic, uint4 *pk, cudaStream_t st)
{
    const uint64_t nb = (n_words + kScanBlockWords - 1) / kScanBlockWords;
    scatter_kernel<<<(unsigned)nb, 256, 0, st>>>(bits, n_words, blk, primes, magic, pk);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_large(const LargeArgs &a, int num_sms, cudaStream_t st)
{
    large_fill_kernel<<<(unsigned)(8 * num_sms), 256, 0, st>>>(a.mask, a.stride, a.nw);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || a.i_end <= a.i_begin) return e;
    const uint64_t n = a.i_end - a.i_begin;
    // large_mark_wheel_kernel keeps integer offsets 6 * 32 * nw in 32 bits
    if ((uint64_t)a.nw * 192 >= (1ull << 32)) return cudaErrorInvalidValue;
    const uint64_t nb = std::min<uint64_t>((n + kLargeBlock - 1) / kLargeBlock, (uint64_t)kLargeGridPerSm * num_sms);
    large_mark_wheel_kernel<<<(unsigned)nb, kLargeBlock, 0, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_result_init(int64_t *res, cudaStream_t st)
{
    result_init_kernel<<<1, 256, 0, st>>>(res);
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
