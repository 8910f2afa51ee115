// gb_verify.cu -- K-VERIFY: the fused segment sieve -> inverted bulk marking ->
// exhaustive fallback, on the mod-6 wheel.
//
// The method (section 2.3.1): "iterate over candidate primes p and
// mark all even n for which q = n - p is prime", in the bitwise bulk-marking form
// of PAPER.md:406-410 ("replacing per-n lookups with bitwise AND/OR operations
// across aligned words"), with the segment sieve on the GPU.
//
// Wheel layout (a B200 design choice; results are the plain definition's):
//   even n = 6m + a, a in {0, 2, 4}     -> U classes U0, U2, U4 (bit m of class a)
//   odd  q = 6m + 1 (class A), 6m + 5 (class B); q divisible by 3 is never prime
//   except 3 itself, so the sieve keeps 1 bit per 3 integers instead of 1 per 2.
// For p = 6j + b the partner q = n - p is:
//   a = 0: b = 1 -> B[m - j - 1]   b = 5 -> A[m - j - 1]   (p = 3 only for n = 6)
//   a = 2: b = 1 -> A[m - j]       b = 5 -> q = 0 mod 3     p = 3 -> B[m - 1]
//   a = 4: b = 1 -> q = 0 mod 3    b = 5 -> B[m - j - 1]    p = 3 -> A[m]
// so U2 only needs p = 3 and p = 1 (mod 6), U4 p = 3 and p = 5 (mod 6): skipping the
// primes that can only give q = 3 (whose n then has p_min = 3 anyway) halves the
// candidate list of two thirds of the evens.  "n - p prime" over a U word is the
// class A or B window shifted up by s = j (+1) bits: funnelshift(O[w-a-1], O[w-a], b)
// with s = 32a + b.
#include <stdint.h>

#include <atomic>
#include <cstdio>

#include "gb_device.cuh"

namespace gb {


// ---------------------------------------------------------------------------
// transitions and compile-time class tables
// ---------------------------------------------------------------------------
struct Trans {
    int ok;           // 0: p never gives an odd prime partner > 3 for this class
    int src;          // 0 = class A window, 1 = class B window
    uint32_t shift;   // U bit m <-> src bit m - shift
};

__host__ __device__ constexpr Trans trans(int a, uint32_t p)
{
    if (p == 3) return a == 2 ? Trans{1, 1, 1} : (a == 4 ? Trans{1, 0, 0} : Trans{0, 0, 0});
    const uint32_t j = p / 6, b = p % 6;
    if (a == 0) return b == 1 ? Trans{1, 1, j + 1} : Trans{1, 0, j + 1};
    if (a == 2) return b == 1 ? Trans{1, 0, j} : Trans{0, 0, 0};
    return b == 5 ? Trans{1, 1, j + 1} : Trans{0, 0, 0};
}

constexpr int kK = 224;          // unrolled candidates per class (96 / 128 / 192 / 256: slower at 4e18)
constexpr int kP1 = 56;          // phase 1: candidates every word goes through (48 / 64: slower at 1e12)
constexpr int kP1L = 64;         // the same in the K-LARGE regime (56: 1.9% slower at 4e18, 48: 3.7%)
constexpr uint32_t kWinSlack = kWinSlackWords;   // words past a window phase-1 lanes may read (U = 0)
constexpr int kQueue = kQueueEntries;   // per-warp survivor queue (<= 31 carried + 32 kW per round)
static_assert(kK % 8 == 0 && kP1 % 8 == 0 && kP1 <= kK && kP1L % 8 == 0 && kP1L <= kK, "blocks of 8 candidates");


struct ClassTable {
    uint32_t p[kK];
    uint32_t bin[kK];     // histogram bin = number of primes <= p (bin 1 = the prime 2)
};

__host__ __device__ constexpr bool is_prime_small(uint32_t x)
{
    if (x < 2) return false;
    if (x % 2 == 0) return x == 2;
    for (uint32_t d = 3; d * d <= x; d += 2)
        if (x % d == 0) return false;
    return true;
}

constexpr ClassTable make_class_table(int a)
{
    ClassTable t{};
    int c = 0;
    uint32_t nprimes = 1;   // the prime 2
    for (uint32_t x = 3; c < kK; x += 2) {
        if (!is_prime_small(x)) continue;
        ++nprimes;
        if (trans(a, x).ok) {
            t.p[c] = x;
            t.bin[c] = nprimes;
            ++c;
        }
    }
    return t;
}

constexpr ClassTable kTab[3] = {make_class_table(0), make_class_table(2), make_class_table(4)};
static_assert(kTab[0].p[0] == 5 && kTab[1].p[0] == 3 && kTab[1].p[1] == 7 && kTab[2].p[1] == 5,
              "class tables");
static_assert(kTab[0].bin[0] == 3 && kTab[1].bin[0] == 2, "bins: 2 -> 1, 3 -> 2, 5 -> 3");
__constant__ ClassTable c_tab[3] = {make_class_table(0), make_class_table(2), make_class_table(4)};

constexpr uint32_t max3(uint32_t a, uint32_t b, uint32_t c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
constexpr uint32_t kUnrollPMax = max3(kTab[0].p[kK - 1], kTab[1].p[kK - 1], kTab[2].p[kK - 1]);
uint32_t unroll_p_max() { return kUnrollPMax; }

// ---------------------------------------------------------------------------
// K-SIEVE on the wheel: class A and class B windows of nw words each, word i
// covering m in [32(g0+i), 32(g0+i)+32).  Bit = 1 iff q = 6m+1 (A) / 6m+5 (B)
// is prime.  Multiples of p in class c are m == r_c (mod p), r_A = -1/6, r_B = -5/6.
// ---------------------------------------------------------------------------
constexpr uint32_t kMedMax = 1024;

struct MedSched {
    const uint16_t *idx;     // medium prime (relative to i_med) per slot, grouped by warp
    const uint32_t *off;     // warp w owns slots [off[w], off[w+1])
};

struct Carry6 {
    uint32_t *off;            // [0, stride): class A offsets, [stride, 2 stride): class B
    uint64_t stride;
    uint32_t n_carry;
    uint32_t n_steady;        // primes [i_med, n_steady): carried, p^2 <= 6 m_lo + 1
    bool init;                // first tile of a run: fill the carry row for [i_med, n_steady) first
    uint32_t tile_m;          // m-span of a tile (window step); kTileM unless p_max forces a smaller tile
    bool have_prev;
};

// (tile_m mod p): precomputed in pk.y for the default tile, else computed
template <bool DEF_TILE>
__device__ __forceinline__ uint32_t tile_mod(const Carry6 *cy, uint4 k)
{
    if constexpr (DEF_TILE) return k.y;
    else return cy->tile_m % k.x;
}

__host__ __device__ constexpr uint32_t inv6(uint32_t p) { return p % 6 == 1 ? (5 * p + 1) / 6 : (p + 1) / 6; }
__host__ __device__ constexpr uint32_t rA_of(uint32_t p) { return p - inv6(p); }
__host__ __device__ constexpr uint32_t rB_of(uint32_t p) { return (5 * rA_of(p)) % p; }

// first hits (local offsets from m_lo) of the progressions m == rA, rB (mod p) with
// m >= (p^2-1)/6 (the first multiple cleared is p^2), 0xFFFFFFFF if p^2 is beyond
// the window; both classes share the start ms and its residue (one modulo)
__device__ __forceinline__ void first_hits6(uint32_t p, uint32_t rA, uint32_t rB, uint64_t magic, int64_t m_lo,
                                            int64_t m_hi, uint32_t &oa, uint32_t &ob)
{
    const int64_t mmin = (int64_t)(((uint64_t)p * p - 1) / 6);
    if (mmin >= m_hi) { oa = ob = 0xFFFFFFFFu; return; }
    const uint64_t ms = (uint64_t)(mmin > m_lo ? mmin : m_lo);
    const uint32_t rem = mod_magic(ms, p, magic);
    const uint64_t base = ms - (uint64_t)m_lo;
    oa = (uint32_t)(base + (rA >= rem ? rA - rem : rA + p - rem));
    ob = (uint32_t)(base + (rB >= rem ? rB - rem : rB + p - rem));
}

// class-B offset of a steady prime from its class-A offset (both residues mod p):
// m == rB and m == rA (mod p) differ by rB - rA
__device__ __forceinline__ uint32_t class_b_off(uint32_t oa, uint4 k)
{
    const uint32_t d = k.w >= k.z ? k.w - k.z : k.w + k.x - k.z;
    const uint32_t ob = oa + d;
    return ob >= k.x ? ob - k.x : ob;
}

// first hits of a steady prime (p^2 below the window) by one modulo of m_lo: the
// offsets (rA - m_lo) mod p and (rB - m_lo) mod p (the carry-free path)
__device__ __forceinline__ void steady_first(uint4 k, int64_t m_lo, uint64_t magic, uint32_t &oa, uint32_t &ob)
{
    const uint32_t rem = mod_magic((uint64_t)m_lo, k.x, magic);
    oa = k.z >= rem ? k.z - rem : k.z + k.x - rem;
    ob = k.w >= rem ? k.w - rem : k.w + k.x - rem;
}

// next tile's first hit (the window moves up by tile_m)
__device__ __forceinline__ uint32_t next_off6(uint32_t off, uint32_t p, uint32_t tm, uint32_t tile_m)
{
    if (off >= tile_m) return off - tile_m;
    const uint32_t om = off < p ? off : off % p;   // off >= p only when p^2 fell in this window
    return om >= tm ? om - tm : om + p - tm;
}

// clear bit b of the window at shared address w (word b / 32)
__device__ __forceinline__ void clear_bit(uint32_t w, uint32_t b)
{
    smem_and(w + ((b >> 5) << 2), clear_mask(b));
}

// One warp, one medium prime, both classes: lane l marks hits l, l + 32, ... of each
// class (bits off + (l + 32i) p).  The stride is p whole words, so a lane's bit-in-
// word (hence its mask) never changes: only the word address moves, by 4p bytes per
// hit.  The two classes' per-lane hit counts differ by at most one, so they share one
// loop (half the loop overhead per RED, two independent address streams).
__device__ __forceinline__ void mark_progression2(uint32_t wA, uint32_t offA, uint32_t hitsA, uint32_t wB,
                                                  uint32_t offB, uint32_t hitsB, uint32_t p, uint32_t lane)
{
    const uint32_t nA = (hitsA + 31 - lane) >> 5, nB = (hitsB + 31 - lane) >> 5;
    const uint32_t bA = offA + lane * p, bB = offB + lane * p;
    const uint32_t mA = clear_mask(bA), mB = clear_mask(bB);
    const uint32_t step = 4 * p;
    uint32_t adA = wA + ((bA >> 5) << 2), adB = wB + ((bB >> 5) << 2);
    const uint32_t n = min(nA, nB);
    uint32_t i = 0;
    for (; i + 2 <= n; i += 2, adA += 2 * step, adB += 2 * step) {
        smem_and(adA, mA);
        smem_and(adB, mB);
        smem_and(adA + step, mA);
        smem_and(adB + step, mB);
    }
    for (; i < n; ++i, adA += step, adB += step) {
        smem_and(adA, mA);
        smem_and(adB, mB);
    }
    if (nA > n) smem_and(adA, mA);
    if (nB > n) smem_and(adB, mB);
}


// Carried sieve offsets (per-CTA rows, ~92 MB at N = 1e12): L2 accesses with an
// evict_last policy so the rows stay resident in L2 across tiles instead of making
// a DRAM round trip per tile (plain .cg accesses: DRAM reads 9.7 vs 2.0 GB per
// 2^36-integer launch).
__device__ __forceinline__ uint64_t carry_policy()
{
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t carry_ld(const uint32_t *p, uint64_t pol)
{
    uint32_t v;
    asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void carry_st(uint32_t *p, uint32_t v, uint64_t pol)
{
    asm volatile("st.global.cg.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}


// K-SIEVE of one tile's two class windows by the whole CTA; ends WITHOUT a barrier
template <bool DEF_TILE, int KB = 2, int KB2 = 2, bool NOCARRY = false>
__device__ __forceinline__ void sieve6_window(uint32_t *wA, uint32_t *wB, int64_t g0, uint32_t nw, const SievePrimes &sp,
                              Carry6 *cy, const MedSched &ms, uint32_t i_b2, uint32_t i_b1,
                              const uint32_t *__restrict__ lm, int64_t lg0, uint64_t lstride, int tid)
{
    const uint32_t lane = (uint32_t)tid & 31;
    constexpr int nt = kThreads;
    const uint32_t sA = smem_addr(wA), sB = smem_addr(wB);
    if (!NOCARRY && cy->init) {
        // first tile of this CTA's run: carried offsets of the steady primes by modulo
        const int64_t m_lo0 = g0 * 32, m_hi0 = (g0 + (int64_t)nw) * 32;
        const uint64_t ipol = carry_policy();
        for (uint32_t pi = sp.i_med + tid; pi < cy->n_steady; pi += nt) {
            const uint4 k = __ldg(sp.pk + pi);
            uint32_t oa, ob;
            first_hits6(k.x, k.z, k.w, __ldg(sp.magic + pi), m_lo0, m_hi0, oa, ob);
            carry_st(cy->off + pi, oa, ipol);
            carry_st(cy->off + cy->stride + pi, ob, ipol);
        }
        __syncthreads();
    }
    // Phase T: primes 5..31 by shifted word patterns, per-thread incremental phases
    {
        int64_t g = g0 + tid;
        const uint64_t gg = g < 0 ? 0 : (uint64_t)g;
#define GB_PH(P)                                                                                   \
    int a##P = (int)((rA_of(P) + 32u * P - (32u * (uint32_t)(gg % P)) % P) % P);                   \
    int b##P = (int)((rB_of(P) + 32u * P - (32u * (uint32_t)(gg % P)) % P) % P);
        GB_PH(5) GB_PH(7) GB_PH(11) GB_PH(13) GB_PH(17) GB_PH(19) GB_PH(23) GB_PH(29) GB_PH(31)
#undef GB_PH
        for (int64_t i = tid; i < (int64_t)nw; i += nt, g += nt) {
            uint32_t va = 0, vb = 0;
            if (g >= 0) {
                const uint32_t ca = (Tiny<5>::value << a5) | (Tiny<7>::value << a7) | (Tiny<11>::value << a11) |
                                    (Tiny<13>::value << a13) | (Tiny<17>::value << a17) |
                                    (Tiny<19>::value << a19) | (Tiny<23>::value << a23) |
                                    (Tiny<29>::value << a29) | (Tiny<31>::value << a31);
                const uint32_t cb = (Tiny<5>::value << b5) | (Tiny<7>::value << b7) | (Tiny<11>::value << b11) |
                                    (Tiny<13>::value << b13) | (Tiny<17>::value << b17) |
                                    (Tiny<19>::value << b19) | (Tiny<23>::value << b23) |
                                    (Tiny<29>::value << b29) | (Tiny<31>::value << b31);
                va = ~ca;
                vb = ~cb;
                if (g == 0) {
                    // restore the tiny primes themselves: A (6m+1): 7, 13, 19, 31 at m = 1, 2, 3, 5;
                    // B (6m+5): 5, 11, 17, 23, 29 at m = 0..4; and 1 = 6*0+1 is not prime
                    va = (va | 0x2Eu) & ~1u;
                    vb |= 0x1Fu;
                }
                if (lm) {   // K-LARGE mask of this chunk (primes above the carried range)
                    va &= __ldcs(lm + (g - lg0));          // read once: evict-first
                    vb &= __ldcs(lm + lstride + (g - lg0));
                }
            }
            wA[i] = va;
            wB[i] = vb;
            if (g >= 0) {
#define GB_ADV(P)                                    \
    a##P -= (int)((32u * nt) % P); if (a##P < 0) a##P += P; \
    b##P -= (int)((32u * nt) % P); if (b##P < 0) b##P += P;
                GB_ADV(5) GB_ADV(7) GB_ADV(11) GB_ADV(13) GB_ADV(17) GB_ADV(19) GB_ADV(23) GB_ADV(29)
                GB_ADV(31)
#undef GB_ADV
            } else if (g + nt >= 0) {
                const uint64_t g2 = (uint64_t)(g + nt);
#define GB_RE(P)                                                                     \
    a##P = (int)((rA_of(P) + 32u * P - (32u * (uint32_t)(g2 % P)) % P) % P);        \
    b##P = (int)((rB_of(P) + 32u * P - (32u * (uint32_t)(g2 % P)) % P) % P);
                GB_RE(5) GB_RE(7) GB_RE(11) GB_RE(13) GB_RE(17) GB_RE(19) GB_RE(23) GB_RE(29) GB_RE(31)
#undef GB_RE
            }
        }
    }
    const int64_t m_lo = g0 * 32;
    const int64_t m_hi = (g0 + (int64_t)nw) * 32;
    const uint32_t nbits = nw * 32;
    const uint32_t ns = cy->n_steady;
    // medium primes (31 < p <= kWarpPrimeMax): both first hits per prime into shared
    // memory (carried or by modulo), one thread per prime; then one warp per prime,
    // handed out dynamically in ascending order (largest work first).
    const uint32_t m_end = sp.i_big < sp.n_use ? sp.i_big : sp.n_use;
    __shared__ uint32_t sh_mA[kMedMax], sh_mB[kMedMax];
    __shared__ uint16_t sh_hA[kMedMax], sh_hB[kMedMax];     // hits per class in this window
    for (uint32_t pi = sp.i_med + tid; pi < m_end; pi += nt) {
        const uint4 k = __ldg(sp.pk + pi);        // p, kTileM mod p, rA, rB
        uint32_t oa = 0xFFFFFFFFu, ob = 0xFFFFFFFFu;
        const bool carried = !NOCARRY && pi < cy->n_carry;
        if (!NOCARRY && pi < ns) {
            oa = cy->off[pi];
            ob = cy->off[cy->stride + pi];
            const uint32_t tm = tile_mod<DEF_TILE>(cy, k);
            cy->off[pi] = oa >= tm ? oa - tm : oa + k.x - tm;
            cy->off[cy->stride + pi] = ob >= tm ? ob - tm : ob + k.x - tm;
        } else {
            const int64_t mmin = (int64_t)(((uint64_t)k.x * k.x - 1) / 6);
            if (mmin < m_hi) {
                if (carried && cy->have_prev && mmin < m_hi - (int64_t)cy->tile_m) {
                    oa = cy->off[pi];
                    ob = cy->off[cy->stride + pi];
                } else {
                    const uint64_t mg = __ldg(sp.magic + pi);
                    first_hits6(k.x, k.z, k.w, mg, m_lo, m_hi, oa, ob);
                }
                if (carried) {
                    const uint32_t tm = tile_mod<DEF_TILE>(cy, k);
                    cy->off[pi] = next_off6(oa, k.x, tm, cy->tile_m);
                    cy->off[cy->stride + pi] = next_off6(ob, k.x, tm, cy->tile_m);
                }
            }
        }
        sh_mA[pi - sp.i_med] = oa;
        sh_mB[pi - sp.i_med] = ob;
        sh_hA[pi - sp.i_med] = (uint16_t)(oa < nbits ? (nbits - oa + k.x - 1) / k.x : 0);
        sh_hB[pi - sp.i_med] = (uint16_t)(ob < nbits ? (nbits - ob + k.x - 1) / k.x : 0);
    }
    __syncthreads();
    // one warp per medium prime: the host's LPT schedule (longest work first onto
    // the least-loaded warp) gives every sieving warp the same share, no atomics
    {
        const uint32_t warp = (uint32_t)tid >> 5;
        const uint32_t k0 = __ldg(ms.off + warp), k1 = __ldg(ms.off + warp + 1);
        for (uint32_t k = k0; k < k1; ++k) {
            const uint32_t rel = __ldg(ms.idx + k);
            const uint32_t pi = sp.i_med + rel;
            if (pi >= m_end) continue;
            const uint32_t p = __ldg(sp.primes + pi);
            mark_progression2(sA, sh_mA[rel], sh_hA[rel], sB, sh_mB[rel], sh_hB[rel], p, lane);
        }
    }
    // large primes: one thread per prime.  Steady primes: kB in flight per thread.
    const uint32_t b_begin = sp.i_big > sp.i_med ? sp.i_big : sp.i_med;
    const uint32_t s_end = ns > b_begin ? (ns < sp.n_use ? ns : sp.n_use) : b_begin;
    const uint32_t b2 = i_b2 < b_begin ? b_begin : (i_b2 < s_end ? i_b2 : s_end);
    const uint32_t b1 = i_b1 < b2 ? b2 : (i_b1 < s_end ? i_b1 : s_end);
    const uint64_t cpol = carry_policy();
    uint32_t *__restrict__ cA = cy->off;                 // this CTA's carry row, class A
    const uint4 *__restrict__ pkp = sp.pk;
    // Steady primes carry only their class-A offset: both progressions step by the
    // same p per tile, so ob = oa + (rB - rA) mod p (both offsets are residues in
    // [0, p) once p^2 lies below the window) -- half the carry-row traffic.
    constexpr int kB = KB;            // steady primes in flight per thread (1 or 4: slower)
    // steady primes with p <= full window / 2: hit loops (>= 2 hits per class)
    for (uint32_t w0 = b_begin + (tid & ~31u); w0 < b2; w0 += kB * nt) {   // warp-uniform trips
        const uint32_t p0 = w0 + lane;
        uint2 pt[kB];
        uint32_t oa[kB], ob[kB];
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const uint32_t pi = p0 + k * nt;
            if (pi < b2) {
                const uint4 q = __ldg(pkp + pi);
                if constexpr (NOCARRY) {
                    pt[k] = make_uint2(q.x, 0);
                    steady_first(q, m_lo, __ldg(sp.magic + pi), oa[k], ob[k]);
                } else {
                    pt[k] = make_uint2(q.x, tile_mod<DEF_TILE>(cy, q));
                    oa[k] = carry_ld(cA + pi, cpol);
                    ob[k] = class_b_off(oa[k], q);
                }
            } else {
                pt[k] = make_uint2(1, 0);
                oa[k] = ob[k] = nbits;
            }
        }
#pragma unroll
        for (int k = 0; k < kB; ++k) {
            const uint32_t p = pt[k].x, tm = pt[k].y;
            {   // both classes in one loop (hit counts differ by at most one)
                uint32_t ba = oa[k], bb = ob[k];
                for (; ba + p < nbits && bb + p < nbits; ba += 2 * p, bb += 2 * p) {   // 2 hits per class
                    clear_bit(sA, ba);
                    clear_bit(sB, bb);
                    clear_bit(sA, ba + p);
                    clear_bit(sB, bb + p);
                }
                for (; ba < nbits && bb < nbits; ba += p, bb += p) {
                    clear_bit(sA, ba);
                    clear_bit(sB, bb);
                }
                for (; ba < nbits; ba += p) clear_bit(sA, ba);
                for (; bb < nbits; bb += p) clear_bit(sB, bb);
            }
            const uint32_t pi = p0 + k * nt;
            if (!NOCARRY && pi < b2) carry_st(cA + pi, oa[k] >= tm ? oa[k] - tm : oa[k] + p - tm, cpol);
        }
        __syncwarp();   // reconverge: the per-lane hit loops diverge
    }
    // steady primes with window/2 < p <= window: at most 2 hits per class, predicated
    constexpr int kB2 = KB2;          // primes in flight per thread: 4 in the out-of-line sieve (below 2^42:
                                      // 29.07 vs 29.34 ms), 2 inlined (4: +1.4% at 4e18; 8: slower)
    for (uint32_t w0 = b2 + (tid & ~31u); w0 < b1; w0 += kB2 * nt) {
        const uint32_t p0 = w0 + lane;
        uint32_t pp[kB2], tt[kB2], oa[kB2], ob[kB2];
#pragma unroll
        for (int k = 0; k < kB2; ++k) {
            const uint32_t pi = p0 + k * nt;
            if (pi < b1) {
                const uint4 q = __ldg(pkp + pi);
                pp[k] = q.x;
                if constexpr (NOCARRY) {
                    tt[k] = 0;
                    steady_first(q, m_lo, __ldg(sp.magic + pi), oa[k], ob[k]);
                } else {
                    tt[k] = tile_mod<DEF_TILE>(cy, q);
                    oa[k] = carry_ld(cA + pi, cpol);
                    ob[k] = class_b_off(oa[k], q);
                }
            } else {
                pp[k] = nbits; tt[k] = 0;
                oa[k] = ob[k] = nbits;
            }
        }
#pragma unroll
        for (int k = 0; k < kB2; ++k) {
            const uint32_t p = pp[k], tm = tt[k];
            if (oa[k] < nbits) clear_bit(sA, oa[k]);
            if (oa[k] + p < nbits) clear_bit(sA, oa[k] + p);
            if (ob[k] < nbits) clear_bit(sB, ob[k]);
            if (ob[k] + p < nbits) clear_bit(sB, ob[k] + p);
            const uint32_t pi = p0 + k * nt;
            if (!NOCARRY && pi < b1) carry_st(cA + pi, oa[k] >= tm ? oa[k] - tm : oa[k] + p - tm, cpol);
        }
    }
    // steady primes with p > a full window: at most 1 hit per class
    for (uint32_t w0 = b1 + (tid & ~31u); w0 < s_end; w0 += kB2 * nt) {
        const uint32_t p0 = w0 + lane;
        uint32_t pp[kB2], tt[kB2], oa[kB2], ob[kB2];
#pragma unroll
        for (int k = 0; k < kB2; ++k) {
            const uint32_t pi = p0 + k * nt;
            if (pi < s_end) {
                const uint4 q = __ldg(pkp + pi);
                pp[k] = q.x;
                if constexpr (NOCARRY) {
                    tt[k] = 0;
                    steady_first(q, m_lo, __ldg(sp.magic + pi), oa[k], ob[k]);
                } else {
                    tt[k] = tile_mod<DEF_TILE>(cy, q);
                    oa[k] = carry_ld(cA + pi, cpol);
                    ob[k] = class_b_off(oa[k], q);
                }
            } else {
                pp[k] = nbits; tt[k] = 0;
                oa[k] = ob[k] = nbits;
            }
        }
#pragma unroll
        for (int k = 0; k < kB2; ++k) {
            const uint32_t p = pp[k], tm = tt[k];
            if (oa[k] < nbits) clear_bit(sA, oa[k]);
            if (ob[k] < nbits) clear_bit(sB, ob[k]);
            const uint32_t pi = p0 + k * nt;
            if (!NOCARRY && pi < s_end) carry_st(cA + pi, oa[k] >= tm ? oa[k] - tm : oa[k] + p - tm, cpol);
        }
    }
    for (uint32_t pi = s_end + tid; pi < sp.n_use; pi += nt) {
        const uint4 k = __ldg(sp.pk + pi);
        const int64_t mmin = (int64_t)(((uint64_t)k.x * k.x - 1) / 6);
        if (mmin >= m_hi) break;
        const bool carried = !NOCARRY && pi < cy->n_carry;
        uint32_t oa, ob;
        if (carried && cy->have_prev && mmin < m_hi - (int64_t)cy->tile_m) {
            oa = cy->off[pi];
            ob = cy->off[cy->stride + pi];
        } else {
            const uint64_t mg = __ldg(sp.magic + pi);
            first_hits6(k.x, k.z, k.w, mg, m_lo, m_hi, oa, ob);
        }
        for (uint32_t b = oa; b < nbits; b += k.x) clear_bit(sA, b);
        for (uint32_t b = ob; b < nbits; b += k.x) clear_bit(sB, b);
        if (carried) {
            const uint32_t tm = tile_mod<DEF_TILE>(cy, k);
            cy->off[pi] = next_off6(oa, k.x, tm, cy->tile_m);
            cy->off[cy->stride + pi] = next_off6(ob, k.x, tm, cy->tile_m);
        }
    }
}

// The sieve as its own function (own register allocation, called once per tile):
// below 2^42 the marking code then compiles without the sieve's pressure (29.31 vs
// 29.51 ms at 1e12); in the K-LARGE regime inlined (93.05 vs 93.76 ms at 4e18) and
// carry-free (steady offsets by modulo per tile: 84.6 vs 90.5 ms; below 2^42 the
// carry rows stay L2-resident and win, 29.0 vs 29.9 ms).
template <bool DEF_TILE>
__device__ __noinline__ void sieve6_window_call(uint32_t *wA, uint32_t *wB, int64_t g0, uint32_t nw,
                                                const SievePrimes &sp, Carry6 *cy, const MedSched &ms,
                                                uint32_t i_b2, uint32_t i_b1, const uint32_t *__restrict__ lm,
                                                int64_t lg0, uint64_t lstride, int tid)
{
    sieve6_window<DEF_TILE, 2, 4, false>(wA, wB, g0, nw, sp, cy, ms, i_b2, i_b1, lm, lg0, lstride, tid);
}
template <bool DEF_TILE, bool OUTLINE>
__device__ __forceinline__ void sieve6(uint32_t *wA, uint32_t *wB, int64_t g0, uint32_t nw, const SievePrimes &sp,
                                       Carry6 *cy, const MedSched &ms, uint32_t i_b2, uint32_t i_b1,
                                       const uint32_t *__restrict__ lm, int64_t lg0, uint64_t lstride, int tid)
{
    if constexpr (OUTLINE) sieve6_window_call<DEF_TILE>(wA, wB, g0, nw, sp, cy, ms, i_b2, i_b1, lm, lg0, lstride, tid);
    else sieve6_window<DEF_TILE, 2, 2, true>(wA, wB, g0, nw, sp, cy, ms, i_b2, i_b1, lm, lg0, lstride, tid);
}

// ---------------------------------------------------------------------------
// accumulators of the verify kernel: per-CTA, in shared memory (shared atomics:
// once per round for the evens, per tile for the histogram share of sum p_min,
// else only on the cold paths) -- the marking loops hold no accumulator registers
// and pass no accumulator by reference to the out-of-line phase-2 batches
// ---------------------------------------------------------------------------
struct CtaAcc {
    unsigned long long evens, fast_unres, unres, sum, praw, first_unres;
    unsigned long long key;    // largest make_key(p_min, n)
};

// one lane's (p, n) max-key candidate (p = 0: none); the whole warp calls it
__device__ __forceinline__ void warp_note_key(CtaAcc *acc, uint64_t p, uint64_t n, uint64_t origin, int lane)
{
    const uint64_t key = p ? make_key(p, n, origin) : 0;
    const uint32_t hi = __reduce_max_sync(FULL, (uint32_t)(key >> 32));
    const uint32_t lo = __reduce_max_sync(FULL, (uint32_t)(key >> 32) == hi ? (uint32_t)key : 0u);
    const uint64_t k = ((uint64_t)hi << 32) | lo;
    if (lane == 0 && k) atomicMax(&acc->key, (unsigned long long)k);
    if (p >= GB_KEY_PMAX) atomicMax(&acc->praw, (unsigned long long)p);
}

// a single lane's note (cold paths: specials, fallback)
__device__ __forceinline__ void lane_note_key(CtaAcc *acc, uint64_t p, uint64_t n, uint64_t origin)
{
    atomicMax(&acc->key, (unsigned long long)make_key(p, n, origin));
    if (p >= GB_KEY_PMAX) atomicMax(&acc->praw, (unsigned long long)p);
}

// ---------------------------------------------------------------------------
// the inverted marking loop on one U word per lane
// ---------------------------------------------------------------------------
struct Lane6 {
    const uint32_t *wa, *wb;   // class A / B window word aligned with this U word
    uint32_t U;                // unresolved evens of the word
    uint32_t lb;               // 1 + index of the last 8-candidate block with a hit (0 = none)
    uint32_t lu;               // U at the start of that block
    uint32_t *dump_w;          // dump entry of bit 0 (bit b at dump_w[3b]) -- DUMP only
};

template <int A, int J, bool DUMP>
__device__ __forceinline__ uint32_t mark_step(Lane6 &m)
{
    constexpr uint32_t P = kTab[A / 2].p[J];
    constexpr Trans T = trans(A, P);
    constexpr int WA = (int)(T.shift >> 5);
    constexpr uint32_t WB = T.shift & 31;
    const uint32_t *src = T.src ? m.wb : m.wa;
    const uint32_t S = __funnelshift_l(src[-(WA + 1)], src[-WA], WB);
    if constexpr (DUMP) {
        uint32_t x = m.U & S;                 // n resolved now: n - P prime, no smaller p worked
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            m.dump_w[3 * b] = P;
        }
    }
    m.U &= ~S;
    return __popc(m.U);                       // A_J: still unresolved after P (see hist8)
}

// Per-warp counts of 8 candidates -> class histogram (two counts per REDUX: 16-bit
// fields, per warp and candidate <= 32 kW 32 = 3072).  The counts are A_J = evens
// still unresolved AFTER candidate J (one AND-NOT + POPC per word and candidate,
// no separate "resolved now" word); h[J] accumulates A_J and h[-1] the evens that
// enter the table, so flush_hist takes hist[J] = A_{J-1} - A_J.
__device__ __forceinline__ void hist8(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t c4,
                                      uint32_t c5, uint32_t c6, uint32_t c7, uint32_t *h, int lane)
{
    const uint32_t t0 = __reduce_add_sync(FULL, c0 + (c1 << 16));
    const uint32_t t1 = __reduce_add_sync(FULL, c2 + (c3 << 16));
    const uint32_t t2 = __reduce_add_sync(FULL, c4 + (c5 << 16));
    const uint32_t t3 = __reduce_add_sync(FULL, c6 + (c7 << 16));
    const uint32_t ts = (lane & 4) ? ((lane & 2) ? t3 : t2) : ((lane & 2) ? t1 : t0);
    const uint32_t v = (lane & 1) ? (ts >> 16) : (ts & 0xffffu);
    if (lane < 8 && v) atomicAdd(h + lane, v);
}

template <int A, int J, bool DUMP>
__device__ __forceinline__ void block8(Lane6 &m, uint32_t *h, int lane)
{
    const uint32_t Ub = m.U;
    const uint32_t c0 = mark_step<A, J + 0, DUMP>(m);
    const uint32_t c1 = mark_step<A, J + 1, DUMP>(m);
    const uint32_t c2 = mark_step<A, J + 2, DUMP>(m);
    const uint32_t c3 = mark_step<A, J + 3, DUMP>(m);
    const uint32_t c4 = mark_step<A, J + 4, DUMP>(m);
    const uint32_t c5 = mark_step<A, J + 5, DUMP>(m);
    const uint32_t c6 = mark_step<A, J + 6, DUMP>(m);
    const uint32_t c7 = mark_step<A, J + 7, DUMP>(m);
    if (m.U != Ub) { m.lb = J / 8 + 1; m.lu = Ub; }
    hist8(c0, c1, c2, c3, c4, c5, c6, c7, h + J, lane);
}

// ---- phase 1 with kW words per lane (words li, li + 32, ..., li + 32(kW-1)) ----
constexpr int kW = 3;            // phase-1 words per lane (2: slower)
static_assert(kW * 32 * 32 < 65536, "16-bit packed per-warp counts");
static_assert(31 + 32 * kW <= kQueue, "survivor queue capacity");

struct LaneQ {
    const uint32_t *wa, *wb;   // class A / B window words aligned with word 0 (word k at +32k)
    uint32_t U[kW];
    uint32_t lb[kW], lu[kW];   // TRACK: last block with a hit and U at its start
    uint32_t *dump0;           // DUMP: dump entry of bit 0 of word 0 (word k at +3072k, bit b at +3b)
};

template <int A, int J, bool DUMP>
__device__ __forceinline__ void qstep(LaneQ &m, int k)
{
    constexpr uint32_t P = kTab[A / 2].p[J];
    constexpr Trans T = trans(A, P);
    constexpr int WA = (int)(T.shift >> 5);
    constexpr uint32_t WB = T.shift & 31;
    const uint32_t *src = (T.src ? m.wb : m.wa) + 32 * k;
    const uint32_t S = __funnelshift_l(src[-(WA + 1)], src[-WA], WB);
    if constexpr (DUMP) {
        uint32_t x = m.U[k] & S;
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            m.dump0[3072 * k + 3 * b] = P;
        }
    }
    m.U[k] &= ~S;
}

// A_J of the lane's kW = 3 words with 2 POPC instead of 3: a carry-save full adder
// (sum = a ^ b ^ c, carry = maj(a, b, c): two LOP3) gives popc(a) + popc(b) + popc(c)
// = popc(sum) + 2 popc(carry).  POPC issues at 16 lanes/clk/SM (a quarter of LOP3,
// profiles/peaks_int.json) through the MIO queue the window loads also use: it,
// not the ALU, bounds the marking loops (mio throttle, profiles/r02b_*).
template <int A, int J, bool DUMP>
__device__ __forceinline__ uint32_t qprime(LaneQ &m)
{
    static_assert(kW == 3, "carry-save count of three words");
#pragma unroll
    for (int k = 0; k < kW; ++k) qstep<A, J, DUMP>(m, k);
    const uint32_t x = m.U[0] ^ m.U[1] ^ m.U[2];
    const uint32_t y = (m.U[0] & m.U[1]) | (m.U[2] & (m.U[0] | m.U[1]));
    return __popc(x) + 2 * __popc(y);
}

template <int A, int J, bool DUMP, bool TRACK>
__device__ __forceinline__ void block8q(LaneQ &m, uint32_t *h, int lane)
{
    uint32_t Ub[kW];
    if constexpr (TRACK) {
#pragma unroll
        for (int k = 0; k < kW; ++k) Ub[k] = m.U[k];
    }
    const uint32_t c0 = qprime<A, J + 0, DUMP>(m);
    const uint32_t c1 = qprime<A, J + 1, DUMP>(m);
    const uint32_t c2 = qprime<A, J + 2, DUMP>(m);
    const uint32_t c3 = qprime<A, J + 3, DUMP>(m);
    const uint32_t c4 = qprime<A, J + 4, DUMP>(m);
    const uint32_t c5 = qprime<A, J + 5, DUMP>(m);
    const uint32_t c6 = qprime<A, J + 6, DUMP>(m);
    const uint32_t c7 = qprime<A, J + 7, DUMP>(m);
    if constexpr (TRACK) {
#pragma unroll
        for (int k = 0; k < kW; ++k)
            if (m.U[k] != Ub[k]) { m.lb[k] = J / 8 + 1; m.lu[k] = Ub[k]; }
    }
    hist8(c0, c1, c2, c3, c4, c5, c6, c7, h + J, lane);   // per warp and prime <= 32 kW 32 hits
}

template <int A, int J, int JEND, bool DUMP, bool TRACK>
__device__ __forceinline__ void phase1q(LaneQ &m, uint32_t *h, int lane)
{
    if constexpr (J < JEND) {
        block8q<A, J, DUMP, TRACK>(m, h, lane);
        phase1q<A, J + 8, JEND, DUMP, TRACK>(m, h, lane);
    }
}

// ---- phase 1b: the words still unresolved after candidate kC1, compacted to S
// words per lane (a round's survivors gathered through the warp's queue area), so
// candidates kC1 .. kP1-1 run only on live words.  Word k of a lane has its own
// window position li[k].
constexpr int kC1 = 32;          // compaction point (40: +0.3% at 1e12; 24 / 48: slower)
constexpr int kC1L = 40;         // the same in the K-LARGE regime (32: +4.9% at 4e18, 48: +1.0%)
static_assert(kC1 % 8 == 0 && kC1 <= kP1 && kC1L % 8 == 0 && kC1L <= kP1L, "compaction point on a block boundary");

template <int S>
struct LaneR {
    const uint32_t *wa[S], *wb[S];  // class A / B window word aligned with U word k
    uint32_t U[S];
    uint32_t lb[S], lu[S];
    uint32_t li[S];                 // word index within the tile
    uint32_t *dump[S];              // DUMP: dump entry of bit 0 of word k (bit b at +3b)
};

template <int A, int J, int S, bool DUMP>
__device__ __forceinline__ uint32_t rstep(LaneR<S> &m, int k)
{
    constexpr uint32_t P = kTab[A / 2].p[J];
    constexpr Trans T = trans(A, P);
    constexpr int WA = (int)(T.shift >> 5);
    constexpr uint32_t WB = T.shift & 31;
    const uint32_t *src = T.src ? m.wb[k] : m.wa[k];
    const uint32_t S_ = __funnelshift_l(src[-(WA + 1)], src[-WA], WB);
    if constexpr (DUMP) {
        uint32_t x = m.U[k] & S_;
        while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            m.dump[k][3 * b] = P;
        }
    }
    m.U[k] &= ~S_;
    return __popc(m.U[k]);
}

template <int A, int J, int S, bool DUMP>
__device__ __forceinline__ uint32_t rprime(LaneR<S> &m)
{
    uint32_t c = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) c += rstep<A, J, S, DUMP>(m, k);
    return c;
}

template <int A, int J, int S, bool DUMP, bool TRACK>
__device__ __forceinline__ void block8r(LaneR<S> &m, uint32_t *h, int lane)
{
    uint32_t Ub[S];
    if constexpr (TRACK) {
#pragma unroll
        for (int k = 0; k < S; ++k) Ub[k] = m.U[k];
    }
    const uint32_t c0 = rprime<A, J + 0, S, DUMP>(m);
    const uint32_t c1 = rprime<A, J + 1, S, DUMP>(m);
    const uint32_t c2 = rprime<A, J + 2, S, DUMP>(m);
    const uint32_t c3 = rprime<A, J + 3, S, DUMP>(m);
    const uint32_t c4 = rprime<A, J + 4, S, DUMP>(m);
    const uint32_t c5 = rprime<A, J + 5, S, DUMP>(m);
    const uint32_t c6 = rprime<A, J + 6, S, DUMP>(m);
    const uint32_t c7 = rprime<A, J + 7, S, DUMP>(m);
    if constexpr (TRACK) {
#pragma unroll
        for (int k = 0; k < S; ++k)
            if (m.U[k] != Ub[k]) { m.lb[k] = J / 8 + 1; m.lu[k] = Ub[k]; }
    }
    hist8(c0, c1, c2, c3, c4, c5, c6, c7, h + J, lane);
}

template <int A, int J, int JEND, int S, bool DUMP, bool TRACK>
__device__ __forceinline__ void phase1r(LaneR<S> &m, uint32_t *h, int lane)
{
    if constexpr (J < JEND) {
        block8r<A, J, S, DUMP, TRACK>(m, h, lane);
        phase1r<A, J + 8, JEND, S, DUMP, TRACK>(m, h, lane);
    }
}

// phase 2: candidates [J, kK) for one word per lane, warp exit test every 8
template <int A, int J, bool DUMP>
__device__ __forceinline__ void phase2(Lane6 &m, uint32_t *h, int lane)
{
    if constexpr (J < kK) {
        if (!__any_sync(FULL, m.U != 0)) return;
        block8<A, J, DUMP>(m, h, lane);
        phase2<A, J + 8, DUMP>(m, h, lane);
    }
}

// max p_min among the unrolled hits: replay the last block with a hit (from the U
// saved at its start), only lanes holding the warp's latest block, and only when
// that block can raise this warp's running maximum best_p
template <int A>
__device__ __forceinline__ void replay_key(const Lane6 &m, uint64_t u, const VerifyArgs &a,
                                           uint32_t &best_p, CtaAcc *acc)
{
    const uint32_t bstar = __reduce_max_sync(FULL, m.lb);
    if (bstar == 0) return;
    const ClassTable &T = c_tab[A / 2];
    if (T.p[8 * bstar - 1] < best_p) return;
    const uint32_t jr = (bstar - 1) * 8;
    best_p = max(best_p, T.p[jr]);
    uint32_t lp = 0, lbits = 0;
    if (m.lb == bstar) {
        uint32_t x = m.lu;
        for (int i = 0; i < 8; ++i) {
            const uint32_t p = T.p[jr + i];
            const Trans t = trans(A, p);
            const uint32_t *src = t.src ? m.wb : m.wa;
            const int wa = (int)(t.shift >> 5);
            const uint32_t S = __funnelshift_l(src[-wa - 1], src[-wa], t.shift & 31);
            const uint32_t nw = x & S;
            x ^= nw;
            if (nw) { lp = p; lbits = nw; }
        }
    }
    const uint64_t n = lp ? 6 * (u * 32 + (uint64_t)(__ffs(lbits) - 1)) + A : 0;
    warp_note_key(acc, lp, n, a.origin, threadIdx.x & 31);
}

template <int A>
__device__ __forceinline__ void replay_key_q(const LaneQ &m, uint64_t u0w, const VerifyArgs &a, uint32_t &best_p,
                                             CtaAcc *acc)
{
    uint32_t mx = 0;
#pragma unroll
    for (int k = 0; k < kW; ++k) mx = max(mx, m.lb[k]);
    const uint32_t bstar = __reduce_max_sync(FULL, mx);
    if (bstar == 0) return;
    const ClassTable &T = c_tab[A / 2];
    if (T.p[8 * bstar - 1] < best_p) return;
    const uint32_t jr = (bstar - 1) * 8;
    best_p = max(best_p, T.p[jr]);
    uint32_t bp = 0;
    uint64_t bn = 0;
#pragma unroll
    for (int k = 0; k < kW; ++k) {
        if (m.lb[k] != bstar) continue;
        uint32_t x = m.lu[k], lp = 0, lbits = 0;
        for (int i = 0; i < 8; ++i) {
            const uint32_t p = T.p[jr + i];
            const Trans t = trans(A, p);
            const uint32_t *src = (t.src ? m.wb : m.wa) + 32 * k;
            const int wa = (int)(t.shift >> 5);
            const uint32_t S = __funnelshift_l(src[-wa - 1], src[-wa], t.shift & 31);
            const uint32_t nw = x & S;
            x ^= nw;
            if (nw) { lp = p; lbits = nw; }
        }
        const uint64_t n = 6 * ((u0w + 32 * k) * 32 + (uint64_t)(__ffs(lbits) - 1)) + A;
        if (lp > bp || (lp == bp && n < bn)) { bp = lp; bn = n; }
    }
    warp_note_key(acc, bp, bn, a.origin, threadIdx.x & 31);
}

template <int A, int S>
__device__ __forceinline__ void replay_key_r(const LaneR<S> &m, uint64_t u0, const VerifyArgs &a, uint32_t &best_p,
                                             CtaAcc *acc)
{
    uint32_t mx = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) mx = max(mx, m.lb[k]);
    const uint32_t bstar = __reduce_max_sync(FULL, mx);
    if (bstar == 0) return;
    const ClassTable &T = c_tab[A / 2];
    if (T.p[8 * bstar - 1] < best_p) return;
    const uint32_t jr = (bstar - 1) * 8;
    best_p = max(best_p, T.p[jr]);
    uint32_t bp = 0;
    uint64_t bn = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
        if (m.lb[k] != bstar) continue;
        uint32_t x = m.lu[k], lp = 0, lbits = 0;
        for (int i = 0; i < 8; ++i) {
            const uint32_t p = T.p[jr + i];
            const Trans t = trans(A, p);
            const uint32_t *src = t.src ? m.wb[k] : m.wa[k];
            const int wa = (int)(t.shift >> 5);
            const uint32_t S_ = __funnelshift_l(src[-wa - 1], src[-wa], t.shift & 31);
            const uint32_t nw = x & S_;
            x ^= nw;
            if (nw) { lp = p; lbits = nw; }
        }
        const uint64_t n = 6 * ((u0 + m.li[k]) * 32 + (uint64_t)(__ffs(lbits) - 1)) + A;
        if (lp > bp || (lp == bp && n < bn)) { bp = lp; bn = n; }
    }
    warp_note_key(acc, bp, bn, a.origin, threadIdx.x & 31);
}

// candidates past the unrolled tables (runtime loop over the resident list, class
// filtered), then the exhaustive on-GPU fallback; folds the word into acc
template <int A, bool DUMP>
__device__ __forceinline__ void finish_word(uint32_t U, uint32_t j0, const uint32_t *wa,
                                            const uint32_t *wb, uint64_t u, uint32_t *sh_hist,
                                            const VerifyArgs &a, CtaAcc *acc, int lane)
{
    uint32_t lastp = 0, lastb = 0;
    for (uint32_t j = j0; j < a.n_cand; ++j) {
        if (!__any_sync(FULL, U != 0)) break;
        const uint32_t p = __ldg(a.sp.primes + j);
        const Trans t = trans(A, p);
        if (!t.ok) continue;
        const uint32_t *src = t.src ? wb : wa;
        const int wsh = (int)(t.shift >> 5);
        const uint32_t S = __funnelshift_l(src[-wsh - 1], src[-wsh], t.shift & 31);
        const uint32_t nw = U & S;
        const uint32_t c = __popc(nw);
        if (nw) {
            U ^= nw;
            atomicAdd(&acc->sum, (unsigned long long)c * p);
            lastp = p; lastb = nw;
            if (DUMP) {
                uint32_t x = nw;
                while (x) {
                    const int b = __ffs(x) - 1;
                    x &= x - 1;
                    a.dump[(6 * (u * 32 + b) + A - a.lo_e) / 2] = p;
                }
            }
        }
        const uint32_t tot = __reduce_add_sync(FULL, c);
        if (lane == 0 && tot) hist_add(sh_hist, a.result, j + 2, tot);
    }
    warp_note_key(acc, lastp, lastp ? 6 * (u * 32 + (uint64_t)(__ffs(lastb) - 1)) + A : 0, a.origin, lane);
    if (U) atomicAdd(&acc->fast_unres, (unsigned long long)__popc(U));
    while (true) {
        const uint32_t m = __ballot_sync(FULL, U != 0);
        if (!m) break;
        const int L = __ffs(m) - 1;
        const uint32_t lw = __shfl_sync(FULL, U, L);
        const uint64_t uL = __shfl_sync(FULL, u, L);
        const int bit = __ffs(lw) - 1;
        const uint64_t n = 6 * (uL * 32 + (uint64_t)bit) + A;
        const uint64_t p = fallback_scan(n, a.p_fallback, a.cap, a.base_bits, a.R);
        if (lane == L) {
            U &= ~(1u << bit);
            if (p) {
                atomicAdd(&acc->sum, (unsigned long long)p);
                hist_add(sh_hist, a.result, bin_of_prime(p, a.sp.primes, a.n_base), 1);
                lane_note_key(acc, p, n, a.origin);
            } else {
                atomicAdd(&acc->unres, 1ull);
                hist_add(sh_hist, a.result, 0, 1);
                atomicMin(&acc->first_unres, (unsigned long long)n);
            }
            if (DUMP) a.dump[(n - a.lo_e) / 2] = (uint32_t)p;
        }
    }
}

template <int A>
__device__ __forceinline__ uint32_t valid_mask(uint64_t u, const VerifyArgs &a)
{
    const uint64_t mb = u * 32, lo = a.m_lo[A / 2], hi = a.m_hi[A / 2];
    uint32_t U = FULL;
    if (mb < lo) U = (lo - mb >= 32) ? 0u : (U << (lo - mb));
    if (mb + 32 > hi) U &= (hi <= mb) ? 0u : (FULL >> (mb + 32 - hi));
    return U;
}

// n = 4 (class 4, m = 0): p_min = 2, the only even p (reading R2); n = 6 (class 0,
// m = 1): p_min = 3 with q = 3, the one partner the wheel windows do not hold
template <int A, bool DUMP>
__device__ __forceinline__ uint32_t take_special(uint32_t U, uint64_t u, uint32_t *sh_hist,
                                                 const VerifyArgs &a, CtaAcc *acc)
{
    if (u != 0) return U;
    if (A == 4 && (U & 1u)) {
        U &= ~1u;
        atomicAdd(&acc->sum, 2ull);
        atomicAdd(sh_hist + 1, 1u);
        lane_note_key(acc, 2, 4, a.origin);
        if (DUMP) a.dump[(4 - a.lo_e) / 2] = 2;
    }
    if (A == 0 && (U & 2u)) {
        U &= ~2u;
        atomicAdd(&acc->sum, 3ull);
        atomicAdd(sh_hist + 2, 1u);
        lane_note_key(acc, 3, 6, a.origin);
        if (DUMP) a.dump[(6 - a.lo_e) / 2] = 3;
    }
    return U;
}

// Steady primes of the window starting at class word g0 (thread 0): carried and
// p^2 <= 6 m_lo + 1, i.e. the progression started below the window.  If the
// previous tile was not done by this CTA (first tile of its run or of a K-LARGE
// chunk) bit 31 asks sieve6_window to compute their offsets into the carry row
// first, so every such prime still takes the balanced steady loops.  ns_run: the
// running (monotone) count of this CTA.
__device__ __forceinline__ uint32_t steady_count(const Carry6 &cy, int64_t g0, const SievePrimes &sp,
                                                 uint32_t &ns_run)
{
    uint32_t ns = 0;
    const int64_t m_lo = g0 * 32;
    if (m_lo > 0) {
        const uint64_t lim = 6 * (uint64_t)m_lo + 1;
        const uint32_t top = min(cy.n_carry, sp.n_use);
        ns = max(ns_run, sp.i_med);
        if (ns == sp.i_med) {
            uint32_t lo = sp.i_med, hi = top;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                const uint64_t pm = __ldg(sp.primes + mid);
                if (pm * pm <= lim) lo = mid + 1; else hi = mid;
            }
            ns = lo;
        } else {
            while (ns < top) {
                const uint64_t pm = __ldg(sp.primes + ns);
                if (pm * pm > lim) break;
                ++ns;
            }
        }
        ns_run = ns;
    }
    // bit 31: the previous tile was not done here, the carry row must be filled first
    return ns | (cy.have_prev || ns <= sp.i_med ? 0u : 0x80000000u);
}

// dynamic shared memory: class A window | class B window | per-warp survivor queues
extern __shared__ uint32_t g_win[];

struct Shared6 {
    uint32_t hist[kHistSmem];          // bins by prime index (runtime loop, fallback, specials)
    uint32_t histc[3][kK + 1];         // per class: [0] evens entering the table, [J + 1] = A_J (hist8)
    uint32_t wint[kMarkWarps][3];      // per warp and class: interior rounds of this tile (no atomics)
    uint32_t next_round[2];            // per window slot
    uint32_t ns[2];
    uint32_t q_base;      // word offset of the queues in dynamic shared memory
    CtaAcc acc;
};

__device__ __forceinline__ uint32_t *sh_qU(const Shared6 &sh, int warp)
{
    return g_win + sh.q_base + (uint32_t)warp * kQueue;
}
__device__ __forceinline__ uint16_t *sh_qli(const Shared6 &sh, int warp)
{
    return (uint16_t *)(g_win + sh.q_base + kMarkWarps * kQueue) + (uint32_t)warp * kQueue;
}

template <int A, bool DUMP, bool UNROLL, bool INB>
struct ClassWork {
    static constexpr int P1 = INB ? kP1L : kP1;     // phase-1 length and compaction point of this regime
    static constexpr int C1 = INB ? kC1L : kC1;
    // one phase-2 batch of `take` queued words of class A (out of line: called from
    // the round loop and the queue flushes; keeps the hot code small)
    // (everything by value: no local-memory round trip of the caller's state; the
    // queue entries [qn - take, qn) are consumed, the caller lowers qn; returns the
    // updated running max best_p)
    static __device__ __forceinline__ uint32_t batch_body(Shared6 &sh, uint32_t qn, uint32_t take, uint64_t u0,
                                                  const uint32_t *wA, const uint32_t *wB, uint32_t halo,
                                                  const VerifyArgs &a, CtaAcc *acc, uint32_t best_p, int lane,
                                                  int warp)
    {
        const uint32_t e = qn - take;
        uint32_t li = 0, U = 0;
        if ((uint32_t)lane < take) { li = sh_qli(sh, warp)[e + lane]; U = sh_qU(sh, warp)[e + lane]; }
        __syncwarp();
        const uint64_t u = u0 + li;
        Lane6 m;
        m.wa = wA + halo + li;
        m.wb = wB + halo + li;
        m.U = U;
        m.lb = 0; m.lu = 0;
        m.dump_w = DUMP ? a.dump + ((int64_t)(192 * u + A) - (int64_t)a.lo_e) / 2 : nullptr;
        phase2<A, P1, DUMP>(m, sh.histc[A / 2] + 1, lane);
        replay_key<A>(m, u, a, best_p, acc);
        constexpr uint32_t j_next = kTab[A / 2].bin[kK - 1] - 1;   // odd-list index after the table
        finish_word<A, DUMP>(m.U, j_next, m.wa, m.wb, u, sh.hist, a, acc, lane);
        return best_p;
    }
    static __device__ __noinline__ uint32_t batch_call(Shared6 &sh, uint32_t qn, uint32_t take, uint64_t u0,
                                                       const uint32_t *wA, const uint32_t *wB, uint32_t halo,
                                                       const VerifyArgs &a, CtaAcc *acc, uint32_t best_p, int lane,
                                                       int warp)
    {
        return batch_body(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, warp);
    }
    // INB: inlined at its single call site in mark_tile (the K-LARGE regime, where
    // phase 2 runs often: 93.5 vs 95.9 ms on the C5 span); else out of line (the
    // smaller hot loop wins at 1e12: 29.50 vs 29.69 ms)
    static __device__ __forceinline__ uint32_t batch(Shared6 &sh, uint32_t qn, uint32_t take, uint64_t u0,
                                                     const uint32_t *wA, const uint32_t *wB, uint32_t halo,
                                                     const VerifyArgs &a, CtaAcc *acc, uint32_t best_p, int lane,
                                                     int warp)
    {
        if constexpr (INB) return batch_body(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, warp);
        else return batch_call(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, warp);
    }

    // one phase-1 round: words pair*32kW + 32k + lane (k < kW) of class A
    template <bool TRACK>
    static __device__ __forceinline__ void round_q(Shared6 &sh, uint32_t &qn, uint32_t pair, uint32_t tw,
                                                   uint64_t u0, const uint32_t *wA, const uint32_t *wB,
                                                   uint32_t halo, const VerifyArgs &a, CtaAcc *acc,
                                                   uint32_t &best_p, int lane, int warp)
    {
        const uint32_t li0 = pair * 32 * kW + lane;
        LaneQ m;
        m.wa = wA + halo + li0;           // words past tw read window slack; their U is 0
        m.wb = wB + halo + li0;
        m.dump0 = DUMP ? a.dump + ((int64_t)(192 * (u0 + li0) + A) - (int64_t)a.lo_e) / 2 : nullptr;
        // warp-uniform: every word of the round inside the tile and the class's m range
        // (and not the word holding n = 4 and 6) -> all 32 evens of each word are live
        const uint64_t ub = u0 + pair * 32 * kW;
        const bool interior = pair * 32 * kW + 32 * kW <= tw && ub != 0 && ub * 32 >= a.m_lo[A / 2] &&
                              (ub + 32 * kW) * 32 <= a.m_hi[A / 2];
        if (interior) {
#pragma unroll
            for (int k = 0; k < kW; ++k) {
                m.U[k] = FULL;
                if (TRACK) { m.lb[k] = 0; m.lu[k] = 0; }
            }
            if (lane == 0) sh.wint[warp][A / 2] += 1;       // warp-private: folded in at the tile flush
        } else {
            uint32_t c = 0, e = 0;
#pragma unroll
            for (int k = 0; k < kW; ++k) {
                const uint32_t li = li0 + 32 * k;
                uint32_t U = li < tw ? valid_mask<A>(u0 + li, a) : 0u;
                e += __popc(U);
                if (k == 0) U = take_special<A, DUMP>(U, u0 + li, sh.hist, a, acc);
                m.U[k] = U;
                c += __popc(U);
                if (TRACK) { m.lb[k] = 0; m.lu[k] = 0; }
            }
            c = __reduce_add_sync(FULL, c + (e << 16));          // <= 3072 each
            if (lane == 0 && c) {
                atomicAdd(&sh.histc[A / 2][0], c & 0xFFFFu);
                atomicAdd(&acc->evens, (unsigned long long)(c >> 16));
            }
        }
        phase1q<A, 0, C1, DUMP, TRACK>(m, sh.histc[A / 2] + 1, lane);
        if (TRACK) replay_key_q<A>(m, u0 + li0, a, best_p, acc);
        // survivors of candidates [0, kC1): staged past the queue's live entries,
        // then compacted to 2 (or 1) words per lane for candidates [kC1, kP1)
        uint32_t tot = 0;
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            const uint32_t bal = __ballot_sync(FULL, m.U[k] != 0);
            if (m.U[k]) {
                const uint32_t pos = qn + tot + __popc(bal & ((1u << lane) - 1));
                sh_qli(sh, warp)[pos] = (uint16_t)(li0 + 32 * k);
                sh_qU(sh, warp)[pos] = m.U[k];
            }
            tot += __popc(bal);
        }
        __syncwarp();
        const uint32_t q0 = qn;
        for (uint32_t base = 0; base < tot; base += 64) {
            const uint32_t cnt = min(64u, tot - base);
            if (cnt > 32) stage<2, TRACK>(sh, qn, q0 + base, cnt, u0, wA, wB, halo, a, acc, best_p, lane, warp);
            else stage<1, TRACK>(sh, qn, q0 + base, cnt, u0, wA, wB, halo, a, acc, best_p, lane, warp);
        }
        if constexpr (!INB) {
            while (qn >= 32) {
                best_p = batch(sh, qn, 32, u0, wA, wB, halo, a, acc, best_p, lane, warp);
                qn -= 32;
            }
        }
    }

    // candidates [kC1, kP1) for cnt staged words at queue entries e0.. (S per lane);
    // survivors are appended to the queue (entries below e0 + 64 * pass: no overlap
    // with staged words not yet read)
    template <int S, bool TRACK>
    static __device__ __forceinline__ void stage(Shared6 &sh, uint32_t &qn, uint32_t e0, uint32_t cnt, uint64_t u0,
                                                 const uint32_t *wA, const uint32_t *wB, uint32_t halo,
                                                 const VerifyArgs &a, CtaAcc *acc, uint32_t &best_p, int lane, int warp)
    {
        LaneR<S> m;
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint32_t idx = 32 * k + lane;
            uint32_t li = 0, U = 0;
            if (idx < cnt) { li = sh_qli(sh, warp)[e0 + idx]; U = sh_qU(sh, warp)[e0 + idx]; }
            m.li[k] = li;
            m.U[k] = U;
            m.wa[k] = wA + halo + li;
            m.wb[k] = wB + halo + li;
            if (TRACK) { m.lb[k] = 0; m.lu[k] = 0; }
            if (DUMP) m.dump[k] = a.dump + ((int64_t)(192 * (u0 + li) + A) - (int64_t)a.lo_e) / 2;
        }
        __syncwarp();                          // staged entries read before any append
        phase1r<A, C1, P1, S, DUMP, TRACK>(m, sh.histc[A / 2] + 1, lane);
        if (TRACK) replay_key_r<A, S>(m, u0, a, best_p, acc);
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const uint32_t bal = __ballot_sync(FULL, m.U[k] != 0);
            if (m.U[k]) {
                const uint32_t pos = qn + __popc(bal & ((1u << lane) - 1));
                sh_qli(sh, warp)[pos] = (uint16_t)m.li[k];
                sh_qU(sh, warp)[pos] = m.U[k];
            }
            qn += __popc(bal);
        }
        __syncwarp();
    }

    static __device__ __forceinline__ void round(Shared6 &sh, uint32_t &qn, uint32_t pair, uint32_t tw,
                                                 uint64_t u0, const uint32_t *wA, const uint32_t *wB,
                                                 uint32_t halo, const VerifyArgs &a, CtaAcc *acc,
                                                 uint32_t &best_p, int lane, int warp)
    {
        if constexpr (UNROLL) {
            // max-key tracking only while phase-1 primes can still raise this warp's max
            constexpr uint32_t kP1Max = kTab[A / 2].p[P1 - 1];
            if (best_p > kP1Max)
                round_q<false>(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, warp);
            else
                round_q<true>(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, warp);
        } else {
            // p_max below the unrolled tables: runtime loop for every word (tests)
            const uint32_t li0 = pair * 32 * kW + lane;
            for (int k = 0; k < kW; ++k) {
                const uint32_t li = li0 + 32 * k;
                const uint64_t u = u0 + li;
                uint32_t U = li < tw ? valid_mask<A>(u, a) : 0u;
                const uint32_t e = __reduce_add_sync(FULL, __popc(U));
                if (lane == 0 && e) atomicAdd(&acc->evens, (unsigned long long)e);
                if (k == 0) U = take_special<A, DUMP>(U, u, sh.hist, a, acc);
                finish_word<A, DUMP>(U, 0, wA + halo + li, wB + halo + li, u, sh.hist, a, acc, lane);
            }
        }
    }
};

template <bool DUMP, bool UNROLL>
__device__ __forceinline__ void flush_queue(int cls, Shared6 &sh, uint32_t &qn, uint64_t u0, const uint32_t *wA,
                                            const uint32_t *wB, uint32_t halo, const VerifyArgs &a, CtaAcc *acc,
                                            uint32_t &best_p, int lane, int warp)
{
    if (!UNROLL || qn == 0) return;
    if (cls == 0) best_p = ClassWork<0, DUMP, UNROLL, false>::batch(sh, qn, qn, u0, wA, wB, halo, a, acc, best_p, lane, warp);
    else if (cls == 1) best_p = ClassWork<2, DUMP, UNROLL, false>::batch(sh, qn, qn, u0, wA, wB, halo, a, acc, best_p, lane, warp);
    else best_p = ClassWork<4, DUMP, UNROLL, false>::batch(sh, qn, qn, u0, wA, wB, halo, a, acc, best_p, lane, warp);
    qn = 0;
}

// marking of one tile: rounds of 32 kW words of one class, handed out dynamically
// (class-major) through the shared counter `next_round`; qwarp indexes the
// survivor queue of this warp
template <bool DUMP, bool UNROLL, bool INB>
__device__ __forceinline__ void mark_tile(Shared6 &sh, uint32_t &next_round, uint64_t u0, uint32_t tw,
                                          const uint32_t *wA, const uint32_t *wB, uint32_t halo,
                                          const VerifyArgs &a, CtaAcc *acc, uint32_t &best_p, int lane, int qwarp)
{
    const uint32_t r1 = (tw + 32 * kW - 1) / (32 * kW);
    uint32_t qn = 0;
    int qcls = 0;
    if constexpr (INB) {
    // phase-2 batches run here, between rounds, from one inlined copy per class: no
    // out-of-line call (whose ABI would save the caller's live registers to local
    // memory); the queue is drained below 32 before every round (a round adds <= 96
    // of the 128 entries) and emptied at a class change and at the end
    while (true) {
        uint32_t r = 0;
        if (lane == 0) r = atomicAdd(&next_round, 1u);
        r = __shfl_sync(FULL, r, 0);
        const bool last = r >= 3 * r1;
        const int cls = last ? -1 : (r >= r1 ? (r >= 2 * r1 ? 2 : 1) : 0);
        const uint32_t keep = cls == qcls ? 31u : 0u;
        while (UNROLL && qn > keep) {
            const uint32_t take = min(qn, 32u);
            if (qcls == 0) best_p = ClassWork<0, DUMP, UNROLL, true>::batch(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
            else if (qcls == 1) best_p = ClassWork<2, DUMP, UNROLL, true>::batch(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
            else best_p = ClassWork<4, DUMP, UNROLL, true>::batch(sh, qn, take, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
            qn -= take;
        }
        if (last) break;
        qcls = cls;
        const uint32_t pair = r - (uint32_t)cls * r1;
        if (cls == 0) ClassWork<0, DUMP, UNROLL, true>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
        else if (cls == 1) ClassWork<2, DUMP, UNROLL, true>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
        else ClassWork<4, DUMP, UNROLL, true>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
    }
    } else {
    while (true) {
        uint32_t r = 0;
        if (lane == 0) r = atomicAdd(&next_round, 1u);
        r = __shfl_sync(FULL, r, 0);
        if (r >= 3 * r1) break;
        const int cls = r >= r1 ? (r >= 2 * r1 ? 2 : 1) : 0;      // no integer division
        const uint32_t pair = r - (uint32_t)cls * r1;
        if (cls != qcls) {
            flush_queue<DUMP, UNROLL>(qcls, sh, qn, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
            qcls = cls;
        }
        if (cls == 0) ClassWork<0, DUMP, UNROLL, false>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
        else if (cls == 1) ClassWork<2, DUMP, UNROLL, false>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
        else ClassWork<4, DUMP, UNROLL, false>::round(sh, qn, pair, tw, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
    }
    flush_queue<DUMP, UNROLL>(qcls, sh, qn, u0, wA, wB, halo, a, acc, best_p, lane, qwarp);
    }
}

// shared histograms -> result vector (all threads; callers barrier around it).  The
// unrolled candidates' counts also give their share of sum p_min (count x p): the
// marking loops keep no per-word sums (every other path adds to acc.sum directly).
__device__ __forceinline__ void flush_hist(Shared6 &sh, const VerifyArgs &a, CtaAcc *acc, int tid)
{
    unsigned long long *R = (unsigned long long *)a.result;
    for (int i = tid; i < kHistSmem; i += kThreads) {
        const uint32_t v = sh.hist[i];
        if (v) {
            atomicAdd(R + GB_R_HIST + i, (unsigned long long)v);
            sh.hist[i] = 0;
        }
    }
    constexpr int kHc = 3 * kK;                                        // class-table entries
    constexpr int kPer = (kHc + kThreads - 1) / kThreads;              // per thread
    uint32_t v[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int i = tid + q * kThreads, c = i / kK, j = i % kK;
        v[q] = i < kHc ? sh.histc[c][j] - sh.histc[c][j + 1] : 0u;      // A_{j-1} - A_j
    }
    __syncthreads();
    for (int i = tid; i < 3 * (kK + 1); i += kThreads) (&sh.histc[0][0])[i] = 0;
    uint64_t sp = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const int i = tid + q * kThreads, c = i / kK, j = i % kK;
        if (v[q]) {
            sp += (uint64_t)v[q] * c_tab[c].p[j];
            atomicAdd(R + GB_R_HIST + c_tab[c].bin[j], (unsigned long long)v[q]);
        }
    }
    if (tid < kHc) {                                   // the warps holding entries: share of sum p_min
        for (int o = 16; o; o >>= 1) sp += __shfl_xor_sync(FULL, sp, o);
        if ((tid & 31) == 0 && sp) atomicAdd(&acc->sum, (unsigned long long)sp);
    }
}

// UNROLL: every unrolled candidate of the three class tables is <= p_max.
// __grid_constant__: the cold out-of-line paths take `a` by reference; without it
// the whole parameter block is copied to the local-memory stack and every field
// read becomes a local load (long-scoreboard stalls in the hot loop).
// INB: phase-2 batches inlined (the K-LARGE regime, see ClassWork::batch).
template <bool DUMP, bool UNROLL, bool INB>
__global__ void __launch_bounds__(kThreads) verify_kernel(const __grid_constant__ VerifyArgs a)
{
    uint32_t *win = g_win;                     // slot windows (class A | class B) | queues
    __shared__ Shared6 sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t halo = a.halo;
    const uint32_t nw_max = halo + a.tile_words + kWinSlack;
    if (tid == 0) sh.q_base = 2 * nw_max;
    for (int i = tid; i < kHistSmem; i += kThreads) sh.hist[i] = 0;
    for (int i = tid; i < 3 * (kK + 1); i += kThreads) (&sh.histc[0][0])[i] = 0;
    for (int i = tid; i < 3 * kMarkWarps; i += kThreads) (&sh.wint[0][0])[i] = 0;
    if (tid == 0) sh.acc = CtaAcc{0, 0, 0, 0, 0, ~0ull, 0};
    CtaAcc *const acc = &sh.acc;
    uint32_t best_p = 0;                       // per warp: replay only blocks that can raise the max
    // contiguous run of tiles per CTA, so the sieve can carry its offsets.  Nothing of
    // the sieve state stays live across the marking phase (register pressure): the
    // carry descriptor is rebuilt per tile from the grid constants, the running
    // steady count lives in shared memory.
    const uint64_t t_begin = (uint64_t)blockIdx.x * a.n_tiles / gridDim.x;
    const uint32_t n_mine = (uint32_t)((uint64_t)(blockIdx.x + 1) * a.n_tiles / gridDim.x - t_begin);
    if (tid == 0) sh.ns[1] = 0;                // running (monotone) steady count

    for (uint32_t t = 0; t < n_mine; ++t) {
        const uint64_t u0 = a.u_first + (t_begin + t) * a.tile_words;
        const uint32_t tw = (uint32_t)min((uint64_t)a.tile_words, a.u_end - u0);
        const int64_t g0 = (int64_t)u0 - (int64_t)halo;
        uint32_t *wA = win, *wB = win + nw_max;
        __syncthreads();                      // previous tile fully consumed
        {
            Carry6 cy;
            cy.off = a.carry + (uint64_t)blockIdx.x * 2 * a.carry_stride;
            cy.stride = a.carry_stride;
            cy.n_carry = a.n_carry;
            cy.have_prev = t > 0;
            cy.tile_m = 32 * a.tile_words;
            if (tid == 0) {
                sh.next_round[0] = 0;
                uint32_t ns_run = sh.ns[1];
                sh.ns[0] = steady_count(cy, g0, a.sp, ns_run);
                sh.ns[1] = ns_run;
            }
            __syncthreads();
            cy.n_steady = sh.ns[0] & 0x7FFFFFFFu;
            cy.init = sh.ns[0] >> 31;
            const MedSched med{a.med_idx, a.med_off};
            if (cy.tile_m == kTileM)
                sieve6<true, !INB>(wA, wB, g0, halo + tw, a.sp, &cy, med, a.i_b2, a.i_b1, a.lmask, a.lmask_g0,
                                   a.lmask_stride, tid);
            else
                sieve6<false, !INB>(wA, wB, g0, halo + tw, a.sp, &cy, med, a.i_b2, a.i_b1, a.lmask, a.lmask_g0,
                                    a.lmask_stride, tid);
        }
        __syncthreads();
        mark_tile<DUMP, UNROLL, INB>(sh, sh.next_round[0], u0, tw, wA, wB, halo, a, acc, best_p, lane, warp);
        // per-tile flush of the shared histograms keeps their 32-bit bins exact
        __syncthreads();
        if (tid < 3) {                 // interior rounds: 32 kW words of 32 live evens each
            uint32_t n = 0;
            for (int w = 0; w < kMarkWarps; ++w) { n += sh.wint[w][tid]; sh.wint[w][tid] = 0; }
            sh.histc[tid][0] += n * 32u * 32u * kW;
            if (n) atomicAdd(&acc->evens, (unsigned long long)n * 32ull * 32ull * kW);
        }
        __syncthreads();
        flush_hist(sh, a, acc, tid);
    }
    // the CTA's counts (thread 0) and the max key (one atomic per warp)
    __syncthreads();
    unsigned long long *R = (unsigned long long *)a.result;
    if (tid == 0) {
        const CtaAcc c = sh.acc;
        if (c.evens) atomicAdd(R + GB_R_EVENS, c.evens);
        if (c.evens - c.unres) atomicAdd(R + GB_R_VERIFIED, c.evens - c.unres);
        if (c.fast_unres) atomicAdd(R + GB_R_FASTPATH_UNRESOLVED, c.fast_unres);
        if (c.unres) atomicAdd(R + GB_R_UNRESOLVED, c.unres);
        if (c.sum) atomicAdd(R + GB_R_SUM_PMIN, c.sum);
        if (c.praw) atomicMax(R + GB_R_MAX_PMIN_RAW, c.praw);
        if (c.first_unres != ~0ull) atomicMin(R + GB_R_FIRST_UNRESOLVED_N, c.first_unres);
        if (c.key) atomicMax(R + GB_R_MAX_KEY, c.key);
    }
}


// ---------------------------------------------------------------------------
// gb_sieve_segment: tiles of the wheel-class sieve (sieve6_window, as in the verify
// kernel) written out in the paper's odd layout.  Odd q = 6m+1
// (class A) is o = 3m - 1, q = 6m+3 is o = 3m (composite but for q = 3), q = 6m+5
// (class B) is o = 3m + 1: the 96 odd bits [96g, 96g+96) hold B bits 32g..32g+31 at
// o = 96g + 3j + 1 and A bits 32g+1..32g+32 at o = 96g + 3j + 2.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) sieve_out_kernel(const __grid_constant__ SieveOutArgs a)
{
    uint32_t *win = g_win;
    const uint32_t nw_max = a.tile_words + 1 + kWinSlack;
    uint32_t *wA = win, *wB = win + nw_max;
    __shared__ uint32_t spread3[256];          // bit j of a byte -> bit 3j
    __shared__ uint32_t sh_ns;
    const int tid = threadIdx.x;
    for (int i = tid; i < 256; i += kThreads) {
        uint32_t v = 0;
        for (int j = 0; j < 8; ++j) v |= ((i >> j) & 1u) << (3 * j);
        spread3[i] = v;
    }
    const uint64_t t_begin = (uint64_t)blockIdx.x * a.n_tiles / gridDim.x;
    const uint64_t t_end = (uint64_t)(blockIdx.x + 1) * a.n_tiles / gridDim.x;
    Carry6 cy;
    cy.off = a.carry + (uint64_t)blockIdx.x * 2 * a.carry_stride;
    cy.stride = a.carry_stride;
    cy.n_carry = a.n_carry;
    cy.have_prev = false;
    cy.n_steady = 0;
    cy.init = false;
    cy.tile_m = 32 * a.tile_words;
    uint32_t ns_run = 0;
    for (uint64_t tile = t_begin; tile < t_end; ++tile) {
        const uint64_t g0 = a.g_first + tile * a.tile_words;
        const uint32_t tw = (uint32_t)min((uint64_t)a.tile_words, a.g_end - g0);
        __syncthreads();                      // previous tile written out
        if (tid == 0) sh_ns = steady_count(cy, (int64_t)g0, a.sp, ns_run);
        __syncthreads();
        cy.n_steady = sh_ns & 0x7FFFFFFFu;
        cy.init = sh_ns >> 31;
        if (cy.tile_m == kTileM)
            sieve6_window<true>(wA, wB, (int64_t)g0, tw + 1, a.sp, &cy, MedSched{a.med_idx, a.med_off}, a.i_b2,
                                a.i_b1, a.lmask, a.lmask_g0, a.lmask_stride, tid);
        else
            sieve6_window<false>(wA, wB, (int64_t)g0, tw + 1, a.sp, &cy, MedSched{a.med_idx, a.med_off}, a.i_b2,
                                 a.i_b1, a.lmask, a.lmask_g0, a.lmask_stride, tid);
        cy.have_prev = true;
        __syncthreads();
        for (uint32_t i = tid; i < tw; i += kThreads) {
            const uint32_t A = __funnelshift_r(wA[i], wA[i + 1], 1);   // A bits 32g+1 .. 32g+32
            const uint32_t B = wB[i];
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v[k] = (spread3[(A >> (8 * k)) & 0xFF] << 2) | (spread3[(B >> (8 * k)) & 0xFF] << 1);
            const uint64_t g = g0 + i;
            uint32_t o0 = v[0] | (v[1] << 24);
            const uint32_t o1 = (v[1] >> 8) | (v[2] << 16);
            const uint32_t o2 = (v[2] >> 16) | (v[3] << 8);
            if (g == 0) o0 |= 1u;                                         // q = 3
            const uint64_t W = 3 * g;
            if (W >= a.w_lo && W < a.w_hi) a.out[W - a.w_lo] = o0;
            if (W + 1 >= a.w_lo && W + 1 < a.w_hi) a.out[W + 1 - a.w_lo] = o1;
            if (W + 2 >= a.w_lo && W + 2 < a.w_hi) a.out[W + 2 - a.w_lo] = o2;
        }
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
// Dynamic shared memory opt-in, once per device, at the largest size these kernels
// are ever launched with (kVerifySmemMax / kSieveOutSmemMax, gb_internal.h).
cudaError_t configure_verify()
{
    static std::atomic<uint64_t> d0{0}, d1{0}, d2{0}, d3{0}, d4{0}, d5{0};
    constexpr int sm = (int)kVerifySmemMax;
    cudaError_t e = ensure_dyn_smem((const void *)verify_kernel<false, false, false>, sm, d0);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void *)verify_kernel<true, false, false>, sm, d1);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void *)verify_kernel<false, true, false>, sm, d2);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void *)verify_kernel<true, true, false>, sm, d3);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void *)verify_kernel<false, true, true>, sm, d4);
    if (e == cudaSuccess) e = ensure_dyn_smem((const void *)verify_kernel<true, true, true>, sm, d5);
    return e;
}

cudaError_t launch_sieve_out(const SieveOutArgs &a, int grid, size_t smem, cudaStream_t st)
{
    static std::atomic<uint64_t> done{0};
    if (smem > kSieveOutSmemMax) return cudaErrorInvalidValue;
    const cudaError_t e = ensure_dyn_smem((const void *)sieve_out_kernel, (int)kSieveOutSmemMax, done);
    if (e != cudaSuccess) return e;
    sieve_out_kernel<<<grid, kThreads, smem, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

int verify_blocks_per_sm(size_t smem)
{
    int nb = 0;
    if (configure_verify() != cudaSuccess) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, verify_kernel<false, true, false>, kThreads, smem) !=
        cudaSuccess)
        return 1;
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_verify(const VerifyArgs &a, int grid, size_t smem, cudaStream_t st)
{
    if (smem > kVerifySmemMax) return cudaErrorInvalidValue;
    const cudaError_t e = configure_verify();
    if (e != cudaSuccess) return e;
    const bool unroll = a.p_fallback - 2 >= kUnrollPMax;   // p_fallback = largest candidate + 2
    const bool inb = a.lmask != nullptr;                    // K-LARGE regime (hi > 2^42): inlined batches
    if (a.dump) {
        if (unroll && inb) verify_kernel<true, true, true><<<grid, kThreads, smem, st>>>(a);
        else if (unroll) verify_kernel<true, true, false><<<grid, kThreads, smem, st>>>(a);
        else verify_kernel<true, false, false><<<grid, kThreads, smem, st>>>(a);
    } else {
        if (unroll && inb) verify_kernel<false, true, true><<<grid, kThreads, smem, st>>>(a);
        else if (unroll) verify_kernel<false, true, false><<<grid, kThreads, smem, st>>>(a);
        else verify_kernel<false, false, false><<<grid, kThreads, smem, st>>>(a);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace gb
