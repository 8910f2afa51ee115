// gb_api.cu -- the C ABI declared in include/gb.h: argument checking, workspace
// carve-out, range planning and kernel launches.  No compute happens here; every
// step of the path runs in the kernels of gb_kernels.cu.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <vector>

#include "gb_internal.h"

using namespace gb;

namespace {

uint64_t isqrt_u64(uint64_t x)
{
    uint64_t lo = 0, hi = 4294967296ull;      // lo^2 <= x < hi^2
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if ((unsigned __int128)mid * mid <= x) lo = mid; else hi = mid;
    }
    return lo;
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

constexpr uint64_t kMaxSms = 160;   // workspace sizing bound (B200: 148)
constexpr uint64_t kMinTileWords = 1024;   // smallest balanced tile (and never below the halo)

struct Layout {
    uint64_t R, bits_words, list_cap, n_blk, carry_stride, carry_ctas, lmask_stride;
    uint64_t off_bits, off_primes, off_magic, off_tmod, off_carry, off_lmask, off_sched, off_blk, off_counter,
        off_res, off_dump, off_seg, total;
};

// pi(x) upper bound (Rosser-Schoenfeld: pi(x) < 1.25506 x / ln x for x > 1) + slack
uint64_t pi_upper(uint64_t x)
{
    if (x < 17) return 8;
    return (uint64_t)(1.25506 * (double)x / __builtin_log((double)x)) + 64;
}

uint32_t verify_halo(uint32_t p_top);

bool plan(uint64_t hi_max, uint32_t p_max, Layout &L)
{
    if (hi_max < 5 || hi_max > GB_HI_LIMIT || p_max < 3 || p_max > GB_PMAX_LIMIT) return false;
    uint64_t R = isqrt_u64(hi_max - 1);
    R = std::max<uint64_t>(R, p_max);
    R = std::max<uint64_t>(R, 1024);
    if (R > 0xFFFFFFFFull - 64) return false;   // primes are u32
    L.R = R;
    L.bits_words = ((R - 3) / 2) / 64 + 1;
    L.list_cap = pi_upper(R);
    // carried offsets: one row per possible resident verify CTA, one u32 per sieving
    // prime p <= min(isqrt(hi_max - 1), kCarryPrimeMax)
    const uint64_t sq = isqrt_u64(hi_max - 1);
    L.carry_stride = align_up(pi_upper(std::min<uint64_t>(sq, kCarryPrimeMax)), 64);
    L.carry_ctas = 0;   // filled by the caller with the device's SM count
    // K-LARGE chunk mask (two wheel classes), only when some sieving prime exceeds
    // the carried range: kLargeTilesPerSm tiles per SM + the largest halo
    L.lmask_stride = sq > kCarryPrimeMax
                         ? align_up((uint64_t)kLargeTilesPerSm * kMaxSms * kTileWords + verify_halo(p_max) + 64, 64)
                         : 0;
    L.n_blk = (L.bits_words + kScanBlockWords - 1) / kScanBlockWords;
    uint64_t o = 0;
    L.off_bits = o;    o = align_up(o + 8 * L.bits_words, 256);
    L.off_primes = o;  o = align_up(o + 4 * L.list_cap, 256);
    L.off_magic = o;   o = align_up(o + 8 * L.list_cap, 256);
    L.off_tmod = o;    o = align_up(o + 16 * L.list_cap, 256);
    L.off_carry = o;   o = align_up(o + 8 * L.carry_stride * (uint64_t)kMaxBlocksPerSm * kMaxSms, 256);
    L.off_lmask = o;   o = align_up(o + 8 * L.lmask_stride, 256);
    L.off_sched = o;   o = align_up(o + 2 * 1024 + 4 * (kThreads / 32 + 1), 256);
    L.off_blk = o;     o = align_up(o + 8 * (L.n_blk + 1), 256);
    L.off_counter = o; o = align_up(o + 256, 256);
    L.off_res = o;     o = align_up(o + 8 * (uint64_t)GB_RESULT_WORDS, 256);
    L.off_dump = o;    o = align_up(o + 4 * kDumpScratch, 256);
    L.off_seg = o;     o = align_up(o + 8 * (kPerNSegEvens / 64 + 4), 256);
    L.total = o;
    return true;
}

inline cudaStream_t S(void *s) { return (cudaStream_t)s; }

// count of list entries <= x
uint32_t count_le(const std::vector<uint32_t> &v, uint64_t x)
{
    if (x >= 0xFFFFFFFFull) return (uint32_t)v.size();
    return (uint32_t)(std::upper_bound(v.begin(), v.end(), (uint32_t)x) - v.begin());
}

// wheel halo: the largest shift of a candidate p is p/6 + 1 bits
uint32_t verify_halo(uint32_t p_top) { return ((p_top / 6 + 1) >> 5) + 1; }
// the two class windows must fit next to the queues and the kernel's static shared
// memory (kVerifyWinSmemMax, gb_internal.h); a large halo shrinks the tile
uint32_t verify_tile_words(uint32_t halo)
{
    if (2 * 4ull * (halo + kTileWords + kWinSlackWords) <= kVerifyWinSmemMax) return kTileWords;
    const uint32_t tw = (kVerifyWinSmemMax / 8 - halo - kWinSlackWords) & ~127u;   // multiple of 128 words
    return tw;
}
size_t verify_smem(uint32_t halo)
{
    return 2 * 4ull * (halo + verify_tile_words(halo) + kWinSlackWords) + kQueueBytes;
}

SievePrimes sieve_primes(const gb_ctx *c, uint64_t sqrt_bound)
{
    SievePrimes sp;
    sp.primes = c->primes;
    sp.magic = c->magic;
    sp.pk = c->pk;
    sp.i_med = count_le(c->h_primes, 31);
    sp.i_big = count_le(c->h_primes, kWarpPrimeMax);
    sp.n_use = count_le(c->h_primes, sqrt_bound);
    return sp;
}

// the device that owns a device pointer (false for host / unregistered memory)
bool pointer_device(const void *p, int &dev)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();                    // clear the sticky-free error state
        return false;
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return false;
    dev = at.device;
    return true;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d)
    {
        cudaGetDevice(&prev);
        if (prev != d) cudaSetDevice(d);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

const char *gb_status_string(gb_status s)
{
    switch (s) {
    case GB_OK: return "GB_OK";
    case GB_EINVAL: return "GB_EINVAL: invalid argument";
    case GB_ERANGE: return "GB_ERANGE: range needs base primes beyond the context's hi_max";
    case GB_EWORKSPACE: return "GB_EWORKSPACE: workspace too small";
    case GB_ECUDA: return "GB_ECUDA: CUDA error";
    case GB_EINTERNAL: return "GB_EINTERNAL: internal error";
    }
    return "unknown gb_status";
}

size_t gb_ctx_workspace_bytes(uint64_t hi_max, uint32_t p_max)
{
    Layout L;
    if (!plan(hi_max, p_max, L)) return 0;
    return (size_t)L.total;
}

gb_status gb_ctx_create(gb_ctx **out, int device, uint64_t origin, uint64_t hi_max, uint32_t p_max,
                        void *d_workspace, size_t ws_bytes, void *stream)
{
    if (!out) return GB_EINVAL;
    *out = nullptr;
    Layout L;
    if (!plan(hi_max, p_max, L) || !d_workspace || ((uintptr_t)d_workspace & 255)) return GB_EINVAL;
    if ((origin & 1) || origin > hi_max || ((hi_max - origin) >> 1) >= (1ull << GB_KEY_SHIFT))
        return GB_EINVAL;
    if (ws_bytes < L.total) return GB_EWORKSPACE;
    DeviceGuard g(device);
    gb_ctx *c = new (std::nothrow) gb_ctx();
    if (!c) return GB_EINTERNAL;
    char *ws = (char *)d_workspace;
    c->device = device;
    c->origin = origin;
    c->hi_max = hi_max;
    c->p_max = p_max;
    c->R = L.R;
    c->bits = (uint64_t *)(ws + L.off_bits);
    c->bits_words = L.bits_words;
    c->primes = (uint32_t *)(ws + L.off_primes);
    c->magic = (uint64_t *)(ws + L.off_magic);
    c->pk = (uint4 *)(ws + L.off_tmod);
    c->carry = (uint32_t *)(ws + L.off_carry);
    c->carry_stride = L.carry_stride;
    c->lmask = L.lmask_stride ? (uint32_t *)(ws + L.off_lmask) : nullptr;
    c->lmask_stride = L.lmask_stride;
    c->med_idx = (uint16_t *)(ws + L.off_sched);
    c->med_off = (uint32_t *)(ws + L.off_sched + 2 * 1024);
    c->blk = (uint64_t *)(ws + L.off_blk);
    c->counter = (uint32_t *)(ws + L.off_counter);
    c->res_scratch = (int64_t *)(ws + L.off_res);
    c->dump_scratch = (uint32_t *)(ws + L.off_dump);
    c->seg_scratch = (uint64_t *)(ws + L.off_seg);
    if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    if ((uint64_t)c->num_sms > kMaxSms) { delete c; return GB_EINTERNAL; }
    c->carry_ctas = (uint32_t)(kMaxBlocksPerSm * c->num_sms);
    cudaStream_t st = S(stream);
    // K-BASE stage 1: seed primes <= isqrt(R) (with per-prime magic)
    const uint64_t s = isqrt_u64(L.R);
    if (launch_seed(s, c->primes, c->magic, c->pk, c->counter, st) != cudaSuccess) { delete c; return GB_ECUDA; }
    uint32_t n_seed = 0;
    if (cudaMemcpyAsync(&n_seed, c->counter, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    c->h_primes.resize(n_seed);
    if (cudaMemcpy(c->h_primes.data(), c->primes, 4ull * n_seed, cudaMemcpyDeviceToHost) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    // K-BASE stage 2: segment sieve of [3, R] with the seeds
    SegmentArgs sa;
    sa.sp = sieve_primes(c, s);
    sa.g_lo = 0;
    sa.n_words32 = 2 * L.bits_words;
    sa.o_limit = (L.R - 3) / 2 + 1;            // odd q <= R only
    sa.out = (uint32_t *)c->bits;
    if (launch_segment(sa, st) != cudaSuccess) { delete c; return GB_ECUDA; }
    // K-BASE stage 3: compaction into the ascending list (+ magic)
    if (launch_count_bits(c->bits, L.bits_words, c->blk, st) != cudaSuccess ||
        launch_scan(c->blk, L.n_blk, st) != cudaSuccess ||
        launch_scatter(c->bits, L.bits_words, c->blk, c->primes, c->magic, c->pk, st) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    uint64_t n_base = 0;
    if (cudaMemcpyAsync(&n_base, c->blk + L.n_blk, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    if (n_base > L.list_cap) { delete c; return GB_EINTERNAL; }
    c->n_base = n_base;
    c->h_primes.resize(n_base);
    if (cudaMemcpy(c->h_primes.data(), c->primes, 4ull * n_base, cudaMemcpyDeviceToHost) != cudaSuccess) {
        delete c;
        return GB_ECUDA;
    }
    // LPT schedule of the medium primes (31 < p <= kWarpPrimeMax) over the verify
    // CTA's warps, by estimated marking work (hits per full window / 32 lanes + setup)
    {
        const uint32_t i_med = count_le(c->h_primes, 31), i_big = count_le(c->h_primes, kWarpPrimeMax);
        const uint32_t nmed = i_big > i_med ? i_big - i_med : 0;
        if (nmed > 1024) { delete c; return GB_EINTERNAL; }
        const int nw = kMarkWarps;                     // every warp of a verify CTA sieves
        const uint32_t h0 = verify_halo(c->h_primes[count_le(c->h_primes, p_max) - 1]);
        const double nbits = 32.0 * (h0 + verify_tile_words(h0));
        std::vector<std::vector<uint16_t>> lists(nw);
        std::vector<double> load(nw, 0.0);
        for (uint32_t r = 0; r < nmed; ++r) {            // ascending p = descending work
            const double p = c->h_primes[i_med + r];
            const double cost = 2.0 * 3.0 * std::ceil(nbits / p / 32.0) + 30.0;
            int best = 0;
            for (int w = 1; w < nw; ++w)
                if (load[w] < load[best]) best = w;
            load[best] += cost;
            lists[best].push_back((uint16_t)r);
        }
        std::vector<uint16_t> idx;
        std::vector<uint32_t> off(1, 0);
        for (int w = 0; w < nw; ++w) {
            idx.insert(idx.end(), lists[w].begin(), lists[w].end());
            off.push_back((uint32_t)idx.size());
        }
        if ((!idx.empty() && cudaMemcpy(c->med_idx, idx.data(), 2 * idx.size(), cudaMemcpyHostToDevice) !=
                                 cudaSuccess) ||
            cudaMemcpy(c->med_off, off.data(), 4 * off.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            delete c;
            return GB_ECUDA;
        }
    }
    // verify kernel dynamic shared memory opt-in on this device
    if (configure_verify() != cudaSuccess) { delete c; return GB_ECUDA; }
    *out = c;
    return GB_OK;
}

void gb_ctx_destroy(gb_ctx *ctx) { delete ctx; }

gb_status gb_ctx_info(const gb_ctx *ctx, uint64_t *n_base_primes, uint64_t *R)
{
    if (!ctx) return GB_EINVAL;
    if (n_base_primes) *n_base_primes = ctx->n_base;
    if (R) *R = ctx->R;
    return GB_OK;
}

gb_status gb_ctx_tables(const gb_ctx *ctx, const uint64_t **d_bits, const uint32_t **d_primes)
{
    if (!ctx) return GB_EINVAL;
    if (d_bits) *d_bits = ctx->bits;
    if (d_primes) *d_primes = ctx->primes;
    return GB_OK;
}

gb_status gb_sieve_segment(gb_ctx *ctx, uint64_t word_lo, uint64_t n_words, uint64_t *d_words,
                           void *stream)
{
    if (!ctx || ((uintptr_t)d_words & 7)) return GB_EINVAL;
    if (n_words == 0) return GB_OK;
    if (!d_words || word_lo > (1ull << 58) || n_words > (1ull << 58)) return GB_EINVAL;
    const uint64_t top_o = 64 * (word_lo + n_words) - 1;   // largest odd index
    if (top_o > (GB_HI_LIMIT - 3) / 2) return GB_EINVAL;
    const uint64_t q_max = 3 + 2 * top_o;
    const uint64_t r = isqrt_u64(q_max);
    if (r > ctx->R) return GB_ERANGE;
    DeviceGuard g(ctx->device);
    cudaStream_t st = S(stream);
    // output u32 words [w_lo, w_hi) <- class words [g_lo, g_hi), tiles of kTileWords
    SieveOutArgs a;
    a.sp = sieve_primes(ctx, r);
    if (a.sp.i_big - a.sp.i_med > 1024) return GB_EINTERNAL;
    a.w_lo = 2 * word_lo;
    a.w_hi = 2 * (word_lo + n_words);
    a.out = (uint32_t *)d_words;
    const uint64_t g_lo = a.w_lo / 3, g_hi = (a.w_hi + 2) / 3;
    a.tile_words = kTileWords;
    const uint64_t n_tiles = (g_hi - g_lo + a.tile_words - 1) / a.tile_words;
    a.carry = ctx->carry;
    a.carry_stride = ctx->carry_stride;
    a.n_carry = (uint32_t)std::min<uint64_t>(std::min<uint32_t>(a.sp.n_use, count_le(ctx->h_primes, kCarryPrimeMax)),
                                             ctx->carry_stride);
    a.med_idx = ctx->med_idx;
    a.med_off = ctx->med_off;
    a.i_b2 = count_le(ctx->h_primes, 16ull * (a.tile_words + 1));
    a.i_b1 = count_le(ctx->h_primes, 32ull * (a.tile_words + 1));
    a.lmask = nullptr;
    a.lmask_g0 = 0;
    a.lmask_stride = 0;
    // the two class windows of a tile
    const size_t smem = kSieveOutSmemMax;
    const int grid_max = (int)std::min<uint64_t>((uint64_t)ctx->num_sms, ctx->carry_ctas);
    const uint32_t i_large = count_le(ctx->h_primes, kCarryPrimeMax);
    const bool large = a.sp.n_use > i_large;
    const uint32_t n_use_all = a.sp.n_use;
    if (large) {
        if (!ctx->lmask) return GB_EINTERNAL;
        a.sp.n_use = i_large;
    }
    // chunks of whole tiles (one chunk unless K-LARGE masks are needed)
    uint64_t chunk_tiles = n_tiles;
    if (large) {
        chunk_tiles = std::min<uint64_t>((ctx->lmask_stride - 64) / a.tile_words, (uint64_t)kLargeTilesPerSm * grid_max);
        if (chunk_tiles > (uint64_t)grid_max) chunk_tiles -= chunk_tiles % (uint64_t)grid_max;
        if (chunk_tiles == 0) return GB_EINTERNAL;
    }
    for (uint64_t t0 = 0; t0 < n_tiles; t0 += chunk_tiles) {
        SieveOutArgs b = a;
        const uint64_t nt = std::min<uint64_t>(chunk_tiles, n_tiles - t0);
        b.g_first = g_lo + t0 * a.tile_words;
        b.g_end = std::min<uint64_t>(g_hi, b.g_first + nt * a.tile_words);
        b.n_tiles = nt;
        if (large) {
            LargeArgs L;
            L.primes = ctx->primes;
            L.magic = ctx->magic;
            L.i_begin = i_large;
            L.i_end = n_use_all;
            L.g0 = (int64_t)b.g_first;
            L.nw = (uint32_t)(b.g_end - b.g_first + 1);   // + the class-A word above the last tile
            L.stride = ctx->lmask_stride;
            L.mask = ctx->lmask;
            b.lmask = ctx->lmask;
            b.lmask_g0 = L.g0;
            b.lmask_stride = L.stride;
            if (launch_large(L, ctx->num_sms, st) != cudaSuccess) return GB_ECUDA;
        }
        const int grid = (int)std::min<uint64_t>((uint64_t)grid_max, nt);
        if (launch_sieve_out(b, grid, smem, st) != cudaSuccess) return GB_ECUDA;
    }
    return GB_OK;
}

gb_status gb_result_init(int64_t *d_result, void *stream)
{
    if (!d_result || ((uintptr_t)d_result & 7)) return GB_EINVAL;
    int dev = -1;
    if (!pointer_device(d_result, dev)) return GB_EINVAL;
    DeviceGuard g(dev);
    return launch_result_init(d_result, S(stream)) == cudaSuccess ? GB_OK : GB_ECUDA;
}

gb_status gb_result_finalize(int64_t *d_result, void *stream)
{
    if (!d_result || ((uintptr_t)d_result & 7)) return GB_EINVAL;
    (void)stream;
    int dev = -1;
    return pointer_device(d_result, dev) ? GB_OK : GB_EINVAL;
}

gb_status gb_verify_range_ex(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                             uint64_t fallback_p_cap, int64_t *d_result, uint32_t *d_pmin_dump,
                             void *stream)
{
    if (!ctx || !d_result || ((uintptr_t)d_result & 7) || ((uintptr_t)d_pmin_dump & 3))
        return GB_EINVAL;
    if (lo > hi || hi > GB_HI_LIMIT || p_max < 3 || p_max > ctx->p_max) return GB_EINVAL;
    const uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return GB_OK;                            // empty range: no launch
    if (hi > ctx->hi_max) return GB_ERANGE;
    if (lo_e < ctx->origin || ((hi - ctx->origin) >> 1) >= (1ull << GB_KEY_SHIFT)) return GB_EINVAL;
    // A range that straddles 2^42 = kCarryPrimeMax^2 only needs the K-LARGE chunks
    // above it: below, every sieving prime is carried in shared memory, so that part
    // runs as one unchunked launch (results add; the dump continues at its offset)
    constexpr uint64_t kSplit = (uint64_t)kCarryPrimeMax * kCarryPrimeMax;
    if (lo_e < kSplit && hi > kSplit) {
        gb_status st = gb_verify_range_ex(ctx, lo_e, kSplit, p_max, fallback_p_cap, d_result, d_pmin_dump, stream);
        if (st != GB_OK) return st;
        return gb_verify_range_ex(ctx, kSplit, hi, p_max, fallback_p_cap, d_result,
                                  d_pmin_dump ? d_pmin_dump + (kSplit - lo_e) / 2 : nullptr, stream);
    }
    VerifyArgs a;
    // wheel classes n = 6m + c (c = 0, 2, 4): valid m in [ceil((lo_e-c)/6), ceil((hi-c)/6))
    uint64_t mlo_min = UINT64_MAX, mhi_max = 0;
    for (int k = 0; k < 3; ++k) {
        const uint64_t c = 2 * (uint64_t)k;
        a.m_lo[k] = (lo_e - c + 5) / 6;
        a.m_hi[k] = (hi - c + 5) / 6;
        if (a.m_lo[k] < a.m_hi[k]) {
            mlo_min = std::min(mlo_min, a.m_lo[k]);
            mhi_max = std::max(mhi_max, a.m_hi[k]);
        }
    }
    if (mhi_max == 0) return GB_OK;                          // no even n in range
    const uint64_t r = isqrt_u64(hi - 1);
    if (r > ctx->R) return GB_ERANGE;
    a.sp = sieve_primes(ctx, r);
    if (a.sp.i_big - a.sp.i_med > 1024) return GB_EINTERNAL;
    a.n_cand = count_le(ctx->h_primes, p_max);
    if (a.n_cand == 0) return GB_EINVAL;
    const uint32_t p_top = ctx->h_primes[a.n_cand - 1];
    a.halo = verify_halo(p_top);
    a.u_first = mlo_min >> 5;
    a.u_end = ((mhi_max - 1) >> 5) + 1;
    a.tile_words = verify_tile_words(a.halo);
    a.n_tiles = (a.u_end - a.u_first + a.tile_words - 1) / a.tile_words;
    a.lo_e = lo_e;
    a.origin = ctx->origin;
    a.p_fallback = (uint64_t)p_top + 2;
    a.cap = fallback_p_cap;
    a.base_bits = ctx->bits;
    a.R = ctx->R;
    a.n_base = (uint32_t)ctx->n_base;
    a.result = d_result;
    a.dump = d_pmin_dump;
    DeviceGuard g(ctx->device);
    const size_t smem = verify_smem(a.halo);
    const int per_sm = verify_blocks_per_sm(smem);
    const uint64_t max_grid = (uint64_t)per_sm * ctx->num_sms;
    {
        // a few tiles per CTA (small ranges): shrink the tile so that every CTA gets
        // the same number of whole tiles (e.g. [4, 1e9]: 254 default tiles on 148
        // CTAs, 106 of them doing two -> 296 tiles of 17,664 words, two each)
        // (fewer tiles than CTAs: tiles of at least kMinTileWords, one per CTA)
        const uint64_t gmax = std::min<uint64_t>(max_grid, ctx->carry_ctas);
        const uint64_t words = a.u_end - a.u_first;
        if (gmax > 0 && a.n_tiles < 8 * gmax) {
            const uint64_t per = (a.n_tiles + gmax - 1) / gmax;
            uint64_t tw = ((words + per * gmax - 1) / (per * gmax) + 127) & ~127ull;
            tw = std::max<uint64_t>(tw, std::max<uint64_t>(kMinTileWords, a.halo));   // re-sieved halo <= tile
            if (tw < a.tile_words) {
                a.tile_words = (uint32_t)tw;
                a.n_tiles = (words + tw - 1) / tw;
            }
        }
    }
    const int grid = (int)std::min<uint64_t>(std::min<uint64_t>(a.n_tiles, max_grid), ctx->carry_ctas);
    a.carry = ctx->carry;
    a.carry_stride = ctx->carry_stride;
    a.n_carry = std::min<uint32_t>(a.sp.n_use, count_le(ctx->h_primes, kCarryPrimeMax));
    a.n_carry = (uint32_t)std::min<uint64_t>(a.n_carry, ctx->carry_stride);
    a.med_idx = ctx->med_idx;
    a.med_off = ctx->med_off;
    a.i_b2 = count_le(ctx->h_primes, 16ull * (a.halo + a.tile_words));   // 2p > 32 (halo + tile) bits
    a.i_b1 = count_le(ctx->h_primes, 32ull * (a.halo + a.tile_words));   // p > 32 (halo + tile) bits
    a.lmask = nullptr;
    a.lmask_g0 = 0;
    a.lmask_stride = 0;
    const uint32_t i_large = count_le(ctx->h_primes, kCarryPrimeMax);
    if (a.sp.n_use <= i_large)
        return launch_verify(a, grid, smem, S(stream)) == cudaSuccess ? GB_OK : GB_ECUDA;
    // Sieving primes above kCarryPrimeMax: chunks of whole tiles (a multiple of the
    // grid), each preceded by K-LARGE over its windows (tiles + the halo below).
    if (!ctx->lmask) return GB_EINTERNAL;
    const uint32_t n_use_all = a.sp.n_use;
    a.sp.n_use = i_large;
    const uint64_t cap_tiles = (ctx->lmask_stride - a.halo - 64) / a.tile_words;
    uint64_t chunk_tiles = std::min<uint64_t>(cap_tiles, (uint64_t)kLargeTilesPerSm * grid);
    if (chunk_tiles > (uint64_t)grid) chunk_tiles -= chunk_tiles % (uint64_t)grid;
    if (chunk_tiles == 0) return GB_EINTERNAL;
    for (uint64_t t0 = 0; t0 < a.n_tiles; t0 += chunk_tiles) {
        VerifyArgs b = a;
        const uint64_t nt = std::min<uint64_t>(chunk_tiles, a.n_tiles - t0);
        b.u_first = a.u_first + t0 * a.tile_words;
        b.u_end = std::min<uint64_t>(a.u_end, b.u_first + nt * a.tile_words);
        b.n_tiles = nt;
        LargeArgs L;
        L.primes = ctx->primes;
        L.magic = ctx->magic;
        L.i_begin = i_large;
        L.i_end = n_use_all;
        L.g0 = (int64_t)b.u_first - (int64_t)a.halo;
        L.nw = (uint32_t)(b.u_end - b.u_first + a.halo);
        L.stride = ctx->lmask_stride;
        L.mask = ctx->lmask;
        b.lmask = ctx->lmask;
        b.lmask_g0 = L.g0;
        b.lmask_stride = L.stride;
        if (launch_large(L, ctx->num_sms, S(stream)) != cudaSuccess) return GB_ECUDA;
        const int gb = (int)std::min<uint64_t>((uint64_t)grid, nt);
        if (launch_verify(b, gb, smem, S(stream)) != cudaSuccess) return GB_ECUDA;
    }
    return GB_OK;
}

gb_status gb_verify_range(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max, int64_t *d_result,
                          uint32_t *d_pmin_dump, void *stream)
{
    return gb_verify_range_ex(ctx, lo, hi, p_max, UINT64_MAX, d_result, d_pmin_dump, stream);
}

gb_status gb_verify_range_host(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max,
                               int64_t *h_result, uint32_t *h_pmin_dump, void *stream)
{
    if (!ctx || !h_result) return GB_EINVAL;
    DeviceGuard g(ctx->device);
    cudaStream_t st = S(stream);
    gb_status s = gb_result_init(ctx->res_scratch, stream);
    if (s != GB_OK) return s;
    const uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (!h_pmin_dump) {
        s = gb_verify_range(ctx, lo, hi, p_max, ctx->res_scratch, nullptr, stream);
        if (s != GB_OK) return s;
    } else {
        // chunks of kDumpScratch evens through the device scratch
        for (uint64_t c = lo_e; c < hi; c += 2 * kDumpScratch) {
            const uint64_t ce = std::min<uint64_t>(hi, c + 2 * kDumpScratch);
            s = gb_verify_range(ctx, c, ce, p_max, ctx->res_scratch, ctx->dump_scratch, stream);
            if (s != GB_OK) return s;
            const uint64_t cnt = (ce - c + 1) / 2;
            if (cudaMemcpyAsync(h_pmin_dump + (c - lo_e) / 2, ctx->dump_scratch, 4 * cnt,
                                cudaMemcpyDeviceToHost, st) != cudaSuccess)
                return GB_ECUDA;
        }
    }
    s = gb_result_finalize(ctx->res_scratch, stream);
    if (s != GB_OK) return s;
    if (cudaMemcpyAsync(h_result, ctx->res_scratch, 8ull * GB_RESULT_WORDS, cudaMemcpyDeviceToHost,
                        st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return GB_ECUDA;
    return GB_OK;
}

gb_status gb_verify_range_pern(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max, int64_t *d_result,
                               uint32_t *d_pmin_dump, void *stream)
{
    if (!ctx || !d_result || ((uintptr_t)d_result & 7) || ((uintptr_t)d_pmin_dump & 3)) return GB_EINVAL;
    if (lo > hi || hi > GB_HI_LIMIT || p_max < 3 || p_max > ctx->p_max) return GB_EINVAL;
    const uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return GB_OK;
    if (hi > ctx->hi_max) return GB_ERANGE;
    if (lo_e < ctx->origin || ((hi - ctx->origin) >> 1) >= (1ull << GB_KEY_SHIFT)) return GB_EINVAL;
    const uint32_t n_cand = count_le(ctx->h_primes, p_max);
    if (n_cand == 0) return GB_EINVAL;
    DeviceGuard g(ctx->device);
    // words of the global odd bitset the ctx can sieve: isqrt(q) <= R for every q
    const uint64_t q_cap = (ctx->R + 1) * (ctx->R + 1) - 1;          // largest q with isqrt(q) <= R
    const uint64_t w_cap = q_cap >= 130 ? (q_cap - 130) / 128 : 0;   // words [0, w_cap] fit
    for (uint64_t s0 = lo_e; s0 < hi; s0 += 2 * kPerNSegEvens) {
        const uint64_t s1 = std::min<uint64_t>(hi, s0 + 2 * kPerNSegEvens);
        PerNArgs a;
        a.n_first = s0;
        a.n_evens = (s1 - s0 + 1) / 2;
        // segment bitset: odd q in [s0, s1), word aligned
        const uint64_t qa = s0 > 3 ? s0 - 1 : 3;
        uint64_t w0 = (qa - 3) / 128, w1 = (s1 - 1 - 3) / 128 + 1;
        w1 = std::min<uint64_t>(w1, w_cap + 1);
        if (w1 <= w0) w1 = w0;
        a.seg_bits = ctx->seg_scratch;
        a.seg_word_lo = w0;
        a.seg_q_lo = 3 + 128 * w0;
        a.seg_q_hi = 3 + 128 * w1;
        if (w1 > w0) {
            const gb_status st = gb_sieve_segment(ctx, w0, w1 - w0, ctx->seg_scratch, stream);
            if (st != GB_OK) return st;
        }
        a.n_cand = n_cand;
        a.primes = ctx->primes;
        a.n_base = (uint32_t)ctx->n_base;
        a.base_bits = ctx->bits;
        a.R = ctx->R;
        a.p_fallback = (uint64_t)ctx->h_primes[n_cand - 1] + 2;
        a.cap = UINT64_MAX;
        a.origin = ctx->origin;
        a.lo_e = lo_e;
        a.result = d_result;
        a.dump = d_pmin_dump;
        if (launch_pern(a, S(stream)) != cudaSuccess) return GB_ECUDA;
    }
    return GB_OK;
}

gb_status gb_verify_range_resident(gb_ctx *ctx, uint64_t lo, uint64_t hi, uint32_t p_max, const uint64_t *d_bits,
                                   uint64_t n_words, int64_t *d_result, uint32_t *d_pmin_dump, void *stream)
{
    if (!ctx || !d_result || !d_bits || ((uintptr_t)d_result & 7) || ((uintptr_t)d_bits & 7) ||
        ((uintptr_t)d_pmin_dump & 3))
        return GB_EINVAL;
    if (lo > hi || hi > GB_HI_LIMIT || p_max < 3 || p_max > ctx->p_max) return GB_EINVAL;
    const uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return GB_OK;
    if (hi > ctx->hi_max) return GB_ERANGE;
    if (lo_e < ctx->origin || ((hi - ctx->origin) >> 1) >= (1ull << GB_KEY_SHIFT)) return GB_EINVAL;
    if (n_words > (1ull << 58) || 3 + 128 * n_words < hi) return GB_EINVAL;   // every odd q < hi resident
    const uint32_t n_cand = count_le(ctx->h_primes, p_max);
    if (n_cand == 0) return GB_EINVAL;
    DeviceGuard g(ctx->device);
    PerNArgs a;
    a.n_first = lo_e;
    a.n_evens = (hi - lo_e + 1) / 2;
    a.n_cand = n_cand;
    a.primes = ctx->primes;
    a.n_base = (uint32_t)ctx->n_base;
    a.base_bits = ctx->bits;
    a.R = ctx->R;
    a.seg_bits = d_bits;               // the whole range's bitset is the "segment"
    a.seg_word_lo = 0;
    a.seg_q_lo = 3;
    a.seg_q_hi = 3 + 128 * n_words;
    a.p_fallback = (uint64_t)ctx->h_primes[n_cand - 1] + 2;
    a.cap = UINT64_MAX;
    a.origin = ctx->origin;
    a.lo_e = lo_e;
    a.result = d_result;
    a.dump = d_pmin_dump;
    return launch_pern(a, S(stream)) == cudaSuccess ? GB_OK : GB_ECUDA;
}

gb_status gb_partition_counts(gb_ctx *ctx, uint64_t lo, uint64_t hi, const uint64_t *d_bits, uint64_t n_words,
                              uint64_t *d_counts, void *stream)
{
    if (!ctx || ((uintptr_t)d_bits & 7) || ((uintptr_t)d_counts & 7)) return GB_EINVAL;
    if (lo > hi || hi > GB_COUNTS_HI_LIMIT) return GB_EINVAL;
    const uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return GB_OK;                            // empty range: no launch
    if (!d_bits || !d_counts) return GB_EINVAL;
    if (n_words > (1ull << 58) || 3 + 128 * n_words < hi) return GB_EINVAL;   // every odd q < hi present
    DeviceGuard g(ctx->device);
    return launch_counts(d_bits, n_words, lo_e, hi, d_counts, ctx->num_sms, S(stream)) == cudaSuccess ? GB_OK
                                                                                                      : GB_ECUDA;
}

gb_status gb_single_check(gb_ctx *ctx, uint64_t n, uint64_t p_limit, uint64_t *d_out, void *stream)
{
    if (!ctx || !d_out || ((uintptr_t)d_out & 7) || n < 4 || (n & 1)) return GB_EINVAL;
    DeviceGuard g(ctx->device);
    return launch_single_check(n, p_limit, ctx->bits, ctx->R, d_out, S(stream)) == cudaSuccess ? GB_OK : GB_ECUDA;
}

gb_status gb_is_prime_u64(const uint64_t *d_x, uint8_t *d_out, uint64_t n, void *stream)
{
    if (n && (!d_x || !d_out || ((uintptr_t)d_x & 7))) return GB_EINVAL;
    if (n == 0) return GB_OK;
    int dev = -1;
    if (!pointer_device(d_x, dev)) return GB_EINVAL;
    DeviceGuard g(dev);
    return launch_is_prime(d_x, d_out, n, nullptr, 0, S(stream)) == cudaSuccess ? GB_OK : GB_ECUDA;
}

}  // extern "C"
