/*
 * gb_oracle.c -- plain, slow, obviously-correct CPU oracle for the minimal
 * Goldbach prime of every even n in a range.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2603_02621_b200/, libgb.so) never touches it, and
 * the two share no source, header, table or helper.
 *
 * What it computes (section 2.1, lines 37-39, "CPU Baseline"):
 *   "A segmented Sieve of Eratosthenes generates all primes up to N. For each
 *    even integer n in [4,N], the verifier scans primes p from 2 to n/2 and
 *    checks whether q = n - p is prime via direct bitset lookup."
 * i.e. for each even n >= 4:
 *      p_min(n) = min{ p prime : n - p prime },  searched for p <= n/2.
 * The result is exact (no approximation), so the oracle is that definition
 * written out: a byte-per-odd segmented sieve and a forward scan of p.
 *
 * Deliberate independence from the GPU path:
 *   - byte arrays, never bit words;
 *   - a forward p-scan per n, never the inverted (bulk-marking) loop;
 *   - trial division (never Miller-Rabin) whenever q falls below the
 *     sieved window or p exceeds the small-prime table.
 *
 * Readings of the paper this file implements (listed in DESIGN.md):
 *   R1 range: the API is half-open [lo, hi); the paper's "n in [4, N]" is
 *      lo = 4, hi = N + 1 (counts N/2 - 1 at PAPER.md:276-279).
 *   R2 p = 2 only resolves n = 4 (n - 2 is even and > 2 otherwise).
 *   R3 a counterexample is an n with no prime p <= n/2 (or <= the optional
 *      test cap) such that n - p is prime: reported, never swallowed
 *      (SPEC.md:209 NOT_FOUND convention).
 *   R4 "fastpath_unresolved" = number of n whose p_min exceeds p_fast (the
 *      paper's Phase-2 invocations) -- counted here
 *      purely from p_min, not from any fast path.
 *   R5 aggregates: histogram of p_min by prime index (bin 0 = unresolved,
 *      bin i = i-th prime, p_1 = 2, ..., p_6542 = 65521, bin 6543 = larger),
 *      max p_min with the SMALLEST n attaining it (A025018 convention),
 *      sum of p_min, and the checksum chk = sum of n * p_min(n) mod 2^64
 *      (the paper defines none; R6): a p_min
 *      placed on the wrong n changes it; optionally chk per chunk of 2^k evens
 *      counted from lo_e (chunk_chk), so full-range goldens can be compared
 *      piece by piece.
 *
 * Build: gcc -O2 -std=c11 -pthread -shared -fPIC gb_oracle.c -o liboracle.so
 */
#define _POSIX_C_SOURCE 200809L
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_NBINS 6544            /* 0 unresolved, 1..6542 primes <= 65521, 6543 overflow */
#define OR_BIN_PRIME_MAX 65521u  /* largest prime < 2^16 */
#define OR_WINDOW_BELOW 20000u   /* sieved odds kept below each segment */

typedef struct {
    int64_t evens;
    int64_t verified;
    int64_t fastpath_unresolved;
    int64_t unresolved;
    int64_t first_unresolved_n;  /* INT64_MAX if none */
    int64_t max_pmin;            /* 0 if no verified n */
    int64_t max_pmin_n;          /* smallest n with p_min == max_pmin */
    int64_t sum_pmin;
    uint64_t chk;                /* sum n * p_min(n)             mod 2^64 */
    int64_t hist[OR_NBINS];
} or_result;

/* ------------------------------------------------------------------ */
/* integer square root: largest r with r*r <= x (exact, 128-bit check) */
uint64_t or_isqrt(uint64_t x)
{
    uint64_t lo = 0, hi = 4294967296ull;      /* answer < 2^32 */
    while (hi - lo > 1) {                     /* invariant: lo^2 <= x < hi^2 */
        uint64_t mid = lo + (hi - lo) / 2;
        unsigned __int128 sq = (unsigned __int128)mid * mid;
        if (sq <= x) lo = mid; else hi = mid;
    }
    return lo;
}

/* trial division: the textbook definition of primality */
int or_is_prime_td(uint64_t x)
{
    if (x < 2) return 0;
    if (x < 4) return 1;
    if (x % 2 == 0) return 0;
    for (uint64_t d = 3; d <= x / d; d += 2)
        if (x % d == 0) return 0;
    return 1;
}

/* ------------------------------------------------------------------ */
/* Small primes: simple Eratosthenes, one byte per integer 0..R.        */
typedef struct {
    uint64_t R;
    uint8_t *isp;       /* isp[i] = 1 iff i prime, i <= R */
    uint32_t *odd;      /* odd primes <= R ascending */
    uint64_t n_odd;
    uint32_t *binp;     /* all primes <= 65521 ascending (2 first), for binning */
    uint64_t n_binp;
} small_primes;

static int small_primes_make(small_primes *sp, uint64_t R)
{
    if (R < OR_BIN_PRIME_MAX) R = OR_BIN_PRIME_MAX;
    sp->R = R;
    sp->isp = (uint8_t *)malloc(R + 1);
    if (!sp->isp) return -1;
    memset(sp->isp, 1, R + 1);
    sp->isp[0] = sp->isp[1] = 0;
    for (uint64_t i = 2; i * i <= R; i++)
        if (sp->isp[i])
            for (uint64_t m = i * i; m <= R; m += i) sp->isp[m] = 0;
    uint64_t c = 0, cb = 0;
    for (uint64_t i = 3; i <= R; i += 2) c += sp->isp[i];
    for (uint64_t i = 2; i <= OR_BIN_PRIME_MAX; i++) cb += sp->isp[i];
    sp->odd = (uint32_t *)malloc(sizeof(uint32_t) * (c + 1));
    sp->binp = (uint32_t *)malloc(sizeof(uint32_t) * (cb + 1));
    if (!sp->odd || !sp->binp) return -1;
    sp->n_odd = 0;
    for (uint64_t i = 3; i <= R; i += 2)
        if (sp->isp[i]) sp->odd[sp->n_odd++] = (uint32_t)i;
    sp->n_binp = 0;
    for (uint64_t i = 2; i <= OR_BIN_PRIME_MAX; i++)
        if (sp->isp[i]) sp->binp[sp->n_binp++] = (uint32_t)i;
    return 0;
}

static void small_primes_free(small_primes *sp)
{
    free(sp->isp); free(sp->odd); free(sp->binp);
}

/* histogram bin of a prime p (R5): 1-based index among all primes, or overflow */
static int bin_of(const small_primes *sp, uint64_t p)
{
    if (p > OR_BIN_PRIME_MAX) return OR_NBINS - 1;
    uint64_t lo = 0, hi = sp->n_binp;         /* binary search for p in binp */
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (sp->binp[mid] < p) lo = mid + 1; else hi = mid;
    }
    return (int)(lo + 1);                     /* binp[0] = 2 -> bin 1 */
}

/* ------------------------------------------------------------------ */
/* Segment sieve: comp[(q - wlo)/2] = 1 iff odd q in [wlo, whi) composite.
 * wlo odd >= 3.  Base primes: odd primes p <= isqrt(whi - 1).             */
static void sieve_odd_window(const small_primes *sp, uint64_t wlo, uint64_t whi,
                             uint8_t *comp)
{
    uint64_t len = (whi - wlo + 1) / 2;       /* odd q in [wlo, whi) */
    memset(comp, 0, len);
    if (whi <= wlo) return;
    uint64_t lim = or_isqrt(whi - 1);
    for (uint64_t i = 0; i < sp->n_odd; i++) {
        uint64_t p = sp->odd[i];
        if (p > lim) break;
        uint64_t m = ((wlo + p - 1) / p) * p;  /* first multiple >= wlo */
        if (m < p * p) m = p * p;              /* never clear p itself */
        if (m % 2 == 0) m += p;                /* odd multiples only */
        for (; m < whi; m += 2 * p) comp[(m - wlo) / 2] = 1;
    }
}

/* ------------------------------------------------------------------ */
typedef struct {
    const small_primes *sp;
    uint64_t lo_e, hi;          /* even n in [lo_e, hi) */
    uint64_t seg_evens;
    uint64_t p_fast, cap;
    int tid, nthreads;
    uint32_t *dump;             /* may be NULL; index (n - lo_e)/2 */
    uint64_t *chunk_chk;        /* may be NULL; chk per chunk_evens evens from lo_e */
    uint64_t chunk_evens;
    uint64_t seg_chk;           /* chk of the current segment */
    or_result res;
    int err;
} worker;

static void result_clear(or_result *r)
{
    memset(r, 0, sizeof(*r));
    r->first_unresolved_n = INT64_MAX;
}

/* is q prime?  from the window bytes if q >= wlo, else trial division */
static int q_is_prime(uint64_t q, uint64_t wlo, const uint8_t *comp)
{
    if (q >= wlo) return comp[(q - wlo) / 2] == 0;
    return or_is_prime_td(q);
}

/* record the outcome for one even n (p = 0 means unresolved) */
static void record(worker *w, uint64_t n, uint64_t p)
{
    or_result *r = &w->res;
    r->evens++;
    if (w->dump) w->dump[(n - w->lo_e) / 2] = (uint32_t)p;
    if (p == 0) {
        r->unresolved++;
        r->fastpath_unresolved++;
        r->hist[0]++;
        if ((int64_t)n < r->first_unresolved_n) r->first_unresolved_n = (int64_t)n;
        return;
    }
    r->verified++;
    if (p > w->p_fast) r->fastpath_unresolved++;
    r->hist[bin_of(w->sp, p)]++;
    r->sum_pmin += (int64_t)p;
    r->chk += n * p;                           /* wraps mod 2^64 */
    w->seg_chk += n * p;
    if ((int64_t)p > r->max_pmin || ((int64_t)p == r->max_pmin && (int64_t)n < r->max_pmin_n)) {
        r->max_pmin = (int64_t)p;
        r->max_pmin_n = (int64_t)n;
    }
}

static void *worker_main(void *arg)
{
    worker *w = (worker *)arg;
    const small_primes *sp = w->sp;
    uint64_t span = w->hi - w->lo_e;                       /* integers */
    uint64_t nseg = (span + 2 * w->seg_evens - 1) / (2 * w->seg_evens);
    uint8_t *comp = (uint8_t *)malloc(w->seg_evens + OR_WINDOW_BELOW / 2 + 4);
    if (!comp) { w->err = 1; return NULL; }
    for (uint64_t s = (uint64_t)w->tid; s < nseg; s += (uint64_t)w->nthreads) {
        uint64_t n0 = w->lo_e + s * 2 * w->seg_evens;
        uint64_t n1 = n0 + 2 * w->seg_evens;
        if (n1 > w->hi) n1 = w->hi;
        uint64_t wlo = (n0 > 3 + OR_WINDOW_BELOW) ? n0 - OR_WINDOW_BELOW : 3;
        if (wlo % 2 == 0) wlo -= 1;
        sieve_odd_window(sp, wlo, n1, comp);
        w->seg_chk = 0;
        for (uint64_t n = n0; n < n1; n += 2) {
            uint64_t found = 0;
            if (n == 4) {
                found = 2;                                  /* R2 */
            } else {
                /* forward scan over odd primes p = 3, 5, 7, ... , p <= n/2 */
                uint64_t i = 0, p = sp->odd[0];
                for (;;) {
                    if (p > n / 2 || p > w->cap) break;     /* R3 */
                    if (q_is_prime(n - p, wlo, comp)) { found = p; break; }
                    i++;                                    /* next odd prime */
                    if (i < sp->n_odd) {
                        p = sp->odd[i];
                    } else {                                /* past the table: trial division */
                        p += 2;
                        while (!or_is_prime_td(p)) p += 2;
                    }
                }
            }
            record(w, n, found);
        }
        if (w->chunk_chk)                           /* a segment lies inside one chunk */
            __atomic_fetch_add(&w->chunk_chk[(n0 - w->lo_e) / 2 / w->chunk_evens], w->seg_chk,
                               __ATOMIC_RELAXED);
    }
    free(comp);
    return NULL;
}

static void merge(or_result *a, const or_result *b)
{
    a->evens += b->evens;
    a->verified += b->verified;
    a->fastpath_unresolved += b->fastpath_unresolved;
    a->unresolved += b->unresolved;
    if (b->first_unresolved_n < a->first_unresolved_n) a->first_unresolved_n = b->first_unresolved_n;
    if (b->max_pmin > a->max_pmin || (b->max_pmin == a->max_pmin && b->max_pmin_n < a->max_pmin_n)) {
        a->max_pmin = b->max_pmin;
        a->max_pmin_n = b->max_pmin_n;
    }
    a->sum_pmin += b->sum_pmin;
    a->chk += b->chk;
    for (int i = 0; i < OR_NBINS; i++) a->hist[i] += b->hist[i];
}

/*
 * or_verify: p_min for every even n with lo <= n < hi and n >= 4.
 *   p_fast   : threshold for fastpath_unresolved (R4)
 *   cap      : test hook -- scan p only up to cap (UINT64_MAX = unbounded)
 *   threads  : worker threads (>= 1)
 *   out      : aggregates (R5)
 *   dump     : optional u32 per even n, index (n - lo_e)/2, lo_e = max(4, lo
 *              rounded up to even); value p_min, 0 = unresolved.
 *   chunk_chk: optional; chunk_chk[c] = chk over the evens with index (n - lo_e)/2
 *              in [c * chunk_evens, (c + 1) * chunk_evens); the caller zeroes
 *              ceil(evens / chunk_evens) entries.  chunk_evens: a power of two.
 * Returns 0 on success, -1 on allocation failure, -2 on bad arguments.
 */
int or_verify(uint64_t lo, uint64_t hi, uint64_t p_fast, uint64_t cap, int threads,
              or_result *out, uint32_t *dump, uint64_t *chunk_chk, uint64_t chunk_evens)
{
    result_clear(out);
    if (threads < 1) threads = 1;
    uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return 0;                               /* empty range */
    if (hi > (1ull << 62)) return -2;
    uint64_t seg_evens = 1u << 22;
    if (chunk_chk) {
        if (chunk_evens == 0 || (chunk_evens & (chunk_evens - 1))) return -2;
        if (chunk_evens < seg_evens) seg_evens = chunk_evens;   /* segments nest in chunks */
    }
    small_primes sp;
    if (small_primes_make(&sp, or_isqrt(hi - 1) + 1) != 0) return -1;
    worker *ws = (worker *)calloc((size_t)threads, sizeof(worker));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    if (!ws || !th) { small_primes_free(&sp); free(ws); free(th); return -1; }
    for (int t = 0; t < threads; t++) {
        ws[t].sp = &sp; ws[t].lo_e = lo_e; ws[t].hi = hi;
        ws[t].seg_evens = seg_evens;
        ws[t].p_fast = p_fast; ws[t].cap = cap;
        ws[t].tid = t; ws[t].nthreads = threads; ws[t].dump = dump;
        ws[t].chunk_chk = chunk_chk; ws[t].chunk_evens = chunk_evens;
        result_clear(&ws[t].res);
        pthread_create(&th[t], NULL, worker_main, &ws[t]);
    }
    int err = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        err |= ws[t].err;
        merge(out, &ws[t].res);
    }
    free(ws); free(th);
    small_primes_free(&sp);
    return err ? -1 : 0;
}

/*
 * or_sieve_window: one byte per odd q in [a, b) (a odd >= 3): 1 iff q prime.
 * out must hold (b - a + 1)/2 bytes.  Returns 0, or -1 on allocation failure.
 */
int or_sieve_window(uint64_t a, uint64_t b, uint8_t *out)
{
    if (b <= a) return 0;
    if (a < 3 || a % 2 == 0) return -2;
    small_primes sp;
    if (small_primes_make(&sp, or_isqrt(b - 1) + 1) != 0) return -1;
    uint64_t len = (b - a + 1) / 2;
    sieve_odd_window(&sp, a, b, out);
    for (uint64_t i = 0; i < len; i++) out[i] = (uint8_t)(out[i] == 0);
    small_primes_free(&sp);
    return 0;
}

/* ---- prime counting pi(x), threaded over windows of odds ---------- */
typedef struct {
    const small_primes *sp;
    uint64_t x, chunk;
    int tid, nthreads;
    uint64_t count;
    int err;
} pi_worker;

static void *pi_main(void *arg)
{
    pi_worker *w = (pi_worker *)arg;
    uint8_t *comp = (uint8_t *)malloc(w->chunk / 2 + 2);
    if (!comp) { w->err = 1; return NULL; }
    uint64_t nch = (w->x - 3 + 1 + w->chunk - 1) / w->chunk;   /* windows over [3, x] */
    for (uint64_t c = (uint64_t)w->tid; c < nch; c += (uint64_t)w->nthreads) {
        uint64_t a = 3 + c * w->chunk;                          /* chunk is even, so a odd */
        uint64_t b = a + w->chunk;
        if (b > w->x + 1) b = w->x + 1;
        sieve_odd_window(w->sp, a, b, comp);
        uint64_t len = (b - a + 1) / 2;
        for (uint64_t i = 0; i < len; i++) w->count += (comp[i] == 0);
    }
    free(comp);
    return NULL;
}

/* pi(x) = number of primes <= x; returns UINT64_MAX on failure */
uint64_t or_prime_pi(uint64_t x, int threads)
{
    if (x < 2) return 0;
    if (x < 3) return 1;
    if (threads < 1) threads = 1;
    small_primes sp;
    if (small_primes_make(&sp, or_isqrt(x) + 1) != 0) return UINT64_MAX;
    pi_worker *ws = (pi_worker *)calloc((size_t)threads, sizeof(pi_worker));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    uint64_t total = 1;                                         /* the prime 2 */
    int err = 0;
    for (int t = 0; t < threads; t++) {
        ws[t].sp = &sp; ws[t].x = x; ws[t].chunk = 1u << 24;
        ws[t].tid = t; ws[t].nthreads = threads;
        pthread_create(&th[t], NULL, pi_main, &ws[t]);
    }
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        total += ws[t].count;
        err |= ws[t].err;
    }
    free(ws); free(th);
    small_primes_free(&sp);
    return err ? UINT64_MAX : total;
}

/* ---- Goldbach partition counts c(n) ------------------------------------
 * NEXT-4 (section 4.5 "large-scale computation
 * of Goldbach partition counts c(n)").  The paper does not define c(n); reading
 * R13: the number of unordered partitions, the Goldbach-comet count
 *      c(n) = #{ p prime : p <= n/2 and n - p prime }    (c(4) = 1: 2 + 2).
 * Written out plainly: a byte-per-integer sieve of [0, hi) and, for each even n,
 * a scan of the primes p <= n/2 with a byte lookup of n - p.                  */
typedef struct {
    const uint8_t *isp;
    const uint32_t *pr;         /* primes ascending (2 first) */
    uint64_t npr;
    uint64_t lo_e, hi;
    int tid, nthreads;
    uint64_t *out;
} cn_worker;

static void *cn_main(void *arg)
{
    cn_worker *w = (cn_worker *)arg;
    uint64_t k = 0;
    for (uint64_t n = w->lo_e; n < w->hi; n += 2, ++k) {
        if ((int)(k % (uint64_t)w->nthreads) != w->tid) continue;
        uint64_t c = 0;
        for (uint64_t i = 0; i < w->npr && w->pr[i] <= n / 2; ++i)
            c += w->isp[n - w->pr[i]];
        w->out[k] = c;
    }
    return NULL;
}

/* out[(n - lo_e)/2] = c(n) for every even n in [lo_e, hi), lo_e = max(4, lo
 * rounded up to even).  Returns 0, -1 on allocation failure, -2 if hi > 2^36. */
int or_partition_counts(uint64_t lo, uint64_t hi, int threads, uint64_t *out)
{
    uint64_t lo_e = lo < 4 ? 4 : lo + (lo & 1);
    if (hi <= lo_e) return 0;
    if (hi > (1ull << 36)) return -2;
    if (threads < 1) threads = 1;
    uint8_t *isp = (uint8_t *)malloc(hi);
    if (!isp) return -1;
    memset(isp, 1, hi);
    isp[0] = 0;
    if (hi > 1) isp[1] = 0;
    for (uint64_t i = 2; i * i < hi; i++)
        if (isp[i])
            for (uint64_t m = i * i; m < hi; m += i) isp[m] = 0;
    uint64_t npr = 0;
    for (uint64_t i = 2; i <= hi / 2; i++) npr += isp[i];
    uint32_t *pr = (uint32_t *)malloc(sizeof(uint32_t) * (npr + 1));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    cn_worker *ws = (cn_worker *)calloc((size_t)threads, sizeof(cn_worker));
    if (!pr || !th || !ws) { free(isp); free(pr); free(th); free(ws); return -1; }
    npr = 0;
    for (uint64_t i = 2; i <= hi / 2; i++)
        if (isp[i]) pr[npr++] = (uint32_t)i;
    for (int t = 0; t < threads; t++) {
        ws[t].isp = isp; ws[t].pr = pr; ws[t].npr = npr;
        ws[t].lo_e = lo_e; ws[t].hi = hi; ws[t].tid = t; ws[t].nthreads = threads; ws[t].out = out;
        pthread_create(&th[t], NULL, cn_main, &ws[t]);
    }
    for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    free(isp); free(pr); free(th); free(ws);
    return 0;
}

int or_nbins(void) { return OR_NBINS; }
size_t or_result_size(void) { return sizeof(or_result); }
