// peaks_int.cu -- measured B200 throughput of the integer / shared-memory / L2
// operations the Goldbach path is built from (SURVEY.md 8(d) "Micro-benchmarked
// peaks"), as roofline denominators for bench.py.  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_int peaks_int.cu
//
// Every throughput kernel runs one 1024-thread CTA per SM on all SMs, each thread
// with 8 INDEPENDENT dependency chains (ILP 8), so the number measures issue /
// pipe throughput, not latency.  Rates are lane-ops per clock per SM (clock64()
// cycles of the CTA between two barriers), and device-wide ops/s at the clock
// measured over the same kernels (cycles / event time).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));             \
            return 1;                                                            \
        }                                                                        \
    } while (0)

constexpr int kT = 1024;
constexpr int kIlp = 8;

enum Op { LOP3, SHF, IADD3, IMAD, POPC, MARK, RED_SHARED, LDS128, ATOM_SHARED_ADD, NOPS };
static const char *kName[NOPS] = {"lop3", "shf", "iadd3", "imad", "popc", "mark_step", "red_shared_and",
                                  "lds128", "atom_shared_add"};
// lane-ops per inner step per chain
static const int kOpsPerStep[NOPS] = {1, 1, 1, 1, 1, 3, 1, 1, 1};

template <int OP>
__global__ void __launch_bounds__(kT) k_pipe(uint32_t *out, uint64_t *cyc, int iters, uint32_t seed)
{
    __shared__ uint32_t sm[8192];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < 8192; i += kT) sm[i] = 0xFFFFFFFFu ^ i;
    uint32_t x[kIlp], y = seed ^ tid, z = seed * 7 + lane;
#pragma unroll
    for (int k = 0; k < kIlp; ++k) x[k] = tid * 2654435761u + k * 40503u + seed;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kIlp; ++k) {
            if constexpr (OP == LOP3) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(y), "r"(z));
            } else if constexpr (OP == SHF) {
                asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(y), "r"(z));
            } else if constexpr (OP == IADD3) {
                asm volatile("add.u32 %0, %0, %1;" : "+r"(x[k]) : "r"(y));
            } else if constexpr (OP == IMAD) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(y), "r"(z));
            } else if constexpr (OP == POPC) {
                asm volatile("popc.b32 %0, %0;" : "+r"(x[k]));
            } else if constexpr (OP == MARK) {
                // the inverted-loop step: S = shf(lo, hi, b); new = U & S; U ^= new
                uint32_t s, nw;
                asm volatile("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(s) : "r"(y), "r"(z), "r"(k + i));
                asm volatile("and.b32 %0, %1, %2;" : "=r"(nw) : "r"(x[k]), "r"(s));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(x[k]) : "r"(nw));
            } else if constexpr (OP == RED_SHARED) {
                // conflict-free: lane l of the warp hits bank (l + 8k + i) mod 32
                const uint32_t a = sbase + 4 * (((uint32_t)(lane + 8 * k + i) & 31) + 32 * ((tid >> 5) & 63));
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(x[k]) : "memory");
            } else if constexpr (OP == ATOM_SHARED_ADD) {
                const uint32_t a = sbase + 4 * (((uint32_t)(lane + 8 * k + i) & 31) + 32 * ((tid >> 5) & 63));
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(x[k] & 7u) : "memory");
            } else if constexpr (OP == LDS128) {
                uint4 v;
                const uint32_t a = sbase + 16 * (((uint32_t)(lane + 8 * k + i) & 31) + 32 * ((tid >> 5) & 15));
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(a));
                x[k] ^= v.x ^ v.w;
            }
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < kIlp; ++k) acc ^= x[k];
    if (acc == 0x12345678u) out[tid] = acc + sm[tid];
    if (tid == 0) cyc[blockIdx.x] = (uint64_t)(t1 - t0);
}

// no-return AND atomics to global memory (L2): `n` u32 words (L2-resident when
// small), pseudo-random word per (thread, step)
__global__ void __launch_bounds__(256) k_red_global(uint32_t *buf, uint32_t nmask, int iters, uint32_t seed)
{
    uint32_t h = (blockIdx.x * 256 + threadIdx.x) * 2654435761u + seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kIlp; ++k) {
            h = h * 1664525u + 1013904223u;
            asm volatile("red.global.and.b32 [%0], %1;" ::"l"(buf + ((h >> 3) & nmask)), "r"(~(1u << (h & 31)))
                         : "memory");
        }
    }
}

__global__ void k_fill(uint32_t *b, uint64_t n)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = 0xFFFFFFFFu;
}

template <int OP>
static int run_pipe(int sms, int iters, double &per_sm, double &mhz)
{
    uint32_t *out;
    uint64_t *cyc;
    CK(cudaMalloc(&out, 4 * kT));
    CK(cudaMalloc(&cyc, 8 * sms));
    k_pipe<OP><<<sms, kT>>>(out, cyc, 64, 1);   // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_pipe<OP><<<sms, kT>>>(out, cyc, iters, 2);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<uint64_t> c(sms);
    CK(cudaMemcpy(c.data(), cyc, 8 * sms, cudaMemcpyDeviceToHost));
    uint64_t cmax = 0;
    for (uint64_t v : c) cmax = v > cmax ? v : cmax;
    const double ops = (double)kT * iters * kIlp * kOpsPerStep[OP];
    per_sm = ops / (double)cmax;
    mhz = (double)cmax / (ms * 1e3);            // lower bound: the event brackets launch overhead too
    cudaFree(out);
    cudaFree(cyc);
    return 0;
}

int main()
{
    int dev = 0, sms = 0, clk_khz = 0, l2 = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    printf("{\n \"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"how\": \"scripts/micro/peaks_int.cu: one 1024-thread CTA "
           "per SM, 8 independent chains per thread; lane-ops/clk/SM from clock64 cycles between barriers\",\n",
           prop.name, sms, l2);
    printf(" \"per_sm_lane_ops_per_clk\": {");
    double mhz_min = 1e9, mhz_max = 0;
    double rates[NOPS];
    for (int op = 0; op < NOPS; ++op) {
        double r = 0, mhz = 0;
        int rc = 0;
        const int iters = 4096;
        switch (op) {
        case LOP3: rc = run_pipe<LOP3>(sms, iters, r, mhz); break;
        case SHF: rc = run_pipe<SHF>(sms, iters, r, mhz); break;
        case IADD3: rc = run_pipe<IADD3>(sms, iters, r, mhz); break;
        case IMAD: rc = run_pipe<IMAD>(sms, iters, r, mhz); break;
        case POPC: rc = run_pipe<POPC>(sms, iters, r, mhz); break;
        case MARK: rc = run_pipe<MARK>(sms, iters, r, mhz); break;
        case RED_SHARED: rc = run_pipe<RED_SHARED>(sms, iters, r, mhz); break;
        case LDS128: rc = run_pipe<LDS128>(sms, iters, r, mhz); break;
        case ATOM_SHARED_ADD: rc = run_pipe<ATOM_SHARED_ADD>(sms, iters, r, mhz); break;
        }
        if (rc) return rc;
        rates[op] = r;
        mhz_min = mhz < mhz_min ? mhz : mhz_min;
        mhz_max = mhz > mhz_max ? mhz : mhz_max;
        printf("%s\"%s\": %.3f", op ? ", " : "", kName[op], r);
    }
    printf("},\n");
    printf(" \"lds128_bytes_per_clk_per_sm\": %.1f,\n", rates[LDS128] * 16);
    printf(" \"clock_mhz_measured\": [%.0f, %.0f], \"clock_mhz_attr\": %.0f,\n", mhz_min, mhz_max, clk_khz / 1e3);

    // L2 atomics: red.global.and into an L2-resident buffer (32 MB) and into a
    // DRAM-sized one (1 GB), pseudo-random words
    printf(" \"red_global_and_per_s\": {");
    const uint64_t sizes[2] = {1ull << 23, 1ull << 28};   // u32 words: 32 MB, 1 GB
    for (int s = 0; s < 2; ++s) {
        uint32_t *buf;
        CK(cudaMalloc(&buf, 4 * sizes[s]));
        k_fill<<<4 * sms, 256>>>(buf, sizes[s]);
        const int blocks = 8 * sms, iters = 256;
        k_red_global<<<blocks, 256>>>(buf, (uint32_t)(sizes[s] - 1), 16, 1);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_red_global<<<blocks, 256>>>(buf, (uint32_t)(sizes[s] - 1), iters, 2);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = (double)blocks * 256 * iters * kIlp;
        printf("%s\"%s\": %.4g", s ? ", " : "", s ? "buffer_1GB" : "buffer_32MB_l2", n / (ms * 1e-3));
        cudaFree(buf);
    }
    printf("}\n}\n");
    return 0;
}
