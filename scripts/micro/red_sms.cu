// red_sms.cu -- is the K-LARGE cost (no-return red.global.and.b32 into an
// L2-resident mask) bound by the L2 or by the SMs issuing it?
// Rate of random 32-bit REDs into a 64 MB / 96 MB buffer with the grid confined to
// G SMs (one 1024-thread CTA per SM, forced by a 150 KB dynamic shared-memory
// request), G = 8 .. all SMs; then the same on G SMs while a compute-bound kernel
// occupies the other SMs (the overlap a split verify / K-LARGE schedule would see).
// Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_sms red_sms.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));             \
            return 1;                                                            \
        }                                                                        \
    } while (0)

constexpr int kT = 1024;
constexpr size_t kPin = 150 * 1024;   // one CTA per SM

__global__ void __launch_bounds__(kT) k_red(uint32_t *buf, uint32_t nwords, int iters, uint32_t seed)
{
    extern __shared__ uint32_t pin[];
    if (iters < 0) pin[threadIdx.x] = 0;   // never: keeps the allocation
    uint32_t x = (blockIdx.x * kT + threadIdx.x) * 2654435761u + seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x = x * 1664525u + 1013904223u;
            const uint32_t w = __umulhi(x, nwords);
            asm volatile("red.global.and.b32 [%0], %1;" ::"l"(buf + w), "r"(~(1u << (x & 31))) : "memory");
        }
    }
}

// compute-bound filler: one 1024-thread CTA per SM, spins on ALU for `iters`
__global__ void __launch_bounds__(kT) k_spin(uint32_t *out, int iters)
{
    extern __shared__ uint32_t pin[];
    uint32_t a = threadIdx.x, b = blockIdx.x, c = 7;
    for (int i = 0; i < iters; ++i) {
        a = a * 3 + b;
        b = b ^ (a >> 3);
        c += a & b;
    }
    if (c == 0x12345678u) { out[0] = a; pin[0] = b; }
}

int main()
{
    int dev = 0, sms = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaFuncSetAttribute(k_red, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPin));
    CK(cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPin));
    const size_t sizes_mb[2] = {64, 96};
    uint32_t *buf = nullptr, *out = nullptr;
    CK(cudaMalloc(&buf, 96u << 20));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(buf, 0xFF, 96u << 20));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int gs[] = {8, 16, 24, 32, 48, 64, 96, 128, sms};
    printf("{\"sms\": %d, \"threads_per_cta\": %d, \"reds_per_s\": {", sms, kT);
    for (int si = 0; si < 2; ++si) {
        const uint32_t nw = (uint32_t)((sizes_mb[si] << 20) / 4);
        printf("%s\"%zuMB\": {", si ? ", " : "", sizes_mb[si]);
        for (int gi = 0; gi < (int)(sizeof(gs) / sizeof(gs[0])); ++gi) {
            const int g = gs[gi];
            const int iters = 64;
            k_red<<<g, kT, kPin, s1>>>(buf, nw, 4, 1);   // warm (pulls the buffer into L2)
            CK(cudaStreamSynchronize(s1));
            CK(cudaEventRecord(e0, s1));
            k_red<<<g, kT, kPin, s1>>>(buf, nw, iters, 2 + gi);
            CK(cudaEventRecord(e1, s1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double reds = (double)g * kT * iters * 8;
            printf("%s\"%d\": %.4g", gi ? ", " : "", g, reds / (ms * 1e-3));
        }
        printf("}");
    }
    printf("}, \"reds_per_s_beside_spin\": {");
    // G SMs of REDs while (sms - G) SMs spin: spin launched first so it takes its SMs
    const uint32_t nw = (uint32_t)((64u << 20) / 4);
    const int gs2[] = {16, 24, 32, 48};
    for (int gi = 0; gi < 4; ++gi) {
        const int g = gs2[gi];
        k_spin<<<sms - g, kT, kPin, s2>>>(out, 4000000);
        k_red<<<g, kT, kPin, s1>>>(buf, nw, 4, 1);
        CK(cudaEventRecord(e0, s1));
        k_red<<<g, kT, kPin, s1>>>(buf, nw, 64, 9 + gi);
        CK(cudaEventRecord(e1, s1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        CK(cudaDeviceSynchronize());
        printf("%s\"%d\": %.4g", gi ? ", " : "", g, (double)g * kT * 64 * 8 / (ms * 1e-3));
    }
    printf("}}\n");
    CK(cudaGetLastError());
    return 0;
}
