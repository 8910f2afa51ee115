// Microbenchmark: shared-memory RED.AND throughput on one SM (conflict-free warp
// addresses), vs plain LDS+STS read-modify-write, vs LOP3 issue.  Used to bound the
// sieve phase of verify_kernel.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
__global__ void __launch_bounds__(1024) k_red(uint32_t *out, int iters, int mode)
{
    __shared__ uint32_t w[8192];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 8192; i += 1024) w[i] = 0xFFFFFFFFu;
    __syncthreads();
    const uint32_t p = 37 + 2 * warp;                  // odd stride: distinct banks per warp
    uint32_t a = (lane * p) & 8191, acc = 0;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(w);
    long long t0 = clock64();
    if (mode == 0) {
        for (int i = 0; i < iters; ++i) {
            asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(base + 4 * a), "r"(~(1u << (i & 31))) : "memory");
            a = (a + 32 * p) & 8191;
        }
    } else if (mode == 1) {
        for (int i = 0; i < iters; ++i) {
            w[a] &= ~(1u << (i & 31));
            a = (a + 32 * p) & 8191;
        }
    } else if (mode == 3) {
        // 2 of 3 lanes active per RED (rotating): does the atomic unit cost scale with lanes?
        const uint32_t pat = 0xB6DB6DB6u >> (lane % 3);     // 2 of every 3 bits set, lane-shifted
        for (int i = 0; i < iters; ++i) {
            if ((pat >> (i & 31)) & 1)
                asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(base + 4 * a), "r"(~(1u << (i & 31))) : "memory");
            a = (a + 32 * p) & 8191;
        }
    } else {
        uint32_t x = tid, y = lane;
        for (int i = 0; i < iters; ++i) {
            x = __funnelshift_l(x, y, i & 31) ^ y;
            y = (y & x) | i;
        }
        acc = x + y;
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (uint32_t)(t1 - t0);
    if (acc == 12345) out[1000] = w[0];
}
int main()
{
    uint32_t *d;
    cudaMalloc(&d, 8192);
    const int iters = 4096;
    for (int mode = 0; mode < 4; ++mode) {
        k_red<<<148, 1024>>>(d, iters, mode);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("kernel error\n"); return 1; }
        uint32_t c;
        cudaMemcpy(&c, d, 4, cudaMemcpyDeviceToHost);
        const double ops = 1024.0 * iters;
        printf("mode %d (%s): %u cycles, %.2f lane-ops/clk/SM\n", mode,
               mode == 0 ? "red.shared.and" : mode == 1 ? "lds+and+sts" : mode == 2 ? "shf+lop3 x3" : "red, 2/3 lanes", c,
               ops / c);
    }
    return 0;
}
