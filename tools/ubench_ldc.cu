// ubench_ldc.cu -- constant-cache loads with a warp-uniform register address:
// throughput alone and while shared-memory gathers saturate the LSU.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__constant__ uint32_t ctab[256 * 8];

template <int MODE>   // 0: LDC only, 1: LDS only, 2: both
__global__ void k_ldc(uint32_t *out, const uint8_t *cidx, int iters, long long *cycles)
{
    __shared__ uint32_t sm[16 * 385 + 64];
    for (int i = threadIdx.x; i < 16 * 385 + 64; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t row = (lane * 7) & 15;
    uint32_t acc0 = 0, acc1 = 0;
    uint32_t c = cidx[blockIdx.x & 255];
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (MODE != 1) {
                const uint32_t cc = (c + u * 13) & 255;
                uint32_t a, b;
                asm volatile("ld.const.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(&ctab[cc * 8 + (it & 3) * 2]));
                acc0 ^= a ^ b;
            }
            if (MODE != 0) {
                uint32_t v;
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&sm[row * 385 + ((it * 8 + u) & 63)]);
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sa));
                acc1 ^= v;
            }
        }
        c = (c * 5 + 1) & 255;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
}

template <typename K>
static void run(const char *name, K kern, int blocks, int threads, int iters, const uint8_t *cidx)
{
    uint32_t *out; long long *cyc;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaMalloc(&cyc, 8);
    cudaMemset(cyc, 0, 8);
    kern<<<blocks, threads>>>(out, cidx, 16, cyc);
    cudaMemset(cyc, 0, 8);
    kern<<<blocks, threads>>>(out, cidx, iters, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: CUDA error\n", name); exit(1); }
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double wps = (double)blocks * threads / 32 / sms;
    printf("%-12s warp-loads/clk/SM per kind = %6.3f  (cycles %lld)\n", name, wps * iters * 8 / c, c);
    cudaFree(out); cudaFree(cyc);
}

int main()
{
    uint32_t h[256 * 8];
    for (int i = 0; i < 256 * 8; i++) h[i] = i * 2246822519u;
    cudaMemcpyToSymbol(ctab, h, sizeof(h));
    uint8_t *cidx; cudaMalloc(&cidx, 256);
    uint8_t hc[256]; for (int i = 0; i < 256; i++) hc[i] = (uint8_t)(i * 37);
    cudaMemcpy(cidx, hc, 256, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("LDC.64 only", k_ldc<0>, sms * 4, 256, 2048, cidx);
    run("LDS only", k_ldc<1>, sms * 4, 256, 2048, cidx);
    run("LDC+LDS", k_ldc<2>, sms * 4, 256, 2048, cidx);
    return 0;
}
