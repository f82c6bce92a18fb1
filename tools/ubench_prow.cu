// ubench_prow.cu -- probes for the product-row encode kernel (encode_prow.cuh):
//  (1) the shared-window address of the first dynamic shared-memory byte (the
//      kernel places its 64 KiB tables at shared addresses 0x10000 / 0x20000
//      so that one PRMT forms a gather address);
//  (2) throughput of LDS.128 gathers whose address is one PRMT of a data word
//      (row = data byte, 256-B rows, 8 lanes of a quarter-warp on 8 distinct
//      16-B bank slots), i.e. the inner loop of the product-row kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_prow tools/ubench_prow.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void base_kernel(uint32_t *out)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    if (threadIdx.x == 0) out[0] = (uint32_t)__cvta_generic_to_shared(dsm);
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}

// 512 threads; table at shared [0x10000, 0x20000) (dynamic smem of 0x20000 B
// minus the base); every lane: 4 gathers per data word, data words from an LCG.
template <bool CONFLICT_FREE>
__global__ void __launch_bounds__(512, 1) gather_kernel(uint32_t *out, int iters, long long *cycles)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(dsm);
    for (uint32_t a = 0x10000u + threadIdx.x * 16u; a < 0x20000u; a += blockDim.x * 16u) {
        const uint32_t v = a * 2654435761u;
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" :: "r"(a), "r"(v));
    }
    (void)base;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // quarter-warp slot: lanes 0-3 source phase 0 chunks 0..3, lanes 4-7 phase 1
    const uint32_t slot = CONFLICT_FREE ? (uint32_t)(((lane >> 2) & 1) * 64 + (lane & 3) * 16)
                                        : (uint32_t)((lane & 3) * 16);
    const uint32_t off = 0x10000u | slot;
    uint32_t x = threadIdx.x * 747796405u + 2891336453u;
    uint32_t acc[16];
#pragma unroll
    for (int j = 0; j < 16; j++) acc[j] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        x = x * 1664525u + 1013904223u;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t a = prmt(x, off, 0x7604u | (j << 4));
            uint32_t v0, v1, v2, v3;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
            acc[4 * j] ^= v0; acc[4 * j + 1] ^= v1; acc[4 * j + 2] ^= v2; acc[4 * j + 3] ^= v3;
        }
    }
    long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) r ^= acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
}

// mixed: warps 0..11 gather as above, warps 12..15 store 16-byte rows into a
// second 64 KiB region (the product-row kernel's producer / gatherer split);
// reports the combined shared-memory bytes per clock
__global__ void __launch_bounds__(512, 1) mixed_kernel(uint32_t *out, int iters, int st_per_iter, long long *cycles)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    for (uint32_t a = 0x10000u + threadIdx.x * 16u; a < 0x20000u; a += blockDim.x * 16u) {
        const uint32_t v = a * 2654435761u;
        asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" :: "r"(a), "r"(v));
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t r = 0;
    long long t0 = clock64();
    if (warp < 12) {
        const uint32_t slot = (uint32_t)(((lane >> 2) & 1) * 64 + (lane & 3) * 16);
        const uint32_t off = 0x10000u | slot;
        uint32_t x = threadIdx.x * 747796405u + 2891336453u;
        uint32_t acc[16];
#pragma unroll
        for (int j = 0; j < 16; j++) acc[j] = 0;
        for (int it = 0; it < iters; it++) {
            x = x * 1664525u + 1013904223u;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t a = prmt(x, off, 0x7604u | (j << 4));
                uint32_t v0, v1, v2, v3;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
                acc[4 * j] ^= v0; acc[4 * j + 1] ^= v1; acc[4 * j + 2] ^= v2; acc[4 * j + 3] ^= v3;
            }
        }
#pragma unroll
        for (int j = 0; j < 16; j++) r ^= acc[j];
    } else {
        // 128 producer threads: thread t writes 16-byte chunk (t & 15) of rows (t >> 4) + 8 n
        const int pt = threadIdx.x - 384;
        uint32_t v = pt * 0x9E3779B9u;
        const int total = iters * st_per_iter;
        for (int n = 0; n < total; n++) {
            v = v * 1664525u + 1013904223u;
            const uint32_t a = 0x0400u + (uint32_t)((((pt >> 4) + 8 * n) & 255) * 256 + (pt & 15) * 16);
            asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" :: "r"(a), "r"(v));
        }
        r = v;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
}

int main()
{
    uint32_t *d_out; long long *d_cyc;
    cudaMalloc(&d_out, 1 << 24);
    cudaMalloc(&d_cyc, 8);
    base_kernel<<<1, 32, 1024>>>(d_out);
    uint32_t base = 0;
    cudaMemcpy(&base, d_out, 4, cudaMemcpyDeviceToHost);
    printf("dynamic smem shared-window base = 0x%x\n", base);
    const size_t smem = 0x20000u - base;
    cudaFuncSetAttribute(gather_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(gather_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    for (int cf = 1; cf >= 0; cf--) {
        for (int threads = (cf ? 256 : 512); threads <= 512; threads += 128) {   // 8 / 12 / 16 gathering warps
            cudaMemset(d_cyc, 0, 8);
            if (cf) gather_kernel<true><<<sms, threads, smem>>>(d_out, iters, d_cyc);
            else gather_kernel<false><<<sms, threads, smem>>>(d_out, iters, d_cyc);
            cudaError_t e = cudaDeviceSynchronize();
            long long cyc = 0;
            cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
            const double warp_lds = threads / 32.0 * iters * 4;
            printf("LDS.128 prmt-gather %-14s %2d warps  err=%d  warp-LDS/clk/SM = %.3f  gathered B/clk/SM = %.1f\n",
                   cf ? "conflict-free" : "2-row-conflict", threads / 32, (int)e, warp_lds / cyc, warp_lds * 512 / cyc);
        }
    }
    // mixed gathers + row stores at the product-row kernel's ratio (12 gatherer warps x 4 LDS.128 per
    // iteration : 4 producer warps x st_per_iter STS.128 per iteration; 1/6 of the wavefronts are stores
    // at st_per_iter = 2)
    cudaFuncSetAttribute(mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int spi = 1; spi <= 4; spi *= 2) {
        cudaMemset(d_cyc, 0, 8);
        mixed_kernel<<<sms, 512, smem>>>(d_out, iters, spi, d_cyc);
        cudaError_t e = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
        const double ld_bytes = 12.0 * iters * 4 * 512, st_bytes = 4.0 * iters * spi * 512;
        printf("mixed LDS.128 gathers (12 warps) + STS.128 rows (4 warps, %d per iter)  err=%d  "
               "B/clk/SM = %.1f (loads %.1f, stores %.1f)\n", spi, (int)e, (ld_bytes + st_bytes) / cyc,
               ld_bytes / cyc, st_bytes / cyc);
    }
    return 0;
}
