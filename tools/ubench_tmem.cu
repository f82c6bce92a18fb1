// ubench_tmem.cu -- tensor-memory (TMEM) load / store throughput on one SM
// from plain warps (no MMA): the planning number for keeping XOR accumulators
// in TMEM (bigger product-row / lane-k tiles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tmem tools/ubench_tmem.cu
// One CTA per SM, W warps; warp w uses TMEM lanes 32 (w % 4) .. + 31 and its own
// column range; each iteration moves 32 lanes x 16 columns x 4 B = 2 KiB per warp
// with tcgen05.ld / tcgen05.st .32x32b.x16.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD16(addr, r)                                                                                   \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
                   "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),      \
                   "=r"(r[14]), "=r"(r[15])                                                             \
                 : "r"(addr))
#define ST16(addr, r)                                                                                   \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 :: "r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),    \
                   "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),             \
                   "r"(r[14]), "r"(r[15]))

template <int MODE>   // 0 = load only, 1 = store only, 2 = load + XOR + store (read-modify-write)
__global__ void tmem_kernel(uint32_t *out, int iters, long long *cycles)
{
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s;
    const int nw = blockDim.x >> 5;
    // lanes 32 (warp % 4) ..; columns: warps sharing a lane quarter split the 512 columns
    const int share = nw / 4, slot = warp / 4;
    const uint32_t cols = 512u / (uint32_t)share;
    const uint32_t addr0 = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)slot * cols;
    uint32_t r[16];
#pragma unroll
    for (int j = 0; j < 16; j++) r[j] = lane * 16 + j;
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const uint32_t a = addr0 + ((uint32_t)(it * 16) % cols);
        if (MODE == 0) {
            LD16(a, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int j = 0; j < 16; j++) acc ^= r[j];
        } else if (MODE == 1) {
            ST16(a, r);
            r[it & 15] += 1u;
        } else {
            LD16(a, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int j = 0; j < 16; j++) r[j] ^= (uint32_t)it;
            ST16(a, r);
        }
    }
    if (MODE != 0) asm volatile("tcgen05.wait::st.sync.aligned;");
    const long long t1 = clock64();
#pragma unroll
    for (int j = 0; j < 16; j++) acc ^= r[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
}

int main()
{
    uint32_t *d_out; long long *d_cyc;
    cudaMalloc(&d_out, 1 << 22);
    cudaMalloc(&d_cyc, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1 << 14;
    const char *names[3] = {"tcgen05.ld x16 (+XOR)", "tcgen05.st x16", "ld + XOR + st (RMW)"};
    for (int mode = 0; mode < 3; mode++) {
        for (int warps = 4; warps <= 16; warps *= 2) {
            cudaMemset(d_cyc, 0, 8);
            if (mode == 0) tmem_kernel<0><<<sms, 32 * warps>>>(d_out, iters, d_cyc);
            else if (mode == 1) tmem_kernel<1><<<sms, 32 * warps>>>(d_out, iters, d_cyc);
            else tmem_kernel<2><<<sms, 32 * warps>>>(d_out, iters, d_cyc);
            const cudaError_t e = cudaDeviceSynchronize();
            long long cyc = 0;
            cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)warps * iters * 32 * 16 * 4 * (mode == 2 ? 2 : 1);
            printf("%-24s %2d warps  err=%s  %.1f B/clk/SM  (%lld cycles)\n", names[mode], warps,
                   cudaGetErrorString(e), bytes / (double)cyc, cyc);
        }
    }
    return 0;
}
