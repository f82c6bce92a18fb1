// ubench_tmem2.cu -- tcgen05.ld throughput by load shape (.32x32b.x1 .. x16)
// with NB loads in flight per wait, from W plain warps on one SM: the
// planning number for TMEM lookup tables (encode_tmem.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tmem2 tools/ubench_tmem2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int S>
struct Ld;
template <> struct Ld<1> {
    static __device__ __forceinline__ void go(uint32_t a, uint32_t *r)
    { asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(a)); }
};
template <> struct Ld<2> {
    static __device__ __forceinline__ void go(uint32_t a, uint32_t *r)
    { asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a)); }
};
template <> struct Ld<4> {
    static __device__ __forceinline__ void go(uint32_t a, uint32_t *r)
    { asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a)); }
};
template <> struct Ld<8> {
    static __device__ __forceinline__ void go(uint32_t a, uint32_t *r)
    { asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(a)); }
};
template <> struct Ld<16> {
    static __device__ __forceinline__ void go(uint32_t a, uint32_t *r)
    { asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(a)); }
};

template <int S, int NB>
__global__ void k_ld(uint32_t *out, int iters, long long *cycles, const uint32_t *cols_g)
{
    __shared__ uint32_t taddr_s;
    __shared__ uint32_t cols[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cols[i] = cols_g[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        uint32_t r[NB][S];
#pragma unroll
        for (int j = 0; j < NB; j++) Ld<S>::go(base + cols[(it * NB + j + warp * 5) & 255], r[j]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < NB; j++)
#pragma unroll
            for (int s = 0; s < S; s++) { asm volatile("" : "+r"(r[j][s])); acc ^= r[j][s]; }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr_s));
}

template <int S, int NB>
static void run(uint32_t *d_out, long long *d_cyc, const uint32_t *d_cols, int sms)
{
    const int iters = 4096;
    for (int warps = 4; warps <= 32; warps *= 2) {
        cudaMemset(d_cyc, 0, 8);
        k_ld<S, NB><<<sms, 32 * warps>>>(d_out, iters, d_cyc, d_cols);
        const cudaError_t e = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
        const double instr = (double)warps * iters * NB;
        printf("x%-2d NB=%d %2d warps %s: %6.1f B/clk/SM  %.3f LDTM/clk/SM\n", S, NB, warps, cudaGetErrorString(e),
               instr * 128.0 * S / (double)cyc, instr / (double)cyc);
    }
}

int main()
{
    uint32_t *d_out, *d_cols; long long *d_cyc;
    cudaMalloc(&d_out, 1 << 22);
    cudaMalloc(&d_cyc, 8);
    cudaMalloc(&d_cols, 1024);
    uint32_t h[256];
    for (int i = 0; i < 256; i++) h[i] = (uint32_t)((i * 37) % 31) * 16;   // columns < 512 - 16
    cudaMemcpy(d_cols, h, 1024, cudaMemcpyHostToDevice);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1, 8>(d_out, d_cyc, d_cols, sms);
    run<1, 16>(d_out, d_cyc, d_cols, sms);
    run<2, 8>(d_out, d_cyc, d_cols, sms);
    run<2, 16>(d_out, d_cyc, d_cols, sms);
    run<4, 8>(d_out, d_cyc, d_cols, sms);
    run<8, 4>(d_out, d_cyc, d_cols, sms);
    run<8, 8>(d_out, d_cyc, d_cols, sms);
    run<16, 2>(d_out, d_cyc, d_cols, sms);
    run<16, 4>(d_out, d_cyc, d_cols, sms);
    return 0;
}
