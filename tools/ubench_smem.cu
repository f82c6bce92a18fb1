// ubench_smem.cu -- microbenchmarks that set the LSU / ALU ceilings used in
// shared-memory load throughput for 32/64/128-bit loads when the
// 32 lanes of a warp touch D distinct rows (broadcast inside a row), and
// ALU-pipe throughput of PRMT / LOP3 and FMA-pipe IMAD.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_smem tools/ubench_smem.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kRowStride = 260;   // words; stride/4 odd -> rows r, r+8 share a bank quad

template <int VEC, int D>
__global__ void lds_kernel(uint32_t *out, int iters, long long *cycles)
{
    __shared__ __align__(16) uint32_t sm[32 * kRowStride + 512];
    for (int i = threadIdx.x; i < 32 * kRowStride + 512; i += blockDim.x) sm[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int row = (lane * 7) % D;           // D distinct rows per warp
    const uint32_t base = row * kRowStride + ((threadIdx.x >> 5) & 7) * 16;
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const uint32_t off = (it & 7) * 4;   // stays 16-B aligned
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const uint32_t a = base + off + u * 32;
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&sm[a]);
            if (VEC == 1) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sa));
                acc0 ^= v;
            } else if (VEC == 2) {
                uint32_t x, y;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(sa));
                acc0 ^= x ^ y;
            } else {
                uint32_t x, y, z, w;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(sa));
                acc0 ^= x ^ y; acc1 ^= z ^ w;
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s)
{
    uint32_t d;
    asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}

template <int OP>
__global__ void alu_kernel(uint32_t *out, int iters, long long *cycles)
{
    uint32_t x[8];
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = threadIdx.x * (j + 3) + blockIdx.x;
    const uint32_t t = x[0] | 0x3210u, m = x[1] ^ 0x5555u;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (OP == 0) x[j] = prmt(x[j], t, x[(j + 1) & 7]);
                else if (OP == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[j]) : "r"(t), "r"(m));
                else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[j]) : "r"(t), "r"(m));
            }
        }
    }
    long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) r ^= x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) atomicMax((unsigned long long *)cycles, (unsigned long long)(t1 - t0));
}

template <typename K>
static void run(const char *name, K kern, int blocks, int threads, int iters, double instr_per_thread_iter,
                double bytes_per_instr_lane)
{
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&out, (size_t)blocks * threads * 4);
    cudaMalloc(&cyc, 8);
    cudaMemset(cyc, 0, 8);
    kern<<<blocks, threads>>>(out, 16, cyc);
    cudaMemset(cyc, 0, 8);
    kern<<<blocks, threads>>>(out, iters, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("%s: CUDA error\n", name); exit(1); }
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double warps_per_sm = (double)blocks * threads / 32 / sms;
    const double winstr = warps_per_sm * iters * instr_per_thread_iter;     // warp-instructions per SM
    printf("%-28s warp-instr/clk/SM = %6.3f   lane-bytes/clk/SM = %7.1f   (cycles %lld)\n", name,
           winstr / c, winstr / c * 32 * bytes_per_instr_lane, c);
    cudaFree(out);
    cudaFree(cyc);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256, it = 4096;
    run("LDS.32  D=1", lds_kernel<1, 1>, blocks, threads, it, 8, 4);
    run("LDS.32  D=16", lds_kernel<1, 16>, blocks, threads, it, 8, 4);
    run("LDS.32  D=32", lds_kernel<1, 32>, blocks, threads, it, 8, 4);
    run("LDS.64  D=1", lds_kernel<2, 1>, blocks, threads, it, 8, 8);
    run("LDS.64  D=4", lds_kernel<2, 4>, blocks, threads, it, 8, 8);
    run("LDS.64  D=8", lds_kernel<2, 8>, blocks, threads, it, 8, 8);
    run("LDS.64  D=16", lds_kernel<2, 16>, blocks, threads, it, 8, 8);
    run("LDS.128 D=1", lds_kernel<4, 1>, blocks, threads, it, 8, 16);
    run("LDS.128 D=2", lds_kernel<4, 2>, blocks, threads, it, 8, 16);
    run("LDS.128 D=4", lds_kernel<4, 4>, blocks, threads, it, 8, 16);
    run("LDS.128 D=8", lds_kernel<4, 8>, blocks, threads, it, 8, 16);
    run("LDS.128 D=16", lds_kernel<4, 16>, blocks, threads, it, 8, 16);
    run("PRMT", alu_kernel<0>, blocks, threads, 1024, 64, 4);
    run("LOP3", alu_kernel<1>, blocks, threads, 1024, 64, 4);
    run("IMAD", alu_kernel<2>, blocks, threads, 1024, 64, 4);
    return 0;
}
