// exp_gf2_uniform.cu -- experiment (rejected): GF(2)
// batched encode (C5 shape) on the ALU pipe with warp-uniform coefficient
// bits from the constant bank (a warp owns one generation): per (i, k) the
// mask sign(bits << (31-k)) is made on the FMA pipe (IMAD.SHL + IMAD.HI) and
// every (i, k, word) costs one LOP3 (acc ^= a & m).  ptxas keeps the masks in
// vector registers (no uniform datapath).  Measured 1201 GB/s of source on
// B200 at G = 256, below the lane-k kernel's 1585.  Checked against a plain
// reference kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/exp_gf2_uniform tools/exp_gf2_uniform.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int N = 32, K = 32;
__constant__ uint32_t c_bits[16384];   // packed coefficient bits [g][i] (bit k), 512 generations

__global__ void pack_bits(const uint8_t *C, uint32_t *bits, int G)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= G * N) return;
    uint32_t b = 0;
    for (int k = 0; k < K; k++) b |= (uint32_t)(C[(size_t)t * K + k] & 1) << k;
    bits[t] = b;
}

template <int W>
__global__ void __launch_bounds__(256) enc2_const(const uint32_t *__restrict__ A, uint32_t *__restrict__ B, uint32_t Mw)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t g = blockIdx.y;
    const uint32_t w0 = (blockIdx.x * 8 + warp) * 32 * W;
    if (w0 >= Mw) return;
    const uint32_t *Ag = A + g * N * (size_t)Mw;
    uint32_t acc[K][W];
#pragma unroll
    for (int k = 0; k < K; k++)
#pragma unroll
        for (int w = 0; w < W; w++) acc[k][w] = 0;
    uint32_t a[W], an[W];
#pragma unroll
    for (int w = 0; w < W; w++) a[w] = __ldg(Ag + w0 + lane + 32 * w);
#pragma unroll 1
    for (int i = 0; i < N; i++) {
        const uint32_t bits = c_bits[blockIdx.y * N + i];
        // masks on the FMA pipe: m = sign(bits << (31 - k)) = mul.hi.s32(bits << (31 - k), 1)
        if (i + 1 < N) {
#pragma unroll
            for (int w = 0; w < W; w++) an[w] = __ldg(Ag + (size_t)(i + 1) * Mw + w0 + lane + 32 * w);
        }
#pragma unroll
        for (int k = 0; k < K; k++) {
            uint32_t sh, m;
            asm("mul.lo.u32 %0, %1, %2;" : "=r"(sh) : "r"(bits), "r"(1u << (31 - k)));
            asm("mul.hi.s32 %0, %1, 1;" : "=r"(m) : "r"(sh));
#pragma unroll
            for (int w = 0; w < W; w++) acc[k][w] ^= a[w] & m;
        }
#pragma unroll
        for (int w = 0; w < W; w++) a[w] = an[w];
    }
#pragma unroll
    for (int k = 0; k < K; k++)
#pragma unroll
        for (int w = 0; w < W; w++) B[(g * K + k) * (size_t)Mw + w0 + lane + 32 * w] = acc[k][w];
}

__global__ void enc2_ref(const uint32_t *A, const uint8_t *C, uint32_t *B, uint32_t Mw, int G)
{
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)G * K * Mw) return;
    const uint32_t w = idx % Mw;
    const int k = (idx / Mw) % K;
    const size_t g = idx / ((size_t)Mw * K);
    uint32_t acc = 0;
    for (int i = 0; i < N; i++)
        if (C[(g * N + i) * K + k] & 1) acc ^= A[(g * N + i) * (size_t)Mw + w];
    B[idx] = acc;
}

int main(int argc, char **argv)
{
    const int G = argc > 1 ? atoi(argv[1]) : 64;
    const uint32_t Mw = (1u << 20) / 4;
    const size_t nA = (size_t)G * N * Mw, nB = (size_t)G * K * Mw;
    uint32_t *A, *B, *R;
    uint8_t *C;
    cudaMalloc(&A, nA * 4); cudaMalloc(&B, nB * 4); cudaMalloc(&R, nB * 4); cudaMalloc(&C, (size_t)G * N * K);
    uint32_t *h = (uint32_t *)malloc(nA * 4);
    uint64_t x = 88172645463325252ull;
    for (size_t j = 0; j < nA; j++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[j] = (uint32_t)x; }
    cudaMemcpy(A, h, nA * 4, cudaMemcpyHostToDevice);
    uint8_t *hc = (uint8_t *)malloc((size_t)G * N * K);
    for (size_t j = 0; j < (size_t)G * N * K; j++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hc[j] = x & 1; }
    cudaMemcpy(C, hc, (size_t)G * N * K, cudaMemcpyHostToDevice);
    enc2_ref<<<(unsigned)((nB + 255) / 256), 256>>>(A, C, R, Mw, G);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    constexpr int W = 2;
    dim3 grid((Mw + 8 * 32 * W - 1) / (8 * 32 * W), G);
    const int reps = 10;
    float ms;
    uint32_t *hb = (uint32_t *)malloc(nB * 4), *hr = (uint32_t *)malloc(nB * 4);
    cudaMemcpy(hr, R, nB * 4, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    // constant-bank masks (uniform datapath), at most 512 generations
    uint32_t *bits;
    cudaMalloc(&bits, (size_t)G * N * 4);
    pack_bits<<<(G * N + 255) / 256, 256>>>(C, bits, G);
    cudaMemcpyToSymbol(c_bits, bits, (size_t)G * N * 4, 0, cudaMemcpyDeviceToDevice);
    cudaMemset(B, 0, nB * 4);
    for (int it = 0; it < 3; it++) enc2_const<W><<<grid, 256>>>(A, B, Mw);
    cudaEventRecord(e0);
    for (int it = 0; it < reps; it++) enc2_const<W><<<grid, 256>>>(A, B, Mw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    cudaMemcpy(hb, B, nB * 4, cudaMemcpyDeviceToHost);
    bad = 0;
    for (size_t j = 0; j < nB; j++) bad += hb[j] != hr[j];
    printf("GF(2) const-mask column W=%d: G=%d %.3f ms  %.1f GB/s source  mismatches=%zu  err=%s\n", W, G, ms,
           (double)nA * 4 / ms / 1e6, bad, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
