// exp_tmem.cu -- experiment harness for encode_tmem_kernel (TMEM lookup
// tables): times C5- / C3-shaped encodes per field and spot-checks sampled
// output words against a naive host product (tool-local shift-and-add
// multiply; the oracle parity lives in tests/).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp_tmem tools/exp_tmem.cu
//   tools/exp_tmem [wpc]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "../paper_1909_02871_b200/csrc/encode_tmem.cuh"

using namespace gfr;

__global__ void fill_kernel(uint8_t *p, size_t n, uint64_t seed, uint8_t mask)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        p[i] = (uint8_t)z & mask;
    }
}

static uint8_t hmul(int q, uint8_t a, uint8_t b)
{
    const int w = q == 2 ? 1 : q == 4 ? 2 : q == 16 ? 4 : 8;
    const unsigned poly = q == 4 ? 0x7 : q == 16 ? 0x13 : 0x11B;
    unsigned r = 0, x = a;
    for (int j = 0; j < w; j++) {
        if (b >> j & 1) r ^= x;
        x <<= 1;
        if (x >> w & 1) x ^= poly;
    }
    return (uint8_t)r;
}
static uint8_t hmul_packed(int q, uint8_t c, uint8_t a)
{
    const int w = q == 2 ? 1 : q == 4 ? 2 : q == 16 ? 4 : 8;
    uint8_t r = 0;
    for (int s = 0; s < 8; s += w) r |= (uint8_t)(hmul(q, (a >> s) & (q - 1), c) << s);
    return r;
}

template <int LOGW, int WPC, int W = 2>
static void run(int N, int K, size_t M, size_t G, int reps)
{
    const int q = 1 << (1 << LOGW);
    const size_t nA = G * N * M, nC = G * N * K, nB = G * K * M;
    uint8_t *A, *C, *B;
    cudaMalloc(&A, nA); cudaMalloc(&C, nC); cudaMalloc(&B, nB);
    fill_kernel<<<1024, 256>>>(A, nA, 1, 0xFF);
    fill_kernel<<<64, 256>>>(C, nC, 2, (uint8_t)(q - 1));
    cudaMemset(B, 0xEE, nB);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    TmParams p{};
    p.A = A; p.C = C; p.B = B;
    p.Mw = (uint32_t)(M / 4);
    p.spans = (p.Mw + tm_span_words(W) - 1) / tm_span_words(W);
    p.N = N; p.K = K;
    const int w = 1 << LOGW;
    int NG = (N * w + 3) / 4;
    NG = (NG + kTmGPB - 1) / kTmGPB * kTmGPB;
    p.NG = NG;
    p.passes = (K + kTmKB - 1) / kTmKB;
    p.units = (uint64_t)G * p.spans;
    const uint64_t warps = (uint64_t)sms * WPC;
    p.upw = (p.units + warps - 1) / warps;
    const size_t smem = (size_t)WPC * tm_warp_bytes(LOGW, NG, p.passes, 0, W);
    auto kern = encode_tmem_kernel<LOGW, WPC, 0, false, W>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int blocks = (int)((p.units + (uint64_t)WPC * p.upw - 1) / ((uint64_t)WPC * p.upw));
    CUtensorMap map;
    CUtensorMap mapb;
    if (!tm_resolve_encoder() || !tm_make_map(&map, A, (uint64_t)G * N, M, LOGW, W) ||
        !tm_make_map_b(&mapb, B, G, K, M, W)) { printf("tensor map failed\n"); exit(1); }
    kern<<<blocks, WPC * 32, smem>>>(p, map, mapb);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("GF(%d) launch error %s (smem %zu)\n", q, cudaGetErrorString(e), smem); exit(1); }
    // spot check: sampled (g, k, m)
    std::vector<uint8_t> hA(nA), hC(nC), hB(nB);
    cudaMemcpy(hA.data(), A, nA, cudaMemcpyDeviceToHost);
    cudaMemcpy(hC.data(), C, nC, cudaMemcpyDeviceToHost);
    cudaMemcpy(hB.data(), B, nB, cudaMemcpyDeviceToHost);
    size_t bad = 0, checked = 0;
    uint64_t s = 12345;
    for (int n = 0; n < 20000; n++) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        const size_t g = (s >> 33) % G, k = (s >> 13) % K;
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        const size_t m = (n < 64) ? (M - 1 - n % M) : (s >> 20) % M;
        uint8_t r = 0;
        for (int i = 0; i < N; i++) r ^= hmul_packed(q, hC[(g * N + i) * K + k], hA[(g * N + i) * M + m]);
        checked++;
        if (r != hB[(g * K + k) * M + m]) {
            if (bad < 5) printf("  mismatch g=%zu k=%zu m=%zu got %02x want %02x\n", g, k, m, hB[(g * K + k) * M + m], r);
            bad++;
        }
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; r++) kern<<<blocks, WPC * 32, smem>>>(p, map, mapb);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double src = (double)G * N * M;
    printf("GF(%3d) W=%d N=%d K=%d M=%zu G=%zu WPC=%d blocks=%d smem=%zu: %.3f ms  %.1f GB/s source  (%.1f%% of 3273)  "
           "check %zu/%zu bad\n", q, W, N, K, M, G, WPC, blocks, smem, ms, src / ms / 1e6, src / ms / 1e6 / 3273 * 100,
           bad, checked);
    cudaFree(A); cudaFree(B); cudaFree(C);
}

int main(int argc, char **argv)
{
    const int wpc = argc > 1 ? atoi(argv[1]) : 12;
    const int sel = argc > 2 ? atoi(argv[2]) : 63;   // bit f: field set f
#define RUNS(W)                                                                      \
    if (wpc == W) {                                                                  \
        if (sel & 1) run<1, W>(32, 32, 1 << 20, 256, 5);                             \
        if (sel & 2) run<0, W>(32, 32, 1 << 20, 256, 5);                             \
        if (sel & 4) run<2, W>(64, 64, 1504, 16384, 5);                              \
        if (sel & 8) run<2, W>(32, 32, 1 << 20, 64, 5);                              \
        if (sel & 16) run<3, W>(64, 64, 1504, 16384, 5);                             \
        if (sel & 32) run<3, W>(32, 32, 1 << 20, 64, 5);                             \
    }
    if (wpc == 4) {                                  // W = 4 (4 words per lane), 8 warps
        if (sel & 1) run<1, 8, 4>(32, 32, 1 << 20, 256, 5);
        if (sel & 2) run<0, 8, 4>(32, 32, 1 << 20, 256, 5);
        if (sel & 8) run<2, 8, 4>(32, 32, 1 << 20, 64, 5);
        if (sel & 32) run<3, 8, 4>(32, 32, 1 << 20, 64, 5);
        if (sel & 64) run<1, 4, 4>(32, 32, 1 << 20, 256, 5);
    }
    RUNS(8)
    RUNS(12)
    RUNS(16)
    return 0;
}
