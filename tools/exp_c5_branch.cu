// exp_c5_branch.cu -- experiment: C5-shape encode (N = K = 32, 1 MiB packets)
// for GF(2) / GF(4) with WARP-UNIFORM BRANCHES on the coefficients instead of
// masks or shared-memory tables (the GPU form of the paper's trivial-
// coefficient shortcut).
// A warp owns one generation, so every coefficient is warp-uniform.  Each lane
// holds its W words of all 32 sources in registers; for every coded packet k
// and every group of 4 GF(2)-terms the 4-bit coefficient pattern selects (one
// uniform indirect branch) the XOR of exactly the terms that are present, so
// each (k, group, word) costs ceil(t/2) 3-input LOP3s and zero terms cost
// nothing.  GF(4): terms are a_i and x*a_i (two sources per group).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/exp_c5_branch tools/exp_c5_branch.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "exp_c5_groups.h"
#include "exp_c5_groups2.h"

constexpr int N = 32, K = 32;

struct V4 { uint32_t x, y, z, w; };

__device__ __forceinline__ V4 ld4(const uint32_t *p)
{
    V4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st4(uint32_t *p, V4 v)
{
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ __forceinline__ V4 x4(V4 a, V4 b) { return {a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w}; }
__device__ __forceinline__ V4 x4(V4 a, V4 b, V4 c) { return {a.x ^ b.x ^ c.x, a.y ^ b.y ^ c.y, a.z ^ b.z ^ c.z, a.w ^ b.w ^ c.w}; }

// acc ^= XOR of the terms t0..t3 selected by the 4 bits of p
#define GROUP(p, acc, t0, t1, t2, t3)                                              \
    switch ((p) & 15u) {                                                           \
    case 0: break;                                                                 \
    case 1: acc = x4(acc, t0); break;                                              \
    case 2: acc = x4(acc, t1); break;                                              \
    case 3: acc = x4(acc, t0, t1); break;                                          \
    case 4: acc = x4(acc, t2); break;                                              \
    case 5: acc = x4(acc, t0, t2); break;                                          \
    case 6: acc = x4(acc, t1, t2); break;                                          \
    case 7: acc = x4(x4(acc, t0, t1), t2); break;                                  \
    case 8: acc = x4(acc, t3); break;                                              \
    case 9: acc = x4(acc, t0, t3); break;                                          \
    case 10: acc = x4(acc, t1, t3); break;                                         \
    case 11: acc = x4(x4(acc, t0, t1), t3); break;                                 \
    case 12: acc = x4(acc, t2, t3); break;                                         \
    case 13: acc = x4(x4(acc, t0, t2), t3); break;                                 \
    case 14: acc = x4(x4(acc, t1, t2), t3); break;                                 \
    default: acc = x4(x4(acc, t0, t1), x4(t2, t3)); break;                         \
    }

// GF(2): lane l of the warp owns uint4 column chunk (span*32 + l) of every packet
__global__ void __launch_bounds__(128) enc2_branch(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                   uint32_t *__restrict__ B, uint32_t Mv, int G, int spans_per_warp)
{
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t spans = Mv / 32;                       // uint4 chunks per packet / 32
    const size_t items = (size_t)G * spans;
    size_t it = warp * spans_per_warp;
    if (it >= items) return;
    size_t g_cur = ~size_t(0);
    uint32_t mk_lane = 0;
    for (int s = 0; s < spans_per_warp && it < items; s++, it++) {
        const size_t g = it / spans;
        const uint32_t sp = (uint32_t)(it % spans);
        if (g != g_cur) {
            g_cur = g;
            uint32_t m = 0;
            const uint8_t *Cg = C + g * N * K;
#pragma unroll 8
            for (int i = 0; i < N; i++) m |= (uint32_t)(Cg[i * K + lane] & 1) << i;
            mk_lane = m;                                  // bit i = C[g][i][lane]
        }
        const uint32_t *Ag = A + (g * N * (size_t)Mv + (size_t)sp * 32 + lane) * 4;
        V4 a[N];
#pragma unroll
        for (int i = 0; i < N; i++) a[i] = ld4(Ag + (size_t)i * Mv * 4);
        uint32_t *Bg = B + (g * K * (size_t)Mv + (size_t)sp * 32 + lane) * 4;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            const uint32_t mk = __shfl_sync(0xffffffffu, mk_lane, k);
            V4 acc = {0, 0, 0, 0};
            const uint32_t i0 = mk & 15u;
            BRX_GROUP4(i0, acc, a[0], a[1], a[2], a[3]);
#pragma unroll
            for (int j = 1; j < 8; j++) {
                const uint32_t ij = (mk >> (4 * j)) & 15u;
                BRX_GROUP4(ij, acc, a[4 * j], a[4 * j + 1], a[4 * j + 2], a[4 * j + 3]);
            }
            st4(Bg + (size_t)k * Mv * 4, acc);
        }
    }
}

__device__ __forceinline__ uint32_t xt4(uint32_t a)   // x * a, 16 GF(4) elements
{
    return ((a >> 1) & 0x55555555u) | (((a ^ (a >> 1)) & 0x55555555u) << 1);
}

struct V2 { uint32_t x, y; };
__device__ __forceinline__ V2 x2(V2 a, V2 b) { return {a.x ^ b.x, a.y ^ b.y}; }
__device__ __forceinline__ V2 x2(V2 a, V2 b, V2 c) { return {a.x ^ b.x ^ c.x, a.y ^ b.y ^ c.y}; }
#define GROUP2(p, acc, t0, t1, t2, t3)                                             \
    switch ((p) & 15u) {                                                           \
    case 0: break;                                                                 \
    case 1: acc = x2(acc, t0); break;                                              \
    case 2: acc = x2(acc, t1); break;                                              \
    case 3: acc = x2(acc, t0, t1); break;                                          \
    case 4: acc = x2(acc, t2); break;                                              \
    case 5: acc = x2(acc, t0, t2); break;                                          \
    case 6: acc = x2(acc, t1, t2); break;                                          \
    case 7: acc = x2(x2(acc, t0, t1), t2); break;                                  \
    case 8: acc = x2(acc, t3); break;                                              \
    case 9: acc = x2(acc, t0, t3); break;                                          \
    case 10: acc = x2(acc, t1, t3); break;                                         \
    case 11: acc = x2(x2(acc, t0, t1), t3); break;                                 \
    case 12: acc = x2(acc, t2, t3); break;                                         \
    case 13: acc = x2(x2(acc, t0, t2), t3); break;                                 \
    case 14: acc = x2(x2(acc, t1, t2), t3); break;                                 \
    default: acc = x2(x2(acc, t0, t1), x2(t2, t3)); break;                         \
    }

// GF(4): lane l owns uint2 chunk (span*32 + l); terms a_i, x*a_i; pattern bits
// of source i at 2i (c0) and 2i+1 (c1): c*a = c0*a + c1*(x a)
__global__ void __launch_bounds__(128) enc4_branch(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                   uint32_t *__restrict__ B, uint32_t Mv2, int G, int spans_per_warp)
{
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t spans = Mv2 / 32;
    const size_t items = (size_t)G * spans;
    size_t it = warp * spans_per_warp;
    if (it >= items) return;
    size_t g_cur = ~size_t(0);
    uint32_t mlo = 0, mhi = 0;
    for (int s = 0; s < spans_per_warp && it < items; s++, it++) {
        const size_t g = it / spans;
        const uint32_t sp = (uint32_t)(it % spans);
        if (g != g_cur) {
            g_cur = g;
            uint32_t lo = 0, hi = 0;
            const uint8_t *Cg = C + g * N * K;
#pragma unroll 8
            for (int i = 0; i < 16; i++) lo |= (uint32_t)(Cg[i * K + lane] & 3) << (2 * i);
#pragma unroll 8
            for (int i = 0; i < 16; i++) hi |= (uint32_t)(Cg[(i + 16) * K + lane] & 3) << (2 * i);
            mlo = lo; mhi = hi;
        }
        const uint32_t *Ag = A + (g * N * (size_t)Mv2 + (size_t)sp * 32 + lane) * 2;
        V2 a[N], xa[N];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const uint2 v = __ldcs(reinterpret_cast<const uint2 *>(Ag + (size_t)i * Mv2 * 2));
            a[i] = {v.x, v.y};
        }
#pragma unroll
        for (int i = 0; i < N; i++) xa[i] = {xt4(a[i].x), xt4(a[i].y)};
        uint32_t *Bg = B + (g * K * (size_t)Mv2 + (size_t)sp * 32 + lane) * 2;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            const uint32_t ml = __shfl_sync(0xffffffffu, mlo, k);
            const uint32_t mh = __shfl_sync(0xffffffffu, mhi, k);
            V2 acc = {0, 0};
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t ij = (ml >> (4 * j)) & 15u;
                BRX_GROUP2(ij, acc, a[2 * j], xa[2 * j], a[2 * j + 1], xa[2 * j + 1]);
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const uint32_t ij = (mh >> (4 * j)) & 15u;
                BRX_GROUP2(ij, acc, a[16 + 2 * j], xa[16 + 2 * j], a[17 + 2 * j], xa[17 + 2 * j]);
            }
            __stcs(reinterpret_cast<uint2 *>(Bg + (size_t)k * Mv2 * 2), make_uint2(acc.x, acc.y));
        }
    }
}


// ---- threaded dispatch: every case ends with the next group's brx.idx -------------
__global__ void __launch_bounds__(128) enc2_thr(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                uint32_t *__restrict__ B, uint32_t Mv, int G, int spans_per_warp)
{
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t spans = Mv / 32;
    const size_t items = (size_t)G * spans;
    size_t it = warp * spans_per_warp;
    if (it >= items) return;
    size_t g_cur = ~size_t(0);
    uint32_t mk_lane = 0;
    for (int s = 0; s < spans_per_warp && it < items; s++, it++) {
        const size_t g = it / spans;
        const uint32_t sp = (uint32_t)(it % spans);
        if (g != g_cur) {
            g_cur = g;
            uint32_t m = 0;
            const uint8_t *Cg = C + g * N * K;
#pragma unroll 8
            for (int i = 0; i < N; i++) m |= (uint32_t)(Cg[i * K + lane] & 1) << i;
            mk_lane = m;
        }
        const uint32_t *Ag = A + (g * N * (size_t)Mv + (size_t)sp * 32 + lane) * 4;
        V4 a[N];
#pragma unroll
        for (int i = 0; i < N; i++) a[i] = ld4(Ag + (size_t)i * Mv * 4);
        uint32_t *Bg = B + (g * K * (size_t)Mv + (size_t)sp * 32 + lane) * 4;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            const uint32_t mk = __shfl_sync(0xffffffffu, mk_lane, k);
            uint32_t id[8];
#pragma unroll
            for (int j = 0; j < 8; j++) id[j] = (mk >> (4 * j)) & 15u;
            V4 acc = {0, 0, 0, 0};
#define TERM2(g, j) a[4 * (g) + (j)]
#define IDX2(g) id[g]
            KITER2_W4(acc, TERM2, IDX2);
            st4(Bg + (size_t)k * Mv * 4, acc);
        }
    }
}

__global__ void __launch_bounds__(128) enc4_thr(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                uint32_t *__restrict__ B, uint32_t Mv2, int G, int spans_per_warp)
{
    const int lane = threadIdx.x & 31;
    const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t spans = Mv2 / 32;
    const size_t items = (size_t)G * spans;
    size_t it = warp * spans_per_warp;
    if (it >= items) return;
    size_t g_cur = ~size_t(0);
    uint32_t mlo = 0, mhi = 0;
    for (int s = 0; s < spans_per_warp && it < items; s++, it++) {
        const size_t g = it / spans;
        const uint32_t sp = (uint32_t)(it % spans);
        if (g != g_cur) {
            g_cur = g;
            uint32_t lo = 0, hi = 0;
            const uint8_t *Cg = C + g * N * K;
#pragma unroll 8
            for (int i = 0; i < 16; i++) lo |= (uint32_t)(Cg[i * K + lane] & 3) << (2 * i);
#pragma unroll 8
            for (int i = 0; i < 16; i++) hi |= (uint32_t)(Cg[(i + 16) * K + lane] & 3) << (2 * i);
            mlo = lo; mhi = hi;
        }
        const uint32_t *Ag = A + (g * N * (size_t)Mv2 + (size_t)sp * 32 + lane) * 2;
        V2 a[N], xa[N];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const uint2 v = __ldcs(reinterpret_cast<const uint2 *>(Ag + (size_t)i * Mv2 * 2));
            a[i] = {v.x, v.y};
        }
#pragma unroll
        for (int i = 0; i < N; i++) xa[i] = {xt4(a[i].x), xt4(a[i].y)};
        uint32_t *Bg = B + (g * K * (size_t)Mv2 + (size_t)sp * 32 + lane) * 2;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            const uint32_t ml = __shfl_sync(0xffffffffu, mlo, k);
            const uint32_t mh = __shfl_sync(0xffffffffu, mhi, k);
            uint32_t id[16];
#pragma unroll
            for (int j = 0; j < 8; j++) { id[j] = (ml >> (4 * j)) & 15u; id[8 + j] = (mh >> (4 * j)) & 15u; }
            V2 acc = {0, 0};
#define TERM4(g, j) ((j) == 0 ? a[2 * (g)] : (j) == 1 ? xa[2 * (g)] : (j) == 2 ? a[2 * (g) + 1] : xa[2 * (g) + 1])
#define IDX4(g) id[g]
            KITER4_W2(acc, TERM4, IDX4);
            __stcs(reinterpret_cast<uint2 *>(Bg + (size_t)k * Mv2 * 2), make_uint2(acc.x, acc.y));
        }
    }
}

// ---- branch-free: IMAD-masked pairs merged by one 3-input LOP3 (FMA pipe) plus
// LOP3-masked terms (ALU pipe), ~2:1, so both pipes carry ~2/3 op per term --------
template <int W>
__global__ void __launch_bounds__(128) enc2_mix(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                uint32_t *__restrict__ B, uint32_t Mw, int spans_per_warp)
{
    __shared__ __align__(16) uint32_t cw[K * N];          // [k][i]: c (0/1) or mask (0/~0) for i % 3 == 2
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = blockIdx.y;
    for (int t = threadIdx.x; t < K * N; t += blockDim.x) {
        const int k = t / N, i = t % N;
        const uint32_t c = C[(g * N + i) * K + k] & 1u;
        cw[t] = (i % 3 == 2) ? 0u - c : c;
    }
    __syncthreads();
    const uint32_t spanw = 32 * W;
    const uint32_t sp0 = (blockIdx.x * 4 + wid) * spans_per_warp;
    for (int s = 0; s < spans_per_warp; s++) {
        const uint32_t w0 = (sp0 + s) * spanw;
        if (w0 >= Mw) break;
        const uint32_t *Ag = A + g * N * (size_t)Mw + w0 + lane * W;
        uint32_t a[N][W];
#pragma unroll
        for (int i = 0; i < N; i++) {
            if constexpr (W == 4) {
                const V4 v = ld4(Ag + (size_t)i * Mw);
                a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
            } else {
                const uint2 v = __ldcs(reinterpret_cast<const uint2 *>(Ag + (size_t)i * Mw));
                a[i][0] = v.x; a[i][1] = v.y;
            }
        }
        uint32_t *Bg = B + g * K * (size_t)Mw + w0 + lane * W;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            uint32_t c[N];
#pragma unroll
            for (int q = 0; q < N / 4; q++) {
                const uint4 v = reinterpret_cast<const uint4 *>(cw + k * N)[q];
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
            uint32_t acc[W];
#pragma unroll
            for (int w = 0; w < W; w++) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < N; i += 3) {
                    if (i + 1 < N) x ^= (a[i][w] * c[i]) ^ (a[i + 1][w] * c[i + 1]);
                    else x ^= a[i][w] * c[i];
                    if (i + 2 < N) x ^= a[i + 2][w] & c[i + 2];
                }
                acc[w] = x;
            }
            if constexpr (W == 4) st4(Bg + (size_t)k * Mw, {acc[0], acc[1], acc[2], acc[3]});
            else __stcs(reinterpret_cast<uint2 *>(Bg + (size_t)k * Mw), make_uint2(acc[0], acc[1]));
        }
    }
}


// GF(4) split: sources i % 3 == 0 masked (acc ^= a & m0, acc ^= xa & m1: 2 ALU),
// the others the paper's imul (Alg. 2): lo*c ^ hi*(x c) (2 IMAD) merged in pairs
template <int MSK>
__global__ void __launch_bounds__(128) enc4_mix(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                uint32_t *__restrict__ B, uint32_t Mw, int spans_per_warp)
{
    constexpr int W = 2;
    __shared__ __align__(16) uint32_t cw[K * N * 2];      // [k][i][2]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = blockIdx.y;
    for (int t = threadIdx.x; t < K * N; t += blockDim.x) {
        const int k = t / N, i = t % N;
        const uint32_t c = C[(g * N + i) * K + k] & 3u;
        const uint32_t xc = ((c << 1) ^ ((c >> 1) * 3u)) & 3u;          // x * c in GF(4)
        if (i % 3 == MSK) { cw[2 * t] = 0u - (c & 1u); cw[2 * t + 1] = 0u - (c >> 1); }
        else { cw[2 * t] = c; cw[2 * t + 1] = xc; }
    }
    __syncthreads();
    const uint32_t spanw = 32 * W;
    const uint32_t sp0 = (blockIdx.x * 4 + wid) * spans_per_warp;
    for (int s = 0; s < spans_per_warp; s++) {
        const uint32_t w0 = (sp0 + s) * spanw;
        if (w0 >= Mw) break;
        const uint32_t *Ag = A + g * N * (size_t)Mw + w0 + lane * W;
        uint32_t u[N][W], v[N][W];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const uint2 x = __ldcs(reinterpret_cast<const uint2 *>(Ag + (size_t)i * Mw));
            const uint32_t xa[2] = {x.x, x.y};
#pragma unroll
            for (int w = 0; w < W; w++) {
                if (i % 3 == MSK) { u[i][w] = xa[w]; v[i][w] = xt4(xa[w]); }
                else { u[i][w] = xa[w] & 0x55555555u; v[i][w] = (xa[w] >> 1) & 0x55555555u; }
            }
        }
        uint32_t *Bg = B + g * K * (size_t)Mw + w0 + lane * W;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            const uint4 *cq = reinterpret_cast<const uint4 *>(cw + k * N * 2);
            uint32_t acc[W] = {0, 0};
#pragma unroll
            for (int q = 0; q < N / 2; q++) {
                const uint4 cc = cq[q];                           // sources 2q, 2q+1: (c0, c1) each
                const int i0 = 2 * q, i1 = 2 * q + 1;
#pragma unroll
                for (int w = 0; w < W; w++) {
                    uint32_t t0 = (i0 % 3 == MSK) ? (u[i0][w] & cc.x) ^ (v[i0][w] & cc.y)
                                                  : (u[i0][w] * cc.x) ^ (v[i0][w] * cc.y);
                    uint32_t t1 = (i1 % 3 == MSK) ? (u[i1][w] & cc.z) ^ (v[i1][w] & cc.w)
                                                  : (u[i1][w] * cc.z) ^ (v[i1][w] * cc.w);
                    acc[w] ^= t0 ^ t1;
                }
            }
            __stcs(reinterpret_cast<uint2 *>(Bg + (size_t)k * Mw), make_uint2(acc[0], acc[1]));
        }
    }
}

// GF(2) split with a selectable masked fraction: sources with (i % P) == P-1 masked
template <int W, int P>
__global__ void __launch_bounds__(128) enc2_mixp(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                 uint32_t *__restrict__ B, uint32_t Mw, int spans_per_warp)
{
    __shared__ __align__(16) uint32_t cw[K * N];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = blockIdx.y;
    for (int t = threadIdx.x; t < K * N; t += blockDim.x) {
        const int k = t / N, i = t % N;
        const uint32_t c = C[(g * N + i) * K + k] & 1u;
        cw[t] = (i % P == P - 1) ? 0u - c : c;
    }
    __syncthreads();
    const uint32_t spanw = 32 * W;
    const uint32_t sp0 = (blockIdx.x * 4 + wid) * spans_per_warp;
    for (int s = 0; s < spans_per_warp; s++) {
        const uint32_t w0 = (sp0 + s) * spanw;
        if (w0 >= Mw) break;
        const uint32_t *Ag = A + g * N * (size_t)Mw + w0 + lane * W;
        uint32_t a[N][W];
#pragma unroll
        for (int i = 0; i < N; i++) {
            const V4 v = ld4(Ag + (size_t)i * Mw);
            a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
        uint32_t *Bp = B + g * K * (size_t)Mw + w0 + lane * W;
#pragma unroll 1
        for (int k = 0; k < K; k++, Bp += Mw) {
            uint32_t c[N];
#pragma unroll
            for (int q = 0; q < N / 4; q++) {
                const uint4 v = reinterpret_cast<const uint4 *>(cw + k * N)[q];
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
            uint32_t acc[W];
#pragma unroll
            for (int w = 0; w < W; w++) {
                uint32_t x = 0, y = 0;
                int pend = -1;
#pragma unroll
                for (int i = 0; i < N; i++) {
                    if (i % P == P - 1) x ^= a[i][w] & c[i];
                    else if (pend < 0) pend = i;
                    else { y ^= (a[pend][w] * c[pend]) ^ (a[i][w] * c[i]); pend = -1; }
                }
                if (pend >= 0) y ^= a[pend][w] * c[pend];
                acc[w] = x ^ y;
            }
            st4(Bp, {acc[0], acc[1], acc[2], acc[3]});
        }
    }
}


// library-form kernel (runtime N, K or compile-time KC) for A/B against enc2_mix<4>
template <int KC>
__global__ void __launch_bounds__(128) enc2_libform(const uint8_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                    uint8_t *__restrict__ B, uint32_t Mw, int Nr, int Kr,
                                                    uint32_t spans, uint32_t blocks_per_gen, int spw)
{
    constexpr int NS = 32;
    extern __shared__ __align__(16) uint32_t cwd[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = blockIdx.x / blocks_per_gen;
    const uint32_t bi = blockIdx.x - (uint32_t)(g * blocks_per_gen);
    const int Nn = Nr, K = KC ? KC : Kr;
    for (int t = threadIdx.x; t < K * NS; t += 128) {
        const int k = t / NS, i = t - k * NS;
        const uint32_t c = i < Nn ? (__ldg(C + g * (size_t)Nn * K + (size_t)i * K + k) & 1u) : 0u;
        cwd[t] = (i % 3 == 2) ? 0u - c : c;
    }
    __syncthreads();
    const size_t M = (size_t)Mw * 4;
    const uint32_t sp0 = (bi * 4 + wid) * (uint32_t)spw;
#pragma unroll 1
    for (int s = 0; s < spw; s++) {
        const uint32_t sp = sp0 + s;
        if (sp >= spans) break;
        const uint32_t w0 = sp * 128 + 4 * lane;
        const bool valid = w0 < Mw;
        const uint8_t *Ag = A + g * (size_t)Nn * M + 4 * (size_t)(valid ? w0 : 0u);
        uint32_t a[NS][4];
#pragma unroll
        for (int i = 0; i < NS; i++) {
            const V4 v = ld4(reinterpret_cast<const uint32_t *>(Ag + (size_t)(i < Nn ? i : 0) * M));
            a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
        uint8_t *Bp = B + g * (size_t)K * M + 4 * (size_t)w0;
#pragma unroll 1
        for (int k = 0; k < K; k++, Bp += M) {
            uint32_t c[NS];
#pragma unroll
            for (int q = 0; q < NS / 4; q++) {
                const uint4 v = reinterpret_cast<const uint4 *>(cwd + k * NS)[q];
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
            uint32_t acc[4];
#pragma unroll
            for (int w = 0; w < 4; w++) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < NS; i += 3) {
                    if (i + 1 < NS) x ^= (a[i][w] * c[i]) ^ (a[i + 1][w] * c[i + 1]);
                    else x ^= a[i][w] * c[i];
                    if (i + 2 < NS) x ^= a[i + 2][w] & c[i + 2];
                }
                acc[w] = x;
            }
            if (KC) { st4(reinterpret_cast<uint32_t *>(Bp), {acc[0], acc[1], acc[2], acc[3]}); }
            else {
                asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.global.v4.u32 [%0], {%1,%2,%3,%4};\n\t}"
                             :: "l"(Bp), "r"(acc[0]), "r"(acc[1]), "r"(acc[2]), "r"(acc[3]), "r"(valid ? 1u : 0u) : "memory");
            }
        }
    }
}


// W words per lane in the strided layout (lane l: words l, l + 32, ...): W = 3
// keeps ~124 registers (16 warps / SM instead of 12)
template <int W>
__global__ void __launch_bounds__(128) enc2_mixs(const uint32_t *__restrict__ A, const uint8_t *__restrict__ C,
                                                 uint32_t *__restrict__ B, uint32_t Mw, int spans_per_warp)
{
    __shared__ __align__(16) uint32_t cw[K * N];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = blockIdx.y;
    for (int t = threadIdx.x; t < K * N; t += blockDim.x) {
        const int k = t / N, i = t % N;
        const uint32_t c = C[(g * N + i) * K + k] & 1u;
        cw[t] = (i % 3 == 2) ? 0u - c : c;
    }
    __syncthreads();
    const uint32_t spanw = 32 * W;
    const uint32_t sp0 = (blockIdx.x * 4 + wid) * spans_per_warp;
    for (int s = 0; s < spans_per_warp; s++) {
        const uint32_t w0 = (sp0 + s) * spanw;
        if (w0 >= Mw) break;
        const uint32_t *Ag = A + g * N * (size_t)Mw + w0 + lane;
        uint32_t a[N][W];
#pragma unroll
        for (int i = 0; i < N; i++)
#pragma unroll
            for (int w = 0; w < W; w++) a[i][w] = (w0 + lane + 32 * w < Mw) ? __ldcs(Ag + (size_t)i * Mw + 32 * w) : 0u;
        uint32_t *Bg = B + g * K * (size_t)Mw + w0 + lane;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            uint32_t c[N];
#pragma unroll
            for (int q = 0; q < N / 4; q++) {
                const uint4 v = reinterpret_cast<const uint4 *>(cw + k * N)[q];
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
#pragma unroll
            for (int w = 0; w < W; w++) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < N; i += 3) {
                    if (i + 1 < N) x ^= (a[i][w] * c[i]) ^ (a[i + 1][w] * c[i + 1]);
                    else x ^= a[i][w] * c[i];
                    if (i + 2 < N) x ^= a[i + 2][w] & c[i + 2];
                }
                if (w0 + lane + 32 * w < Mw) __stcs(Bg + (size_t)k * Mw + 32 * w, x);
            }
        }
    }
}

// plain reference (bytewise, any field): B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]
__device__ uint8_t mulb(int q, uint8_t c, uint8_t v)
{
    const int w = q == 2 ? 1 : 2;
    const unsigned P = 7, msk = (1u << w) - 1;
    uint8_t out = 0;
    for (int s = 0; s < 8; s += w) {
        unsigned a = (v >> s) & msk, r = 0;
        for (int b = 0; b < w; b++)
            if (c >> b & 1) r ^= a << b;
        if (w == 2 && (r & 4)) r ^= P;
        out |= (uint8_t)((r & msk) << s);
    }
    return out;
}
__global__ void enc_ref(int q, const uint8_t *A, const uint8_t *C, uint8_t *B, size_t M, int G)
{
    const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (idx >= (size_t)G * K * M) return;
    const size_t m = idx % M;
    const int k = (idx / M) % K;
    const size_t g = idx / (M * K);
    uint8_t acc = 0;
    for (int i = 0; i < N; i++) acc ^= mulb(q, C[(g * N + i) * K + k] & (q - 1), A[(g * N + i) * M + m]);
    B[idx] = acc;
}

__global__ void fill(uint8_t *p, size_t n, uint64_t seed, uint8_t mask)
{
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n / 8; j += (size_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (j + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        reinterpret_cast<uint64_t *>(p)[j] = z & (0x0101010101010101ull * mask);
    }
}

int main(int argc, char **argv)
{
    const int q = argc > 1 ? atoi(argv[1]) : 2;
    const int G = argc > 2 ? atoi(argv[2]) : 256;
    const int spw = argc > 3 ? atoi(argv[3]) : 16;
    const size_t M = 1u << 20;
    const size_t nA = (size_t)G * N * M, nB = (size_t)G * K * M, nC = (size_t)G * N * K;
    uint8_t *A, *B, *R, *C;
    cudaMalloc(&A, nA); cudaMalloc(&B, nB); cudaMalloc(&R, nB); cudaMalloc(&C, nC);
    fill<<<1184, 256>>>(A, nA, 12345, 0xFF);
    fill<<<1184, 256>>>(C, nC, 777, (uint8_t)(q - 1));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    // check on the first 4 generations against the reference kernel
    const int Gc = 4;
    enc_ref<<<(unsigned)(((size_t)Gc * K * M + 255) / 256), 256>>>(q, A, C, R, M, Gc);
    const int var = argc > 4 ? atoi(argv[4]) : 0;   // 0 branch, 1 threaded, 2 mix W=4, 3 mix W=2
    auto launch = [&](int Gl) {
        if (var == 11 || var == 12) {
            const uint32_t Mw = M / 4;
            const int W = var == 11 ? 3 : 4;
            const uint32_t spans = (Mw + 32 * W - 1) / (32 * W);
            dim3 grid((spans + 4 * spw - 1) / (4 * spw), Gl);
            if (W == 3) enc2_mixs<3><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else enc2_mixs<4><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
        } else if (var == 9 || var == 10) {
            const uint32_t Mw = M / 4, spans = Mw / 128;
            const uint32_t bpg = (spans + 63) / 64;
            if (var == 9) enc2_libform<0><<<Gl * bpg, 128, 4096>>>(A, C, B, Mw, 32, 32, spans, bpg, 16);
            else enc2_libform<32><<<Gl * bpg, 128, 4096>>>(A, C, B, Mw, 32, 32, spans, bpg, 16);
        } else if (var >= 4) {
            const uint32_t Mw = M / 4;
            const int W = var == 4 || var == 5 ? 2 : 4;
            const uint32_t spans = Mw / (32 * W);
            dim3 grid((spans + 4 * spw - 1) / (4 * spw), Gl);
            if (var == 4) enc4_mix<0><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else if (var == 5) enc4_mix<99><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else if (var == 6) enc2_mixp<4, 3><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else if (var == 7) enc2_mixp<4, 4><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else if (var == 13) enc2_mixp<4, 1><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else enc2_mixp<4, 2><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
        } else if (var >= 2) {
            const uint32_t Mw = M / 4;
            const int W = var == 2 ? 4 : 2;
            const uint32_t spans = Mw / (32 * W);
            dim3 grid((spans + 4 * spw - 1) / (4 * spw), Gl);
            if (W == 4) enc2_mix<4><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
            else enc2_mix<2><<<grid, 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mw, spw);
        } else if (q == 2) {
            const uint32_t Mv = M / 16;
            const size_t items = (size_t)Gl * (Mv / 32);
            const size_t warps = (items + spw - 1) / spw;
            if (var == 1) enc2_thr<<<(unsigned)((warps + 3) / 4), 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mv, Gl, spw);
            else enc2_branch<<<(unsigned)((warps + 3) / 4), 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mv, Gl, spw);
        } else {
            const uint32_t Mv2 = M / 8;
            const size_t items = (size_t)Gl * (Mv2 / 32);
            const size_t warps = (items + spw - 1) / spw;
            if (var == 1) enc4_thr<<<(unsigned)((warps + 3) / 4), 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mv2, Gl, spw);
            else enc4_branch<<<(unsigned)((warps + 3) / 4), 128>>>((const uint32_t *)A, C, (uint32_t *)B, Mv2, Gl, spw);
        }
    };
    launch(Gc);
    cudaDeviceSynchronize();
    uint8_t *hb = (uint8_t *)malloc((size_t)Gc * K * M), *hr = (uint8_t *)malloc((size_t)Gc * K * M);
    cudaMemcpy(hb, B, (size_t)Gc * K * M, cudaMemcpyDeviceToHost);
    cudaMemcpy(hr, R, (size_t)Gc * K * M, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t j = 0; j < (size_t)Gc * K * M; j++) bad += hb[j] != hr[j];
    for (int it = 0; it < 3; it++) launch(G);
    const int reps = argc > 5 ? atoi(argv[5]) : 10;
    cudaEventRecord(e0);
    for (int it = 0; it < reps; it++) launch(G);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("GF(%d) var=%d: G=%d spw=%d %.3f ms  %.1f GB/s source (%.1f%% of 3273)  mismatches=%zu  err=%s\n", q, var, G,
           spw, ms, (double)nA / ms / 1e6, (double)nA / ms / 1e6 / 3273 * 100, bad,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
