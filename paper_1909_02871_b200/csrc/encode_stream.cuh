// encode_stream.cuh -- batched RLNC encode for few coded packets (K <= 4),
// the paper's own measurement shape (N = 16 source packets, K = 1 coded
// packet):
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// With K = 1 the encode is a streaming reduction: every source byte is read
// once and multiplied once, so it is bound by HBM (17 bytes of traffic per 16
// source bytes for N = 16), not by arithmetic -- provided the multiply stays
// under ~12 ALU operations per 32-bit word at HBM speed.  One thread owns one
// 16-byte column chunk of one generation: it loads the chunks of eight (GF(2),
// GF(4)) or four source packets at a time (16-byte non-allocating loads, all
// in flight together),
// multiplies each by its coefficient and XORs into K accumulators.  Per-field
// word arithmetic (coefficient tables from gf_init's table of tables,
// L1-resident):
//   GF(2):   acc ^= a & M0                                 1 LOP3
//   GF(4):   the paper's imul (Alg. 2): 2 IMAD + 1 LOP3
//            (a & 0x55..)*c ^ ((a>>1) & 0x55..)*(x c)
//   GF(16):  imul on the four nibble bit planes: 4 IMAD + 2 LOP3
//   GF(256): three byte-permute split tables over bit groups {0-2}, {3-5},
//            {6-7} (Alg. 1's shuffle): 3 PRMT + 3 AND +
//            2 LOP3 on the ALU pipe, selector packing on the FMA pipe;
//            results in PRMT byte order, un-permuted once per output word.
// Grid-stride over (generation, chunk); packets of 512 B or more give
// warp-uniform coefficients (broadcast table loads).
#pragma once
#include <cstdint>

#include "gf_device.cuh"
#include "tables.h"

namespace gfr {

constexpr int kStThreads = 256;

struct StreamParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    const uint32_t *tabs;   // table of tables of the field (16 words per coefficient)
    size_t M16;             // chunks per packet (16-byte chunks, or 4-byte ones for word-aligned packets)
    size_t total;           // batch * chunks per packet
    int N, K;
    uint32_t qmask;
};

__device__ __forceinline__ uint4 st_ld_stream(const uint4 *p)
{
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// acc ^= c * x for one 32-bit word, e = the coefficient's table entry
template <int F> struct StreamOp;
template <> struct StreamOp<2> {
    static constexpr bool kPermuted = false;
    struct E { uint32_t m0; };
    __device__ __forceinline__ static E entry(const uint32_t *t) { return E{__ldg(t + 5)}; }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e) { return x & e.m0; }
};
template <> struct StreamOp<4> {
    static constexpr bool kPermuted = false;
    struct E { uint32_t p0, p1; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(t + 8));
        return E{v.x, v.y};
    }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e)
    {
        return ((x & 0x55555555u) * e.p0) ^ ((mul_hi(x, 1u << 31) & 0x55555555u) * e.p1);
    }
};
template <> struct StreamOp<16> {
    static constexpr bool kPermuted = false;
    struct E { uint32_t p0, p1, p2, p3; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(t + 8));
        return E{v.x, v.y, v.z, v.w};
    }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e)
    {
        const uint32_t n0 = x & 0x11111111u, n1 = mul_hi(x, 1u << 31) & 0x11111111u;
        const uint32_t n2 = mul_hi(x, 1u << 30) & 0x11111111u, n3 = mul_hi(x, 1u << 29) & 0x11111111u;
        return (n0 * e.p0) ^ (n1 * e.p1) ^ (n2 * e.p2) ^ (n3 * e.p3);
    }
};
template <> struct StreamOp<256> {
    static constexpr bool kPermuted = true;
    struct E { PrmtTab T; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(t));
        E e;
        e.T.t0lo = v.x; e.T.t0hi = v.y; e.T.t1lo = v.z; e.T.t1hi = v.w; e.T.t2 = __ldg(t + 4);
        return e;
    }
    // three split-table PRMTs (bit groups {0-2}, {3-5}, {6-7}): 8 ALU + 5 FMA-pipe ops
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e) { return lookup_perm(e.T, make_sel(x)); }
};

// generic V-word chunks; used with V = 1 (4-byte chunks) for packets that are
// only word aligned (e.g. C1's M = 1500)
template <int V> __device__ __forceinline__ void st_load(uint32_t (&a)[V], const uint8_t *p)
{
    if constexpr (V == 4) {
        const uint4 v = st_ld_stream(reinterpret_cast<const uint4 *>(p));
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
    } else {
        a[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    }
}
template <int V> __device__ __forceinline__ void st_store(uint8_t *p, const uint32_t (&r)[V])
{
    if constexpr (V == 4) *reinterpret_cast<uint4 *>(p) = make_uint4(r[0], r[1], r[2], r[3]);
    else *reinterpret_cast<uint32_t *>(p) = r[0];
}

// 16-byte chunks (packets 16-byte aligned): the measured fast form, kept as
// written for uint4 (a generic word-array version of it measured 2-6% slower)
template <int F, int KT>
__global__ void __launch_bounds__(kStThreads) encode_stream_kernel(StreamParams p)
{
    using Op = StreamOp<F>;
    constexpr int kStBatch = F <= 4 ? 8 : 4;                  // source chunks loaded together (measured)
    const size_t stride = (size_t)gridDim.x * kStThreads;
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t g = t / p.M16, ch = t - g * p.M16;
        const uint4 *Ag = reinterpret_cast<const uint4 *>(p.A + g * (size_t)p.N * (p.M16 * 16)) + ch;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint4 acc[KT];
#pragma unroll
        for (int k = 0; k < KT; k++) acc[k] = make_uint4(0u, 0u, 0u, 0u);
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint4 a[kStBatch];
#pragma unroll
            for (int b = 0; b < kStBatch; b++)
                a[b] = i0 + b < p.N ? st_ld_stream(Ag + (size_t)(i0 + b) * p.M16) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int b = 0; b < kStBatch; b++) {
                if (i0 + b >= p.N) break;
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    if (k < p.K) {
                        const uint32_t c = __ldg(Cg + (size_t)(i0 + b) * p.K + k) & p.qmask;
                        const typename Op::E e = Op::entry(p.tabs + (size_t)c * kTableWords);
                        acc[k].x ^= Op::mul(a[b].x, e);
                        acc[k].y ^= Op::mul(a[b].y, e);
                        acc[k].z ^= Op::mul(a[b].z, e);
                        acc[k].w ^= Op::mul(a[b].w, e);
                    }
                }
            }
        }
        uint4 *Bg = reinterpret_cast<uint4 *>(p.B + g * (size_t)p.K * (p.M16 * 16)) + ch;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
                uint4 r = acc[k];
                if (Op::kPermuted) r = make_uint4(unperm(r.x), unperm(r.y), unperm(r.z), unperm(r.w));
                Bg[(size_t)k * p.M16] = r;
            }
        }
    }
}

template <int F, int KT, int V>
__global__ void __launch_bounds__(kStThreads) encode_stream_words_kernel(StreamParams p)
{
    using Op = StreamOp<F>;
    constexpr int kStBatch = F <= 4 ? 8 : 4;                  // source chunks loaded together (measured)
    constexpr size_t kChunk = 4 * V;                           // bytes per chunk
    const size_t Mc = p.M16;                                   // chunks per packet
    const size_t M = Mc * kChunk;
    const size_t stride = (size_t)gridDim.x * kStThreads;
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t g = t / Mc, ch = t - g * Mc;
        const uint8_t *Ag = p.A + g * (size_t)p.N * M + ch * kChunk;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint32_t acc[KT][V];
#pragma unroll
        for (int k = 0; k < KT; k++)
#pragma unroll
            for (int v = 0; v < V; v++) acc[k][v] = 0u;
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint32_t a[kStBatch][V];
#pragma unroll
            for (int b = 0; b < kStBatch; b++) {
                if (i0 + b < p.N) st_load<V>(a[b], Ag + (size_t)(i0 + b) * M);
                else
#pragma unroll
                    for (int v = 0; v < V; v++) a[b][v] = 0u;
            }
#pragma unroll
            for (int b = 0; b < kStBatch; b++) {
                if (i0 + b >= p.N) break;
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    if (k < p.K) {
                        const uint32_t c = __ldg(Cg + (size_t)(i0 + b) * p.K + k) & p.qmask;
                        const typename Op::E e = Op::entry(p.tabs + (size_t)c * kTableWords);
#pragma unroll
                        for (int v = 0; v < V; v++) acc[k][v] ^= Op::mul(a[b][v], e);
                    }
                }
            }
        }
        uint8_t *Bg = p.B + g * (size_t)p.K * M + ch * kChunk;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
                uint32_t r[V];
#pragma unroll
                for (int v = 0; v < V; v++) r[v] = Op::kPermuted ? unperm(acc[k][v]) : acc[k][v];
                st_store<V>(Bg + (size_t)k * M, r);
            }
        }
    }
}

}  // namespace gfr
