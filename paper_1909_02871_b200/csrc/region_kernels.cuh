// region_kernels.cuh -- gf_maddrc / gf_mulrc / XOR over one byte region.
//
// The paper's madd b := b + c a streamed over HBM: 3 bytes of
// traffic per source byte (read a, read b, write b), so the kernel is a
// grid-stride loop of 16-byte accesses with several chunks in flight per
// thread; per-coefficient tables arrive as kernel parameters (<= 24 B), so
// there is no shared-memory or global table traffic at all.
//
// Any length and alignment (reading X6): the body is the dst range aligned to
// 16 B; the < 16 B head and tail go through the same arithmetic one byte at a
// time (a byte in the low lane of a 32-bit word is a valid packed word).  When
// src is not 16-B aligned relative to dst the body loads 5 aligned 32-bit
// words of src and funnel-shifts them into place.
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

enum RegionOp {
    OP_XOR = 0,         // dst ^= src                       (c == 1, any field; GF(2) madd)
    OP_MADD_PRMT = 1,   // dst ^= c * src                   (GF(16), GF(256))
    OP_MADD_GF4 = 2,    // dst ^= c * src, c in {2, 3}      (GF(4) bit planes)
    OP_MUL_PRMT = 3,    // dst = c * dst                    (GF(16), GF(256))
    OP_MUL_GF4 = 4,     // dst = c * dst, c in {2, 3}
    OP_ZERO = 5         // dst = 0                          (mulrc with c == 0)
};

struct RegionParams {
    PrmtTab tab;        // tables of c (PRMT ops)
    uint32_t m0, m1;    // GF(4): masks of coefficient bits 0 and 1
};

template <int OP>
__device__ __forceinline__ uint32_t region_word(uint32_t d, uint32_t s, const RegionParams &p)
{
    if (OP == OP_XOR) return d ^ s;
    if (OP == OP_MADD_PRMT) return d ^ unperm(lookup_perm(p.tab, make_sel(s)));
    if (OP == OP_MUL_PRMT) return unperm(lookup_perm(p.tab, make_sel(d)));
    if (OP == OP_MADD_GF4) return d ^ (s & p.m0) ^ (gf4_xtime(s) & p.m1);
    if (OP == OP_MUL_GF4) return (d & p.m0) ^ (gf4_xtime(d) & p.m1);
    return 0u;  // OP_ZERO
}

__host__ __device__ constexpr bool op_reads_src(int op) { return op == OP_XOR || op == OP_MADD_PRMT || op == OP_MADD_GF4; }
__host__ __device__ constexpr bool op_reads_dst(int op) { return op != OP_ZERO; }

template <int OP>
__device__ __forceinline__ uint4 region_vec(uint4 d, uint4 s, const RegionParams &p)
{
    uint4 r;
    r.x = region_word<OP>(d.x, s.x, p);
    r.y = region_word<OP>(d.y, s.y, p);
    r.z = region_word<OP>(d.z, s.z, p);
    r.w = region_word<OP>(d.w, s.w, p);
    return r;
}

__device__ __forceinline__ uint4 ld_stream(const uint8_t *p)
{
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ld_plain(const uint8_t *p)
{
    return *reinterpret_cast<const uint4 *>(p);
}

// 16 source bytes at any address (src - (src & 3) is 4-B aligned)
__device__ __forceinline__ uint4 ld_src_unaligned(const uint8_t *src)
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(src);
    const uint32_t *w = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    const uint32_t sh = (uint32_t)(a & 3u) * 8u;
    uint32_t w0 = w[0], w1 = w[1], w2 = w[2], w3 = w[3];
    uint32_t w4 = sh ? w[4] : 0u;   // only touched when it holds a needed byte
    uint4 r;
    r.x = __funnelshift_r(w0, w1, sh);
    r.y = __funnelshift_r(w1, w2, sh);
    r.z = __funnelshift_r(w2, w3, sh);
    r.w = __funnelshift_r(w3, w4, sh);
    return r;
}

// SRC_MODE: 0 = src 16-B aligned and distinct from dst (read-only streaming
// path), 1 = src at any address, 2 = src == dst (exact aliasing, plain loads).
template <int OP, int SRC_MODE, int UNROLL>
__global__ void __launch_bounds__(256) region_kernel(uint8_t *dst, const uint8_t *src, size_t bytes,
                                                     RegionParams p)
{
    const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
    size_t head = (size_t)((16u - (da & 15u)) & 15u);
    if (head > bytes) head = bytes;
    const size_t nvec = (bytes - head) / 16;
    const size_t body_end = head + nvec * 16;
    const size_t tail = bytes - body_end;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nthreads = (size_t)gridDim.x * blockDim.x;

    // head / tail bytes, one per thread of the first 32 threads
    if (tid < 32) {
        size_t j = (size_t)-1;
        if (tid < head) j = tid;
        else if (tid >= 16 && tid - 16 < tail) j = body_end + (tid - 16);
        if (j != (size_t)-1) {
            uint32_t d = op_reads_dst(OP) ? dst[j] : 0u;
            uint32_t s = op_reads_src(OP) ? src[j] : 0u;
            dst[j] = (uint8_t)(region_word<OP>(d, s, p) & 0xFFu);
        }
    }

    uint8_t *db = dst + head;
    const uint8_t *sb = op_reads_src(OP) ? src + head : nullptr;
    for (size_t v0 = tid; v0 < nvec; v0 += nthreads * UNROLL) {
        uint4 d[UNROLL], s[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const size_t v = v0 + (size_t)u * nthreads;
            if (v < nvec) {
                if (op_reads_dst(OP)) d[u] = ld_plain(db + v * 16);
                if (op_reads_src(OP))
                    s[u] = SRC_MODE == 0 ? ld_stream(sb + v * 16)
                         : SRC_MODE == 1 ? ld_src_unaligned(sb + v * 16) : ld_plain(sb + v * 16);
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            const size_t v = v0 + (size_t)u * nthreads;
            if (v < nvec) {
                uint4 r = region_vec<OP>(op_reads_dst(OP) ? d[u] : make_uint4(0, 0, 0, 0),
                                         op_reads_src(OP) ? s[u] : make_uint4(0, 0, 0, 0), p);
                *reinterpret_cast<uint4 *>(db + v * 16) = r;
            }
        }
    }
}

}  // namespace gfr
