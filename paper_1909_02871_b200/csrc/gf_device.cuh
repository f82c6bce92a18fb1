// gf_device.cuh -- sm_100a device primitives for packed GF(2^w) bytes.
//
// Byte-permute lookup (the GPU form of the paper's shuffle algorithm,
// Alg. 1, "split each byte, look each part up in a small
// per-coefficient table, XOR the parts"): PRMT selects one of 8 bytes of a
// register pair with a 3-bit index per output byte, so a source byte splits
// into bit groups {0-2}, {3-5}, {6-7} and three PRMTs give the three partial
// products of 4 bytes at once.  Selector nibble 3 must stay clear (it means
// "replicate the sign bit"), which the masks 0x07 / 0x03 guarantee.
//
// Selector packing: t = (x >> s) & 0x07070707 holds the 4 indices in byte
// positions; t | (t >> 12) moves them into the four low nibbles in the order
// [b0, b2, b1, b3], so every lookup result is in that byte order.  Results
// are XOR-accumulated in permuted order and un-permuted once at the end with
// prmt(y, y, 0x3120).
#pragma once
#include <cstdint>

namespace gfr {

struct PrmtTab {            // per-coefficient split tables (tables.cpp)
    uint32_t t0lo, t0hi;    // T0[0..3], T0[4..7]   (bits 0-2 of the byte)
    uint32_t t1lo, t1hi;    // T1[0..3], T1[4..7]   (bits 3-5)
    uint32_t t2;            // T2[0..3]             (bits 6-7)
};

struct Sel {                // PRMT selectors of one 32-bit source word
    uint32_t s0, s1, s2;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
    return d;
}

// ((a * b) >> 32) + c on the FMA pipe (IMAD.HI), keeping shifts off the ALU pipe
__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ uint32_t mul_hi(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ Sel make_sel(uint32_t x)
{
    // t | (t >> 12) == t + (t >> 12) (disjoint bits) == mad.hi(t, 2^20, t)
    const uint32_t t0 = x & 0x07070707u;
    const uint32_t t1 = mul_hi(x, 1u << 29) & 0x07070707u;   // (x >> 3) & ..
    const uint32_t t2 = mul_hi(x, 1u << 26) & 0x03030303u;   // (x >> 6) & ..
    Sel s;
    s.s0 = mad_hi(t0, 1u << 20, t0);
    s.s1 = mad_hi(t1, 1u << 20, t1);
    s.s2 = mad_hi(t2, 1u << 20, t2);
    return s;
}

// c * x for 4 packed bytes, result in permuted byte order [b0, b2, b1, b3]
__device__ __forceinline__ uint32_t lookup_perm(const PrmtTab &T, const Sel &s)
{
    return prmt(T.t0lo, T.t0hi, s.s0) ^ prmt(T.t1lo, T.t1hi, s.s1) ^ prmt(T.t2, T.t2, s.s2);
}

__device__ __forceinline__ uint32_t unperm(uint32_t y) { return prmt(y, y, 0x3120u); }

// GF(4) on packed 2-bit words (PAPER.md:276-277 masks 0x55 / 0xaa):
// x * (a1 x + a0) = (a0 + a1) x + a1 mod x^2 + x + 1.
__device__ __forceinline__ uint32_t gf4_xtime(uint32_t a)
{
    const uint32_t hi = (a >> 1) & 0x55555555u;          // a1 at even positions
    return hi | (((a & 0x55555555u) ^ hi) << 1);         // new a0 = a1, new a1 = a0 ^ a1
}

}  // namespace gfr
