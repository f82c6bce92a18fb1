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
// Selector packing: the indices of bit group g sit at 3-bit fields in byte
// positions; the four low nibbles of the selector must hold them in the order
// [b0, b2, b1, b3], so every lookup result is in that byte order.  Results
// are XOR-accumulated in permuted order and un-permuted once at the end with
// prmt(y, y, 0x3120).  One AND and one IMAD.HI per group (make_sel).
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

// Selector multipliers, read from the constant bank: ptxas strength-reduces a
// multiply by a known power of two into SHF / LEA.HI on the ALU pipe (the pipe
// the PRMTs and XORs need), but must issue IMAD.HI (FMA pipe) for a value it
// cannot see.  Never written after load.
__constant__ uint32_t c_selmul[3] = {1u << 20, (1u << 29) | (1u << 17), (1u << 26) | (1u << 14)};

__device__ __forceinline__ Sel make_sel(uint32_t x)
{
    // t0 = x & 0x07..: fields at bits 8j; t0 + (t0 >> 12) = hi(t0 * 2^20) + t0
    //   adds b2 -> nibble 1 and b3 -> nibble 3 (disjoint bits, so + is |).
    // t1 = x & 0x38..: hi(t1 * (2^29 + 2^17)) = (t1 >> 3) + (t1 >> 15): every
    //   bit of t1 is >= 3, so the low word of t1 * 2^29 is 0 and that of
    //   t1 * 2^17 is < 2^31 -- no carry into the high word.
    // t2 = x & 0xC0..: hi(t2 * (2^26 + 2^14)) = (t2 >> 6) + (t2 >> 18), same
    //   argument (bits >= 6).
    // Nibble bit 3 stays clear in all three (it would mean "replicate sign").
    const uint32_t t0 = x & 0x07070707u, t1 = x & 0x38383838u, t2 = x & 0xC0C0C0C0u;
    Sel s;
    s.s0 = mad_hi(t0, c_selmul[0], t0);
    s.s1 = mul_hi(t1, c_selmul[1]);
    s.s2 = mul_hi(t2, c_selmul[2]);
    return s;
}

// c * x for 4 packed bytes, result in permuted byte order [b0, b2, b1, b3]
__device__ __forceinline__ uint32_t lookup_perm(const PrmtTab &T, const Sel &s)
{
    return prmt(T.t0lo, T.t0hi, s.s0) ^ prmt(T.t1lo, T.t1hi, s.s1) ^ prmt(T.t2, T.t2, s.s2);
}

__device__ __forceinline__ uint32_t unperm(uint32_t y) { return prmt(y, y, 0x3120u); }

// mbarrier helpers (shared-memory addresses): producer / consumer rings of the
// product-row and lane-k kernels
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a)
{
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" :: "r"(a) : "memory");
}
__device__ __forceinline__ void mbar_arrive_n(uint32_t a, uint32_t n)
{
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0], %1; }" :: "r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t a, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{ .reg .pred p;\n"
                 "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    return ok != 0;
}
// a waiter that is known to run ahead (the producers): poll rarely, every
// failed poll is a shared-memory access on the pipe the gatherers are bound by
__device__ __forceinline__ void mbar_wait_sleepy(uint32_t a, uint32_t parity)
{
    while (!mbar_test(a, parity)) __nanosleep(256);
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity)
{
    asm volatile("{ .reg .pred p;\n"
                 "PR_WAIT_%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
                 "@!p bra PR_WAIT_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}

// number of nonzero bytes of x (the fused Freivalds checks count differing bytes)
__device__ __forceinline__ uint32_t nz_bytes(uint32_t x)
{
    x |= x >> 4;
    x |= x >> 2;
    x |= x >> 1;
    return __popc(x & 0x01010101u);
}

// GF(4) on packed 2-bit words (PAPER.md:276-277 masks 0x55 / 0xaa):
// x * (a1 x + a0) = (a0 + a1) x + a1 mod x^2 + x + 1.
__device__ __forceinline__ uint32_t gf4_xtime(uint32_t a)
{
    const uint32_t hi = (a >> 1) & 0x55555555u;          // a1 at even positions
    return hi | (((a & 0x55555555u) ^ hi) << 1);         // new a0 = a1, new a1 = a0 ^ a1
}

}  // namespace gfr
