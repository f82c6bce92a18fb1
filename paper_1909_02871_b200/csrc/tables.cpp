// tables.cpp -- host-side builder of the per-coefficient lookup tables the
// sm_100a kernels consume.  Product code: independent of oracle/ (no shared
// code, header or generator).
//
// Field arithmetic (Sec. II): the product of two elements is the
// carry-less polynomial product reduced modulo the field polynomial (reading
// X1: x^2+x+1, x^4+x+1, x^8+x^4+x^3+x+1).  Here it is computed by first
// forming the full 2w-1 bit carry-less product and then folding every bit of
// degree >= w with a precomputed residue x^d mod P.
//
// Packed bytes (reading X4): multiplication by c is linear
// over GF(2)^8 on the byte, so c * v = XOR over set bits b of v of the basis
// product c * e_b, where e_b = x^(b mod w) placed in word slot b / w.
//
// GPU table cut: the paper's 16-entry nibble
// tables tl[c] / th[c] (Alg. 1) become three byte tables
// indexed by bit groups {0-2}, {3-5}, {6-7} of a source byte, because the
// sm_100a byte permute (PRMT) selects among 8 bytes with a 3-bit index:
//     T0[v] = c * v,  T1[v] = c * (v << 3),  T2[v] = c * (v << 6)
// and c * byte = T0[b & 7] ^ T1[(b >> 3) & 7] ^ T2[b >> 6] by linearity.
// Each entry also carries the bit-plane masks of c (GF(2)/GF(4)) and the imul
// constants pow[c][j] = c * x^j of Alg. 2.
#include <cstdint>
#include <cstring>

#include "tables.h"

namespace gfr {

int field_width(int field)
{
    switch (field) {
    case 2: return 1;
    case 4: return 2;
    case 16: return 4;
    case 256: return 8;
    default: return -1;
    }
}

static uint32_t field_polynomial(int field)
{
    switch (field) {
    case 2: return 0x3u;
    case 4: return 0x7u;
    case 16: return 0x13u;
    case 256: return 0x11Bu;
    default: return 0u;
    }
}

// element product: full carry-less product, then fold high degrees
uint32_t elem_mul(int field, uint32_t a, uint32_t b)
{
    const int w = field_width(field);
    const uint32_t P = field_polynomial(field);
    uint32_t wide = 0;
    for (int k = 0; k < w; k++)
        wide ^= ((b >> k) & 1u) ? (a << k) : 0u;
    // residue[d] = x^d mod P for w <= d <= 2w-2
    uint32_t residue[16];
    uint32_t r = P ^ (1u << w);            // x^w = P - x^w (mod P)
    for (int d = w; d <= 2 * w - 2; d++) {
        residue[d - w] = r;
        r <<= 1;
        if (r >> w & 1u) r ^= P;
    }
    uint32_t out = wide & ((1u << w) - 1u);
    for (int d = w; d <= 2 * w - 2; d++)
        if (wide >> d & 1u) out ^= residue[d - w];
    return out;
}

uint32_t packed_mul(int field, uint32_t c, uint32_t v)
{
    const int w = field_width(field);
    uint32_t out = 0;
    for (int b = 0; b < 8; b++)
        if (v >> b & 1u)
            out ^= elem_mul(field, c, 1u << (b % w)) << (w * (b / w));
    return out & 0xFFu;
}

static uint32_t pack4(int field, uint32_t c, int shift, int first, int count)
{
    uint32_t word = 0;
    for (int j = 0; j < count; j++)
        word |= packed_mul(field, c, (uint32_t)(first + j) << shift) << (8 * j);
    return word;
}

int build_tables(int field, uint32_t *out, size_t cap_words)
{
    const int w = field_width(field);
    if (w < 0) return -1;
    const int q = field;
    if (cap_words < (size_t)q * kTableWords) return -2;
    for (int c = 0; c < q; c++) {
        uint32_t *t = out + (size_t)c * kTableWords;
        t[0] = pack4(field, c, 0, 0, 4);    // T0[0..3]
        t[1] = pack4(field, c, 0, 4, 4);    // T0[4..7]
        t[2] = pack4(field, c, 3, 0, 4);    // T1[0..3]
        t[3] = pack4(field, c, 3, 4, 4);    // T1[4..7]
        t[4] = pack4(field, c, 6, 0, 4);    // T2[0..3]
        t[5] = (c & 1) ? 0xFFFFFFFFu : 0u;  // bit-plane mask of coefficient bit 0
        t[6] = (c & 2) ? 0xFFFFFFFFu : 0u;  // bit-plane mask of coefficient bit 1
        t[7] = 0u;
        // imul constants (Alg. 2): pow[c][j] = c * x^j
        for (int j = 0; j < 8; j++) t[8 + j] = j < w ? elem_mul(field, c, 1u << j) : 0u;
    }
    return 0;
}

int build_products(int field, uint8_t *mul)
{
    if (field_width(field) < 0) return -1;
    for (uint32_t a = 0; a < 256; a++)
        for (uint32_t b = 0; b < 256; b++)
            mul[a * 256 + b] = (a < (uint32_t)field && b < (uint32_t)field) ? (uint8_t)elem_mul(field, a, b) : 0;
    return 0;
}

int build_inverses(int field, uint8_t *inv)
{
    if (field_width(field) < 0) return -1;
    for (int a = 0; a < 256; a++) inv[a] = 0;
    for (uint32_t a = 1; a < (uint32_t)field; a++)
        for (uint32_t x = 1; x < (uint32_t)field; x++)
            if (elem_mul(field, a, x) == 1u) { inv[a] = (uint8_t)x; break; }
    return 0;
}

}  // namespace gfr
