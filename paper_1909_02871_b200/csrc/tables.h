// tables.h -- host table builder (see tables.cpp)
#pragma once
#include <cstddef>
#include <cstdint>

namespace gfr {

constexpr int kTableWords = 16;  // uint32 words per coefficient entry

int field_width(int field);                                  // -1 if unsupported
uint32_t elem_mul(int field, uint32_t a, uint32_t b);        // a * b in F_q
uint32_t packed_mul(int field, uint32_t c, uint32_t v);      // c * byte v (packed words)
int build_tables(int field, uint32_t *out, size_t cap_words);  // 0, -1 field, -2 cap
int build_inverses(int field, uint8_t *inv);                  // inv[a] * a = 1, inv[0] = 0
int build_products(int field, uint8_t *mul);                  // mul[a*256 + b] = a * b (elements)

}  // namespace gfr
