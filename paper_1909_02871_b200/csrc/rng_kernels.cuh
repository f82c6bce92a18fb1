// rng_kernels.cuh -- harness-only seeded input generator (not the method).
// Device twin of seeded_inputs (see its docstring for the definition):
//   word(seed, stream, w) = mix64(key + (w + 1) * GAMMA),  key = seed ^ stream * STREAM_MUL
//   byte(j) = byte (j & 7) of word(j >> 3)
#pragma once
#include <cstdint>

namespace gfr {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kStreamMul = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t rng_word(uint64_t key, uint64_t w)
{
    return mix64(key + (w + 1u) * kGamma);
}

// dst[r * cols + c] = byte(base + r * row_stride + c) & mask.
// Fast path (WORDS): cols, base, row_stride multiples of 8 and dst 8-B aligned:
// one 64-bit store per generator word.  Otherwise one byte per thread-step.
template <bool WORDS>
__global__ void __launch_bounds__(256) fill_random_kernel(uint8_t *dst, size_t rows, size_t cols,
                                                          uint64_t key, uint64_t base,
                                                          uint64_t row_stride, uint8_t mask)
{
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    if (WORDS) {
        const size_t wpr = cols / 8;                     // words per row
        const size_t total = rows * wpr;
        const uint64_t m8 = 0x0101010101010101ull * mask;
        for (size_t e = tid; e < total; e += nth) {
            const size_t r = e / wpr, cw = e % wpr;
            const uint64_t abs_byte = base + r * row_stride + cw * 8;
            reinterpret_cast<uint64_t *>(dst + r * cols)[cw] = rng_word(key, abs_byte >> 3) & m8;
        }
    } else {
        const size_t total = rows * cols;
        for (size_t e = tid; e < total; e += nth) {
            const size_t r = e / cols, c = e % cols;
            const uint64_t j = base + r * row_stride + c;
            dst[e] = (uint8_t)((rng_word(key, j >> 3) >> (8 * (j & 7))) & mask);
        }
    }
}

}  // namespace gfr
