// encode_tmem.cuh -- batched RLNC encode with the multiples of the source words
// held as lookup tables in tensor memory (TMEM), indexed by the coefficients.
//
//   B[g][k][m] = XOR_{i < N} C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Over F_q, q = 2^w, multiplication by c is linear over GF(2):
//   c * a = XOR_{j < w} c_j * (x^j a)        (c_j = bit j of c; §II)
// so a coded word b_k is the XOR of the basis words e_t = x^j a_i (t = i w + j)
// selected by the coefficient bits.  The basis words of a span are cut into
// groups of four; a group's 16 XOR-subsets form a table T[0..15], and the
// contribution of the group to coded packet k is ONE lookup T[idx(k)], idx(k)
// = the four coefficient bits that select the group's basis words.  This is the
// paper's split-table idea (Alg. 1: precompute the products
// of a 4-bit part once, look them up, XOR the parts) turned around: the
// tables hold products of the DATA with every 4-bit coefficient part, so the
// table index depends only on C and is the same for all 32 lanes of a warp.
//   GF(2):   group = 4 sources,                   idx = c_i c_i+1 c_i+2 c_i+3
//   GF(4):   group = 2 sources {a, xa, b, xb},    idx = c_i | c_i+1 << 2
//   GF(16):  group = 1 source {a, xa, x^2a, x^3a}, idx = c_i
//   GF(256): 2 groups per source (x^0..3 a, x^4..7 a), idx = low / high nibble
// A warp-uniform index is what TMEM serves: tcgen05.ld reads one column (a
// uniform address) for all 32 lanes of the warp's lane quarter, on the tensor
// memory datapath beside the shared-memory pipe (.x2 loads
// ~130 B/clk per SM from ordinary warps, tools/ubench_tmem2.cu).
//
// Layout (W = 2 words per lane, the instantiated width): warp wid owns TMEM
// lanes 32 (wid % 4) .. +31 and 128 columns (4 groups x 16 combos x 2 words).
// Lane l holds words 2l, 2l+1 of a 64-word (256-byte) span of every packet; a
// work unit is (generation, span), and each warp walks a contiguous range of
// units.  A unit is processed in passes of 32 coded packets (accumulators
// acc[32][2] in registers) and steps of 4 groups: per step the lane builds
// the 4 x 16 combos of its two words (11 XORs per group and word, plus the
// field's x-multiples), stores them with one tcgen05.st.32x32b.x32 per group,
// and each coded packet XORs four tcgen05.ld.32x32b.x2 results into its
// accumulator (two LOP3 per word).  (W = 4, .x4 loads and 16-byte stores,
// compiles and is bit-exact but measured slower: 128 accumulator registers
// spill at 8 warps.)
// The TMEM column addresses of every (pass, group, k) are precomputed per
// warp and generation in shared memory and read with broadcast LDS.128.
// Source words stream through a per-warp ring of kTmRing steps: one lane
// issues one TMA tile load per step (2-D tensor map over A viewed as
// [batch N rows][M / 4 words], box SPS rows x 32 W words), completing on the
// stage's mbarrier; rows and words past the end of A are zero-filled.  B
// leaves per (unit, pass) through a staging tile and one 3-D TMA tile store
// (GF(4) / GF(16) / GF(256)) or 8-byte stores (GF(2)); see tm_tma_store_on.
// HBM traffic is the algorithmic N*M + K*M (+ N*K) per generation (each
// pass > 0 re-reads the span's sources, from L2).
//
// Requirements (checked by the router): M % 16 == 0, 16-byte aligned A and B.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "gf_device.cuh"

namespace gfr {

// W (template parameter, 2 or 4): 32-bit words per lane per span; a span is
// 32 W words of every packet, a lookup one tcgen05.ld.32x32b.xW
constexpr int kTmKB = 32;                       // coded packets per pass
constexpr int kTmGPB = 4;                       // groups per step
constexpr int kTmRing = 4;                      // steps of source words in flight per warp
__host__ __device__ constexpr int tm_span_words(int W) { return 32 * W; }
__host__ __device__ constexpr int tm_cols_per_warp(int W) { return kTmGPB * 16 * W; }   // 128 / 256

struct TmParams {
    const uint8_t *A;      // [batch][N][M]
    const uint8_t *C;      // [batch][N][K]
    uint8_t *B;            // [batch][K][M]
    uint32_t Mw;           // 32-bit words per packet
    uint32_t spans;        // ceil(Mw / 64)
    int N, K;
    int NG;                // groups, ceil(N w / 4) rounded up to kTmGPB
    int passes;            // ceil(K / 32)
    uint64_t units;        // batch * spans
    uint64_t upw;          // units per warp
    // fused Freivalds check (T > 0 instantiations; gf_encode_verify_batch, K <= 64)
    const uint8_t *U;      // [batch][1][2][N]: u_j = C r_j over F_q
    const uint32_t *RB;    // [batch][2][kw]: bit k of word k / 32 = r_jk
    int kw;
    unsigned long long *mismatch;   // [batch] += differing bytes
    uint64_t fault;        // harness fault injection (FT): g << 32 | k << 20 | word
};

// sources per step (kTmGPB groups of 4 basis words, w basis words per source)
__host__ __device__ constexpr int tm_sps(int logw) { return (4 * kTmGPB) >> logw; }

// per-warp shared memory: TMEM addresses [passes][steps][kTmKB / 4][kTmGPB][4]
// (one word per (pass, group, k)), the check's addresses [NG][T] (T > 0),
// the store staging tile [kTmKB][32 W] words, the source ring, then one
// mbarrier per ring stage
__host__ __device__ constexpr size_t tm_tab_bytes(int NG, int passes) { return (size_t)passes * NG * kTmKB * 4; }
// B leaves through TMA stores from a staging tile for GF(4) / GF(16) / GF(256)
// (C5 GF(4): 1.81 -> 2.06 TB/s: the per-row store addresses and their memory
// descriptors had cost ~45 ALU instructions per step), through 8-byte STG
// for GF(2), whose HBM-bound loop lost 7% with the TMA stores
// (profiles/r02_exp_tmem_v9.txt)
__host__ __device__ constexpr bool tm_tma_store_on(int logw) { return logw != 0; }
__host__ __device__ constexpr size_t tm_stage_bytes(int logw, int W)
{
    return tm_tma_store_on(logw) ? (size_t)kTmKB * tm_span_words(W) * 4 : 0;
}
__host__ __device__ constexpr size_t tm_tabu_bytes(int NG, int T) { return ((size_t)NG * T * 4 + 127) / 128 * 128; }
__host__ __device__ constexpr size_t tm_warp_bytes(int logw, int NG, int passes, int T = 0, int W = 2)
{
    // (a multiple of 128 bytes: TMA destinations are 128-byte aligned)
    return (tm_tab_bytes(NG, passes) + tm_tabu_bytes(NG, T) + tm_stage_bytes(logw, W) + (size_t)kTmRing * tm_sps(logw) * tm_span_words(W) * 4 + kTmRing * 8 + 127) / 128 * 128;
}

// x * a on packed w-bit elements (bit j of an element = coefficient of x^j)
template <int LOGW>
__device__ __forceinline__ uint32_t tm_xtime(uint32_t a)
{
    if constexpr (LOGW == 1) {
        // x (a1 x + a0) = (a0 + a1) x + a1: with t = a >> 1, new a0 = t & 0x55..,
        // new a1 = ((a ^ t) & 0x55..) << 1 (two LOP3, one SHF, one IMAD)
        const uint32_t t = a >> 1, u = (a ^ t) & 0x55555555u;
        return (t & 0x55555555u) | (u + u);
    } else if constexpr (LOGW == 2) {                         // x^4 + x + 1
        const uint32_t h = (a >> 3) & 0x11111111u;
        return ((a << 1) & 0xEEEEEEEEu) ^ (h * 3u);
    } else {                                                  // x^8 + x^4 + x^3 + x + 1
        const uint32_t h = (a >> 7) & 0x01010101u;
        return ((a << 1) & 0xFEFEFEFEu) ^ (h * 0x1Bu);
    }
}

#define TM_R8(v, o) "r"(v[o]), "r"(v[o + 1]), "r"(v[o + 2]), "r"(v[o + 3]), "r"(v[o + 4]), "r"(v[o + 5]), "r"(v[o + 6]), "r"(v[o + 7])
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&v)[32])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                 "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 :: "r"(taddr), TM_R8(v, 0), TM_R8(v, 8), TM_R8(v, 16), TM_R8(v, 24) : "memory");
}
#undef TM_R8

__device__ __forceinline__ void tm_ld2(uint32_t taddr, uint32_t &x, uint32_t &y)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(taddr));
}

__device__ __forceinline__ void tm_ld4(uint32_t taddr, uint32_t *x)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(taddr));
}
template <int W>
__device__ __forceinline__ void tm_ldw(uint32_t taddr, uint32_t *x)
{
    if constexpr (W == 2) tm_ld2(taddr, x[0], x[1]);
    else tm_ld4(taddr, x);
}

// wait for this thread's outstanding tcgen05.ld; the loaded registers pass
// through the asm so that no use of them is scheduled above the wait
#define TM_P8(v, o) "+r"(v[o]), "+r"(v[o + 1]), "+r"(v[o + 2]), "+r"(v[o + 3]), "+r"(v[o + 4]), "+r"(v[o + 5]), "+r"(v[o + 6]), "+r"(v[o + 7])
__device__ __forceinline__ void tm_wait_ld32(uint32_t (&v)[32])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : TM_P8(v, 0), TM_P8(v, 8), TM_P8(v, 16), TM_P8(v, 24) :: "memory");
}
#undef TM_P8

#define TM_Q8(v, o) "+r"(v[o]), "+r"(v[o + 1]), "+r"(v[o + 2]), "+r"(v[o + 3]), "+r"(v[o + 4]), "+r"(v[o + 5]), "+r"(v[o + 6]), "+r"(v[o + 7])
__device__ __forceinline__ void tm_wait_ld16(uint32_t (&v)[16])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" : TM_Q8(v, 0), TM_Q8(v, 8) :: "memory");
}
#undef TM_Q8

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one TMA tile store: box of 32 W words x kTmKB rows x 1 generation from
// shared memory to B (3-D tensor map [batch][K][M / 4]: rows past K and words
// past M are clipped by the hardware)
__device__ __forceinline__ void tm_tma_store(const CUtensorMap *map, uint32_t x, uint32_t y, uint32_t z, uint32_t ssrc)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                 :: "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(ssrc) : "memory");
}

// f(integral_constant<int, i>) for i = 0 .. NI-1, unrolled at compile time
template <int I, int NI, class F>
__device__ __forceinline__ void tm_unroll_i(F &&f)
{
    if constexpr (I < NI) {
        f(std::integral_constant<int, I>{});
        tm_unroll_i<I + 1, NI>(f);
    }
}
template <int NI, class F>
__device__ __forceinline__ void tm_unroll(F &&f) { tm_unroll_i<0, NI>(f); }

// one TMA tile load (box SPS rows x 32 W words at word x, row y of A) into
// shared memory, completing its bytes on an mbarrier
__device__ __forceinline__ void tm_tma_load(uint32_t sdst, const CUtensorMap *map, uint32_t x, uint32_t y, uint32_t bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(sdst), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar) : "memory");
}

// Host: the tensor map of B for the TMA stores (3-D: M / 4 words, K rows,
// batch generations; box 32 W words x kTmKB rows x 1).
static inline bool tm_make_map_b(CUtensorMap *map, void *B, uint64_t batch, uint64_t K, uint64_t M, int W = 2);

// Host: the driver's tensor-map encoder, resolved once by gf_init (no driver
// call on the launch path but the encode itself, which is host-only work).
static inline PFN_cuTensorMapEncodeTiled_v12000 &tm_encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    return fn;
}
static inline bool tm_resolve_encoder()
{
    if (__atomic_load_n(&tm_encode_fn(), __ATOMIC_ACQUIRE)) return true;
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
        return false;
    __atomic_store_n(&tm_encode_fn(), reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f), __ATOMIC_RELEASE);
    return true;
}

// Host: the tensor map of A for the kernel's source ring (2-D: M / 4 words
// per row, rows of stride M bytes; box 32 W words x SPS rows).  M % 16 == 0
// and 16-byte aligned A (TMA's stride / address rules).  Returns false when
// the encoder was not resolved (tm_resolve_encoder) or the encode fails.
static inline bool tm_make_map(CUtensorMap *map, const void *A, uint64_t rows, uint64_t M, int logw, int W = 2)
{
    const PFN_cuTensorMapEncodeTiled_v12000 fn = __atomic_load_n(&tm_encode_fn(), __ATOMIC_ACQUIRE);
    if (!fn) return false;
    const cuuint64_t dims[2] = {M / 4, rows};
    const cuuint64_t strides[1] = {M};
    const cuuint32_t box[2] = {(cuuint32_t)tm_span_words(W), (cuuint32_t)tm_sps(logw)};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(A), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static inline bool tm_make_map_b(CUtensorMap *map, void *B, uint64_t batch, uint64_t K, uint64_t M, int W)
{
    const PFN_cuTensorMapEncodeTiled_v12000 fn = __atomic_load_n(&tm_encode_fn(), __ATOMIC_ACQUIRE);
    if (!fn) return false;
    const cuuint64_t dims[3] = {M / 4, K, batch};
    const cuuint64_t strides[2] = {M, K * M};
    const cuuint32_t box[3] = {(cuuint32_t)tm_span_words(W), (cuuint32_t)kTmKB, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, B, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

__device__ __forceinline__ void tm_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}

// Grid: 1-D, WPC warps per block, one block per SM (TMEM: WPC / 4 x 64 W columns).
//
// T > 0: the fused Freivalds check of gf_encode_verify_batch (SURVEY 8(c) step
// 7, 8(f) NEXT-4) with T binary projections r_j (K <= 64): B == A C iff
// sum_k r_jk b_k == sum_i u_ji a_i with u_j = C r_j.  The A side is one more
// lookup per group and projection in the first pass (u_j restricted to the
// group's basis words is a 4-bit index into the same table); the B side XORs
// every finished coded word into y2_j where r_jk = 1, before its store.  At the
// end of a unit the differing bytes of y1_j and y2_j are counted into
// mismatch[g].  FT: the harness fault injection (gf_set_verify_fault), a
// separate instantiation.
template <int LOGW, int WPC, int T = 0, bool FT = false, int W = 2>
__global__ void __launch_bounds__(WPC * 32, 1) encode_tmem_kernel(TmParams p, const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmB)
{
    constexpr int w = 1 << LOGW;
    constexpr int SPS = tm_sps(LOGW);
    constexpr int SPG = SPS / kTmGPB > 0 ? SPS / kTmGPB : 1;      // sources per group (GF(256): 2 groups per source)
    constexpr int SW = tm_span_words(W), CPW = tm_cols_per_warp(W);
    static_assert(W == 2 || W == 4, "2 or 4 words per lane");
    static_assert((WPC / 4) * CPW <= 512, "TMEM columns");
    constexpr uint32_t kCols = (WPC / 4) * CPW <= 128 ? 128 : (WPC / 4) * CPW <= 256 ? 256 : 512;
    extern __shared__ __align__(1024) uint8_t smem8[];
    __shared__ uint32_t s_tbase;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(&s_tbase)), "n"(kCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this warp's TMEM: lanes 32 (wid % 4) .., columns (wid / 4) * CPW ..
    const uint32_t tb = s_tbase + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(wid >> 2) * CPW;

    const int N = p.N, K = p.K, NG = p.NG, passes = p.passes, steps = NG / kTmGPB;
    const uint32_t Mw = p.Mw, spans = p.spans;
    const size_t tabb = tm_tab_bytes(NG, passes);
    uint8_t *wbase = smem8 + (size_t)wid * tm_warp_bytes(LOGW, NG, passes, T, W);
    uint32_t *tab = reinterpret_cast<uint32_t *>(wbase);
    uint32_t *tabu = reinterpret_cast<uint32_t *>(wbase + tabb);               // [NG][T]
    const uint32_t stg_s = (uint32_t)__cvta_generic_to_shared(wbase + tabb + tm_tabu_bytes(NG, T));   // [kTmKB][SW]
    const uint32_t *ring = reinterpret_cast<const uint32_t *>(wbase + tabb + tm_tabu_bytes(NG, T) + tm_stage_bytes(LOGW, W));
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    const uint32_t bar_s = ring_s + kTmRing * SPS * SW * 4;
    if (lane < kTmRing) mbar_init(bar_s + 8 * lane, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    const uint64_t u0 = ((uint64_t)blockIdx.x * WPC + wid) * p.upw;
    const uint64_t u1 = u0 + p.upw < p.units ? u0 + p.upw : p.units;
    const int64_t nsteps = u0 < u1 ? (int64_t)(u1 - u0) * passes * steps : 0;

    // Step cursors (no divisions in the loop): a step is (unit, pass, group
    // step gs); unit = (generation g, span sp).  The producer runs
    // kTmRing - 1 steps ahead of the consumer.
    struct Cur {
        uint64_t g; uint32_t sp; int pass, gs; int64_t t;
    };
    auto advance = [&](Cur &c) {
        c.t++;
        if (++c.gs == steps) {
            c.gs = 0;
            if (++c.pass == passes) {
                c.pass = 0;
                if (++c.sp == spans) { c.sp = 0; c.g++; }
            }
        }
    };
    Cur pc{u0 / spans, (uint32_t)(u0 % spans), 0, 0, 0};
    Cur cc = pc;
    // producer: one TMA tile load per step, rows g N + gs SPS .. + SPS - 1,
    // words sp SW .. + SW - 1 (rows past the generation's N belong to the next
    // one or lie past the end of A, and only meet zero coefficients; bytes past
    // the packet end belong to lanes that never store)
    auto issue = [&]() {
        if (pc.t < nsteps) {
            if (lane == 0) {
                const uint32_t st = (uint32_t)(pc.t % kTmRing);
                tm_expect_tx(bar_s + 8 * st, SPS * SW * 4u);
                tm_tma_load(ring_s + st * (SPS * SW * 4u), &tmA, pc.sp * (uint32_t)SW,
                            (uint32_t)(pc.g * N) + (uint32_t)(pc.gs * SPS), bar_s + 8 * st);
            }
            advance(pc);
        }
    };

#pragma unroll 1
    for (int t = 0; t < kTmRing - 1; t++) issue();

    uint64_t cur_g = ~0ull;
    uint32_t bad = 0;                                // check: differing bytes of this warp's current generation
    int fk = -1;                                     // FT: coded packet to corrupt in this generation
    uint32_t y1[T > 0 ? T : 1][W], y2[T > 0 ? T : 1][W], rw[T > 0 ? T : 1];
#pragma unroll
    for (int j = 0; j < (T > 0 ? T : 1); j++) {
        rw[j] = 0u;
#pragma unroll
        for (int wd = 0; wd < W; wd++) y1[j][wd] = y2[j][wd] = 0u;
    }
    (void)fk; (void)y1; (void)y2; (void)rw;
    uint32_t acc[kTmKB][W];
#pragma unroll
    for (int k = 0; k < kTmKB; k++)
#pragma unroll
        for (int wd = 0; wd < W; wd++) acc[k][wd] = 0u;

#pragma unroll 1
    for (int64_t t = 0; t < nsteps; t++) {
        __syncwarp();                                // every lane is done with the stage issue() refills
        issue();
        const uint64_t g = cc.g;
        const int pass = cc.pass, gs = cc.gs;
        if (g != cur_g) {                            // this warp's TMEM lookup addresses for generation g
            if constexpr (T > 0) {
                bad = __reduce_add_sync(0xffffffffu, bad);
                if (lane == 0 && bad && cur_g != ~0ull) atomicAdd(p.mismatch + cur_g, (unsigned long long)bad);
                bad = 0;
                if constexpr (FT)
                    fk = (g == ((p.fault >> 32) & 0x7FFFFFFFu)) ? (int)((p.fault >> 20) & 0xFFFu) : -1;
            }
            cur_g = g;
            const uint8_t *Cg = p.C + g * (size_t)N * K;
            __syncwarp();
            for (int e = lane; e < (int)(tabb / 4); e += 32) {
                // e = (((ps * steps + st) * 8 + kq) * kTmGPB + sl) * 4 + kk
                const int kk = e & 3, sl = (e >> 2) & (kTmGPB - 1), kq = (e >> 4) & 7;
                const int pst = e >> 7, st = pst % steps, ps = pst / steps;
                const int k = ps * kTmKB + kq * 4 + kk, grp = st * kTmGPB + sl;
                uint32_t idx = 0;
                if (k < K) {
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        const int tt = 4 * grp + b, i = tt >> LOGW, j = tt & (w - 1);
                        if (i < N) idx |= ((__ldg(Cg + (size_t)i * K + k) >> j) & 1u) << b;
                    }
                }
                tab[e] = tb + (uint32_t)sl * (16 * W) + idx * W;
            }
            if constexpr (T > 0) {
                const uint8_t *Ug = p.U + g * 2 * (size_t)N;
                for (int e = lane; e < NG * T; e += 32) {
                    const int grp = e / T, j = e - grp * T;
                    uint32_t idx = 0;
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        const int tt = 4 * grp + b, i = tt >> LOGW, jj = tt & (w - 1);
                        if (i < N) idx |= ((__ldg(Ug + (size_t)j * N + i) >> jj) & 1u) << b;
                    }
                    tabu[e] = tb + (uint32_t)(grp % kTmGPB) * (16 * W) + idx * W;
                }
            }
            __syncwarp();
        }
        mbar_wait(bar_s + 8 * (uint32_t)(t % kTmRing), (uint32_t)(t / kTmRing) & 1u);   // stage t has landed
        const uint32_t *rs = ring + (size_t)(t % kTmRing) * SPS * SW + W * lane;
        uint32_t hi4[SPG][W];                        // GF(256): x^3 a of the step's source
        (void)hi4;
#pragma unroll
        for (int sl = 0; sl < kTmGPB; sl++) {
            uint32_t e[4][W];
#pragma unroll
            for (int wd = 0; wd < W; wd++) {
                if constexpr (LOGW == 0) {
#pragma unroll
                    for (int b = 0; b < 4; b++) e[b][wd] = rs[(sl * 4 + b) * SW + wd];
                } else if constexpr (LOGW == 1) {
                    const uint32_t a = rs[(sl * 2) * SW + wd], c = rs[(sl * 2 + 1) * SW + wd];
                    e[0][wd] = a; e[1][wd] = tm_xtime<1>(a); e[2][wd] = c; e[3][wd] = tm_xtime<1>(c);
                } else if constexpr (LOGW == 2) {
                    const uint32_t a = rs[sl * SW + wd];
                    e[0][wd] = a; e[1][wd] = tm_xtime<2>(a); e[2][wd] = tm_xtime<2>(e[1][wd]);
                    e[3][wd] = tm_xtime<2>(e[2][wd]);
                } else {
                    const uint32_t a = (sl & 1) ? tm_xtime<3>(hi4[0][wd]) : rs[(sl >> 1) * SW + wd];
                    e[0][wd] = a; e[1][wd] = tm_xtime<3>(a); e[2][wd] = tm_xtime<3>(e[1][wd]);
                    e[3][wd] = tm_xtime<3>(e[2][wd]);
                    if (!(sl & 1)) hi4[0][wd] = e[3][wd];     // x^3 a; x^4 a = x * that
                }
            }
            // combos c = 0 .. 15 at columns c W + wd, stored 32 registers at a time
            // (W = 2: all 16 combos; W = 4: combos 0-7, then 8-15 = e3 ^ those)
            uint32_t v[32];
#pragma unroll
            for (int wd = 0; wd < W; wd++) {
                v[0 * W + wd] = 0u;
                v[1 * W + wd] = e[0][wd];
                v[2 * W + wd] = e[1][wd];
                v[3 * W + wd] = e[0][wd] ^ e[1][wd];
#pragma unroll
                for (int c = 4; c < 8; c++) v[c * W + wd] = e[2][wd] ^ v[(c - 4) * W + wd];
                if constexpr (W == 2) {
#pragma unroll
                    for (int c = 8; c < 16; c++) v[c * W + wd] = e[3][wd] ^ v[(c - 8) * W + wd];
                }
            }
            tm_st32(tb + (uint32_t)sl * (16 * W), v);
            if constexpr (W == 4) {
#pragma unroll
                for (int c = 0; c < 8; c++)
#pragma unroll
                    for (int wd = 0; wd < W; wd++) v[c * W + wd] ^= e[3][wd];
                tm_st32(tb + (uint32_t)sl * (16 * W) + 32, v);
            }
        }
        tm_wait_st();
        const uint4 *ta = reinterpret_cast<const uint4 *>(tab + ((size_t)pass * steps + gs) * (kTmKB * kTmGPB));
        const int kpass = K - pass * kTmKB;          // coded packets of this pass (warp-uniform)
        // one kq step: lookups of coded packets 4 kq .. 4 kq + 3, in two
        // half-batches of 2 coded packets x 4 groups (8 loads in flight per wait)
        auto kstep = [&](auto kqc) {
            constexpr int kq = decltype(kqc)::value;
            uint4 a4[kTmGPB];                       // addresses of k = 4 kq .. 4 kq + 3, per group
#pragma unroll
            for (int sl = 0; sl < kTmGPB; sl++) a4[sl] = ta[kq * kTmGPB + sl];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                uint32_t r[8 * W];                  // [kk][sl][wd]
#pragma unroll
                for (int sl = 0; sl < kTmGPB; sl++) {
                    tm_ldw<W>(h ? a4[sl].z : a4[sl].x, r + (0 * kTmGPB + sl) * W);
                    tm_ldw<W>(h ? a4[sl].w : a4[sl].y, r + (1 * kTmGPB + sl) * W);
                }
                if constexpr (W == 2) tm_wait_ld16(*reinterpret_cast<uint32_t(*)[16]>(r));
                else tm_wait_ld32(*reinterpret_cast<uint32_t(*)[32]>(r));
#pragma unroll
                for (int kk = 0; kk < 2; kk++)
#pragma unroll
                    for (int wd = 0; wd < W; wd++) {
                        uint32_t &y = acc[kq * 4 + 2 * h + kk][wd];
                        const uint32_t x = y ^ r[(kk * kTmGPB + 0) * W + wd] ^ r[(kk * kTmGPB + 1) * W + wd];
                        y = x ^ r[(kk * kTmGPB + 2) * W + wd] ^ r[(kk * kTmGPB + 3) * W + wd];
                    }
            }
        };
        if (kpass >= kTmKB) {
            tm_unroll<kTmKB / 4>([&](auto kqc) { kstep(kqc); });
        } else {                                     // K < 32: no lookups for absent coded packets
            tm_unroll<kTmKB / 4>([&](auto kqc) { if (decltype(kqc)::value * 4 < kpass) kstep(kqc); });
        }
        if constexpr (T > 0) {
            if (gs == 0)
#pragma unroll
                for (int j = 0; j < T; j++) rw[j] = __ldg(p.RB + (g * 2 + j) * (size_t)p.kw + pass);
            if (pass == 0) {                         // A side: u_j's 4-bit index per group, same tables
                uint32_t r[32];                      // kTmGPB T W <= 32
#pragma unroll
                for (int e = 0; e < 32; e++) r[e] = 0u;
                const uint32_t *tu = tabu + (size_t)gs * kTmGPB * T;
#pragma unroll
                for (int e = 0; e < kTmGPB * T; e++) tm_ldw<W>(tu[e], r + W * e);
                tm_wait_ld32(r);
#pragma unroll
                for (int e = 0; e < kTmGPB * T; e++)
#pragma unroll
                    for (int wd = 0; wd < W; wd++) y1[e % T][wd] ^= r[W * e + wd];
            }
        }
        if (gs == steps - 1) {                       // the pass is complete: store and reset
            const uint32_t wi = cc.sp * SW + W * lane;
            uint32_t *Bg = reinterpret_cast<uint32_t *>(p.B) + (g * K + (size_t)pass * kTmKB) * Mw + wi;
            const int kn = K - pass * kTmKB;
            if constexpr (T > 0) {
#pragma unroll
                for (int k = 0; k < kTmKB; k++) {
                    if constexpr (FT)
                        if (pass * kTmKB + k == fk && wi == ((uint32_t)p.fault & 0xFFFFFu & ~(uint32_t)(W - 1))) {
#pragma unroll
                            for (int wd = 0; wd < W; wd++)          // harness: one wrong byte
                                if ((p.fault & (W - 1)) == (uint64_t)wd) acc[k][wd] ^= 0x5Au;
                        }
#pragma unroll
                    for (int j = 0; j < T; j++)
                        if ((rw[j] >> k) & 1u) {
#pragma unroll
                            for (int wd = 0; wd < W; wd++) y2[j][wd] ^= acc[k][wd];
                        }
                }
            }
            if constexpr (tm_tma_store_on(LOGW)) {
                // the pass's 32 coded rows of the span leave through one TMA store:
                // stage them (lane l: words W l ..), make the writes visible to the
                // async proxy, lane 0 issues the store (rows past K and words past
                // M are clipped).  The staging tile is rewritten only after the
                // previous store has read it.
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                __syncwarp();
#pragma unroll
                for (int k = 0; k < kTmKB; k++) {
                    const uint32_t a = stg_s + (uint32_t)(k * SW + W * lane) * 4u;
                    if constexpr (W == 2)
                        asm volatile("st.shared.v2.u32 [%0], {%1,%2};" :: "r"(a), "r"(acc[k][0]), "r"(acc[k][1]) : "memory");
                    else
                        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(acc[k][0]), "r"(acc[k][1]),
                                     "r"(acc[k][2]), "r"(acc[k][3]) : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    tm_tma_store(&tmB, cc.sp * (uint32_t)SW, (uint32_t)(pass * kTmKB), (uint32_t)g, stg_s);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            } else if (wi < Mw) {                    // row k of the pass: one pointer step of Mw words
                uint32_t *q = Bg;
#pragma unroll
                for (int k = 0; k < kTmKB; k++) {
                    if (k < kn) {
                        if constexpr (W == 2)
                            asm volatile("st.global.v2.u32 [%0], {%1,%2};" :: "l"(q), "r"(acc[k][0]), "r"(acc[k][1])
                                         : "memory");
                        else
                            asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(q), "r"(acc[k][0]),
                                         "r"(acc[k][1]), "r"(acc[k][2]), "r"(acc[k][3]) : "memory");
                    }
                    q += Mw;
                }
            }
#pragma unroll
            for (int k = 0; k < kTmKB; k++)
#pragma unroll
                for (int wd = 0; wd < W; wd++) acc[k][wd] = 0u;
            if constexpr (T > 0) {
                if (pass == passes - 1) {            // the unit is complete: compare the projections
#pragma unroll
                    for (int j = 0; j < T; j++) {
#pragma unroll
                        for (int wd = 0; wd < W; wd++) {
                            if (wi < Mw) bad += nz_bytes(y1[j][wd] ^ y2[j][wd]);
                            y1[j][wd] = y2[j][wd] = 0u;
                        }
                    }
                }
            }
        }
        advance(cc);
    }
    if constexpr (T > 0) {
        bad = __reduce_add_sync(0xffffffffu, bad);
        if (lane == 0 && bad && cur_g != ~0ull) atomicAdd(p.mismatch + cur_g, (unsigned long long)bad);
    }
    if constexpr (tm_tma_store_on(LOGW))
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // the last TMA stores
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wid == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(s_tbase), "n"(kCols) : "memory");
}

}  // namespace gfr
