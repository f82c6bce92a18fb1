// gfrlnc.cu -- the C ABI declared in include/gfrlnc.h: argument validation,
// per-field kernel dispatch and launches on the calling thread's stream.
// See the header for the contract of every entry point and DESIGN.md for the
// kernels.  Compiled for sm_100a only.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/gfrlnc.h"
#include "encode_kernels.cuh"
#include "encode_lanek.cuh"
#include "encode_prow.cuh"
#include "encode_prow16.cuh"
#include "encode_stream.cuh"
#include "encode_gf2.cuh"
#include "encode_tmem.cuh"
#include "decode_kernels.cuh"
#include "region_kernels.cuh"
#include "rng_kernels.cuh"
#include "tables.h"

namespace gfr {

constexpr int kMaxDevices = 64;
constexpr int kVersion = 201;   // 0.2.01: TMEM lookup-table engine for GF(2) / GF(4)

__device__ uint32_t g_dev_tabs[4][256 * kTableWords];
__device__ uint8_t g_dev_inv[4][256];
__device__ uint8_t g_dev_mul[4][256 * 256];

static uint32_t g_host_tabs[4][256 * kTableWords];
static uint8_t g_host_inv[4][256];
static uint8_t g_host_mul[4][256 * 256];
static bool g_host_ready[4];
static uint32_t g_dev_ready[kMaxDevices];     // bit f: field index f uploaded and its kernels configured
static int g_sm_count[kMaxDevices];
static uint32_t g_smem_base[kMaxDevices];     // shared-window address of the first dynamic smem byte
static std::mutex g_lock;                     // gf_init and the host pipeline's one-time setup only
static thread_local cudaStream_t tls_stream = nullptr;
static thread_local int tls_path = 0;          // harness: forced encode path (gf_set_encode_path)
static thread_local uint64_t tls_fault = 0;    // harness: gf_set_verify_fault (bit 63 on)

static int field_index(int field)
{
    switch (field) {
    case 2: return 0;
    case 4: return 1;
    case 16: return 2;
    case 256: return 3;
    default: return -1;
    }
}

static int current_device(int *dev)
{
    if (cudaGetDevice(dev) != cudaSuccess || *dev < 0 || *dev >= kMaxDevices) return GF_ECUDA;
    return GF_OK;
}

static int check_ready(int field, int *fi, int *dev)
{
    *fi = field_index(field);
    if (*fi < 0) return GF_EFIELD;
    if (current_device(dev) != GF_OK) return GF_ECUDA;
    if (!(__atomic_load_n(&g_dev_ready[*dev], __ATOMIC_ACQUIRE) >> *fi & 1u)) return GF_ENOINIT;
    return GF_OK;
}

// device addresses of the table symbols, cached per device (cudaGetSymbolAddress
// costs microseconds, which matters for single-generation calls such as C1)
static void *g_sym_cache[3][kMaxDevices];
static int symbol_address(int which, void **out)
{
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    void *v = __atomic_load_n(&g_sym_cache[which][dev], __ATOMIC_ACQUIRE);
    if (!v) {
        const cudaError_t e = which == 0 ? cudaGetSymbolAddress(&v, g_dev_tabs)
                            : which == 1 ? cudaGetSymbolAddress(&v, g_dev_inv)
                                         : cudaGetSymbolAddress(&v, g_dev_mul);
        if (e != cudaSuccess) return GF_ECUDA;
        __atomic_store_n(&g_sym_cache[which][dev], v, __ATOMIC_RELEASE);
    }
    *out = v;
    return GF_OK;
}

static bool overlaps(const void *a, size_t na, const void *b, size_t nb)
{
    const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return na && nb && x < y + nb && y < x + na;
}

static int launch_status()
{
    return cudaGetLastError() == cudaSuccess ? GF_OK : GF_ECUDA;
}

// ---------------------------------------------------------------- regions

template <int OP>
static int launch_region(int dev, uint8_t *dst, const uint8_t *src, size_t bytes,
                         const RegionParams &p, cudaStream_t st)
{
    const size_t nvec = bytes / 16 + 1;
    constexpr int kThreads = 256, kUnroll = 4;
    size_t blocks = (nvec + (size_t)kThreads * kUnroll - 1) / ((size_t)kThreads * kUnroll);
    const size_t cap = (size_t)(g_sm_count[dev] > 0 ? g_sm_count[dev] : 148) * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    int mode = 0;
    if (op_reads_src(OP)) {
        if (src == dst) mode = 2;
        else if (((reinterpret_cast<uintptr_t>(src) - reinterpret_cast<uintptr_t>(dst)) & 15u) != 0)
            mode = 1;
    }
    if (mode == 0)
        region_kernel<OP, 0, kUnroll><<<(unsigned)blocks, kThreads, 0, st>>>(dst, src, bytes, p);
    else if (mode == 1)
        region_kernel<OP, 1, kUnroll><<<(unsigned)blocks, kThreads, 0, st>>>(dst, src, bytes, p);
    else
        region_kernel<OP, 2, kUnroll><<<(unsigned)blocks, kThreads, 0, st>>>(dst, src, bytes, p);
    return launch_status();
}

static RegionParams region_params(int fi, unsigned c)
{
    RegionParams p;
    const uint32_t *t = g_host_tabs[fi] + (size_t)c * kTableWords;
    p.tab.t0lo = t[0]; p.tab.t0hi = t[1]; p.tab.t1lo = t[2]; p.tab.t1hi = t[3]; p.tab.t2 = t[4];
    p.m0 = t[5]; p.m1 = t[6];
    return p;
}

// ---------------------------------------------------------------- encode

static int pow2_at_least(int k)
{
    int t = 1;
    while (t < k) t <<= 1;
    return t;
}

template <int F, int W, int KT, bool BW>
static int launch_encode_t(EncodeParams p, cudaStream_t st)
{
    const size_t spans = (p.Mw + 32u * W - 1) / (32u * W);
    p.spans_per_gen = (int)spans;
    int wpb;
    if (spans <= 8) {
        size_t gpc = 8 / spans;
        if (gpc > p.batch) gpc = p.batch;
        if (gpc < 1) gpc = 1;
        p.gens_per_cta = (int)gpc;
        p.ctas_per_gen = 1;
        wpb = (int)(gpc * spans);
    } else {
        p.gens_per_cta = 1;
        wpb = 8;
        p.ctas_per_gen = (int)((spans + 7) / 8);
    }
    p.k_tiles = (p.K + KT - 1) / KT;
    const size_t gen_groups = (p.batch + p.gens_per_cta - 1) / p.gens_per_cta;
    const size_t grid = (size_t)p.k_tiles * gen_groups * (size_t)p.ctas_per_gen;
    if (grid > 0x7FFFFFFFu) return GF_EARG;
    constexpr int S = enc_stages<F>();
    const size_t smem = (size_t)p.gens_per_cta * enc_table_bytes_per_gen<F, KT>() +
                        (BW ? 0 : (size_t)S * W * wpb * 32 * 4);
    // (the > 48 KiB dynamic shared-memory opt-in was set once by gf_init)
    encode_kernel<F, W, KT, S, BW><<<(unsigned)grid, wpb * 32, smem, st>>>(p);
    return launch_status();
}

template <int F, int W, int KTMAX, bool BW>
static int launch_encode_kt(EncodeParams p, cudaStream_t st)
{
    int kt = pow2_at_least(p.K);
    if (kt > KTMAX) kt = KTMAX;
    switch (kt) {
    case 1: return launch_encode_t<F, W, 1, BW>(p, st);
    case 2: return launch_encode_t<F, W, 2, BW>(p, st);
    case 4: return launch_encode_t<F, W, 4, BW>(p, st);
    case 8: return launch_encode_t<F, W, 8, BW>(p, st);
    case 16: return launch_encode_t<F, W, 16, BW>(p, st);
    default:
        if constexpr (KTMAX >= 32) return launch_encode_t<F, W, 32, BW>(p, st);
        return GF_EARG;
    }
}

template <bool BW>
static int launch_encode_field(int field, EncodeParams p, cudaStream_t st)
{
    switch (field) {
    case 256: return launch_encode_kt<256, 4, 16, BW>(p, st);
    case 16: return launch_encode_kt<16, 4, 16, BW>(p, st);
    // GF(2) / GF(4): 4 words per lane (the table entries of each shared-memory
    // load reused over twice the words) for K <= 8 (GF(2) also K <= 16 on long
    // packets): N = 16, 1500 B, K = 8: GF(2) 2.32 -> 2.87 TB/s, GF(4) 1.57 ->
    // 1.80; GF(2) K = 16 at 16 KiB 1.62 -> 1.85 (at 1500 B it loses 7%);
    // profiles/r01_column_w4_v38.txt
    case 4:
        if (p.K <= 8) return launch_encode_kt<4, 4, 16, BW>(p, st);
        return launch_encode_kt<4, 2, 32, BW>(p, st);
    case 2:
        if (p.K <= 8 || (p.K <= 16 && p.Mw >= 1024)) return launch_encode_kt<2, 4, 16, BW>(p, st);
        return launch_encode_kt<2, 2, 32, BW>(p, st);
    default: return GF_EFIELD;
    }
}

template <int F, int KG, int VT = 0>
static int launch_lanek(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M,
                        size_t batch, cudaStream_t st, const LanekParams *vp = nullptr)
{
    using G = LkGeom<KG, F == 2 && KG == 1>;
    LanekParams p{};
    if (vp) p = *vp;                                           // verification fields (VT > 0)
    p.A = A; p.C = C; p.B = B; p.M = M; p.Mw = (uint32_t)(M / 4); p.batch = batch;
    p.N = N; p.K = K; p.qmask = F - 1;
    p.tiles = (int)((p.Mw + G::TW - 1) / G::TW);
    p.k_tiles = (K + 32 * KG - 1) / (32 * KG);
    const size_t grid = batch * (size_t)p.tiles * (size_t)p.k_tiles;
    if (grid > 0x7FFFFFFFu) return GF_EARG;
    const size_t smem = lk_smem_bytes<F, KG, VT>(N);
    if (smem > 227 * 1024) return GF_EARG;
    if (VT > 0 && (p.fault >> 63))                             // harness fault injection armed
        encode_lanek_kernel<F, KG, VT, true><<<(unsigned)grid, G::THREADS, smem, st>>>(p);
    else
        encode_lanek_kernel<F, KG, VT><<<(unsigned)grid, G::THREADS, smem, st>>>(p);
    return launch_status();
}

// shared-window address of the first dynamic shared-memory byte (the product-
// row kernel places its tables at fixed addresses above it), probed once per device
__global__ void smem_base_probe(uint32_t *out)
{
    extern __shared__ __align__(16) uint8_t dsm[];
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(dsm);
}

// gf_init (once per device): allocate, launch the probe, read it back
static int probe_smem_base(int dev)
{
    uint32_t *d = nullptr;
    if (cudaMalloc(&d, 4) != cudaSuccess) return GF_ECUDA;
    smem_base_probe<<<1, 32, 16>>>(d);
    uint32_t h = 0;
    const bool ok = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    cudaFree(d);
    if (!ok) return GF_ECUDA;
    g_smem_base[dev] = h;
    return GF_OK;
}

template <int F, int KC, int TW = kPrTW>
static int launch_prow(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M,
                       size_t batch, cudaStream_t st)
{
    ProwParams p{};
    p.A = A; p.C = C; p.B = B; p.M = M; p.Mw = (uint32_t)(M / 4);
    p.N = N; p.K = K; p.NS = (N + PrCfg<KC, TW>::S - 1) / PrCfg<KC, TW>::S;
    p.tiles = (int)((p.Mw + TW - 1) / TW);
    p.k_tiles = (K + KC - 1) / KC;
    p.qmask4 = (uint32_t)(F - 1) * 0x01010101u;
    p.cword = (K % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 3u) == 0) ? 1 : 0;
    p.ntiles = batch * (size_t)p.tiles * (size_t)p.k_tiles;
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    const size_t sms = (size_t)(g_sm_count[dev] > 0 ? g_sm_count[dev] : 148);
    const size_t grid = p.ntiles < sms ? p.ntiles : sms;      // persistent: one CTA per SM
    // steps per CTA must fit 32 bits
    if ((p.ntiles + grid - 1) / grid * (size_t)p.NS > 0x7FFFFFF0u) return GF_EARG;
    const uint32_t base = g_smem_base[dev];                   // probed by gf_init (checked <= 0x400 there)
    const size_t smem = kPrSmemEnd - base;
    encode_prow_kernel<F, KC, TW><<<(unsigned)grid, kPrThreads, smem, st>>>(p);
    return launch_status();
}

// GF(16), 64 coded packets per CTA: the nibble-table product-row kernel (encode_prow16.cuh)
static int launch_prow16(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M, size_t batch,
                         cudaStream_t st)
{
    ProwParams p;
    std::memset(&p, 0, sizeof(p));
    p.A = A; p.C = C; p.B = B; p.M = M; p.Mw = (uint32_t)(M / 4);
    p.N = N; p.K = K; p.NS = (N + 3) / 4;
    p.tiles = (int)((p.Mw + kPrTW - 1) / kPrTW);
    p.k_tiles = (K + 63) / 64;
    p.qmask4 = 0x0F0F0F0Fu;
    p.cword = (K % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 3u) == 0) ? 1 : 0;
    p.ntiles = batch * (size_t)p.tiles * (size_t)p.k_tiles;
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    const size_t sms = (size_t)(g_sm_count[dev] > 0 ? g_sm_count[dev] : 148);
    const size_t grid = p.ntiles < sms ? p.ntiles : sms;
    if ((p.ntiles + grid - 1) / grid * (size_t)p.NS > 0x7FFFFFF0u) return GF_EARG;
    const size_t smem = kNbSmemEnd - g_smem_base[dev];
    encode_prow16_kernel<<<(unsigned)grid, kPrThreads, smem, st>>>(p);
    return launch_status();
}

// product-row kernel with 64 (path 6), 32 (path 9) or 16 (path 10) coded packets per CTA
template <int F>
static int launch_prow_kc(int path, const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M,
                          size_t batch, cudaStream_t st)
{
    if (path == 10) return launch_prow<F, 16>(A, C, B, N, K, M, batch, st);
    if (path == 13) return launch_prow<F, 32, 768>(A, C, B, N, K, M, batch, st);
    if (path == 9) return launch_prow<F, 32>(A, C, B, N, K, M, batch, st);
    return launch_prow<F, 64>(A, C, B, N, K, M, batch, st);
}

// layout L: 0 = 16-byte chunks, 1 = 4-byte chunks (latency: few words),
// 2 / 4 / 5 = strided 4- / 8- / 12-word blocks per thread (bulk word-aligned
// packets), 3 = two 16-byte chunks per thread (16-byte-aligned packets >= 1 KiB)
template <class Op, int KT, int L>
static int launch_stream_t(const StreamParams &p, cudaStream_t st)
{
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    const size_t sms = (size_t)(g_sm_count[dev] > 0 ? g_sm_count[dev] : 148);
    size_t grid = (p.total + kStThreads - 1) / kStThreads;
    if (grid > sms * 8) grid = sms * 8;                       // grid-stride: 8 CTAs of 256 per SM
    if constexpr (L == 0) encode_stream_kernel<Op, KT><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else if constexpr (L == 3) encode_stream_wide2_kernel<Op, KT, 2><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else if constexpr (L == 6) encode_stream_wide2_kernel<Op, KT, 4><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else if constexpr (L == 1) encode_stream_words_kernel<Op, KT, 1><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else if constexpr (L == 2) encode_stream_strided_kernel<Op, KT, 4><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else if constexpr (L == 4) encode_stream_strided_kernel<Op, KT, 8><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    else encode_stream_strided_kernel<Op, KT, 12><<<(unsigned)grid, kStThreads, 0, st>>>(p);
    return launch_status();
}

template <class Op, int L>
static int launch_stream_v(const StreamParams &p, cudaStream_t st)
{
    if (p.K == 1) return launch_stream_t<Op, 1, L>(p, st);
    if (p.K == 2) return launch_stream_t<Op, 2, L>(p, st);
    return launch_stream_t<Op, 4, L>(p, st);
}

template <class Op>
static int launch_stream_f(const StreamParams &p, int layout, cudaStream_t st)
{
    if (layout == 0) return launch_stream_v<Op, 0>(p, st);
    if (layout == 1) return launch_stream_v<Op, 1>(p, st);
    if (layout == 2) return launch_stream_v<Op, 2>(p, st);
    if (layout == 4) return launch_stream_v<Op, 4>(p, st);
    if (layout == 5) return launch_stream_v<Op, 5>(p, st);
    if (layout == 6) return launch_stream_v<Op, 6>(p, st);
    return launch_stream_v<Op, 3>(p, st);
}

static int launch_stream(int field, int fi, const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K,
                         size_t M, size_t batch, cudaStream_t st)
{
    StreamParams p;
    void *tabs = nullptr;
    if (symbol_address(0, &tabs) != GF_OK) return GF_ECUDA;
    p.tabs = reinterpret_cast<const uint32_t *>(tabs) + (size_t)fi * 256 * kTableWords;
    // 16-byte chunks when packets are 16-byte aligned; else 4-byte words, one
    // per thread while the job is small (C1: latency) and in strided 4-word
    // blocks per thread in bulk
    const bool wide = M % 16 == 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0 &&
                      (reinterpret_cast<uintptr_t>(B) & 15u) == 0;
    // 16-byte-aligned packets of >= 1 KiB: two chunks per thread (per-source
    // costs halved: NEXT-2 GF(16)/GF(256) +7%, GF(4) +4%); smaller packets
    // would leave most lanes of a 64-chunk block idle
    // harness-only forced layouts (gf_set_encode_path, thread-local): strided
    // word blocks at any job size with W = 4 / 8 / 12, 16-byte chunks two or four
    // per thread at any packet size
    const int force = tls_path;
    const size_t strided_min = (force >= GF_PATH_STREAM_STRIDED4 && force <= GF_PATH_STREAM_STRIDED12) ? 1 : (1u << 20);
    const size_t wide2_min = (force == GF_PATH_STREAM_WIDE2 || force == GF_PATH_STREAM_WIDE4) ? 1 : 64;
    const int strided_wmax_env = force == GF_PATH_STREAM_STRIDED4 ? 4 : force == GF_PATH_STREAM_STRIDED8 ? 8
                               : force == GF_PATH_STREAM_STRIDED12 ? 12 : 0;
    int layout = wide ? (M / 16 >= wide2_min ? 3 : 0) : batch * (M / 4) < strided_min ? 1 : 2;
    // strided: the widest of 12 / 8 / 4 words per thread whose (32 W)-word
    // blocks cover >= 90% of the packet (layouts 5 / 4 / 2); GF(2) / GF(4)
    // stay at 4 (their 8-source batches at W = 12 need 180 registers: 1500 B,
    // N = 16: GF(2) 5.79 -> 4.81 TB/s, while GF(16) 3.74 -> 4.07, GF(256)
    // 3.61 -> 4.03; profiles/r01_stream_strided_w_v34.txt)
    const int strided_wmax = field >= 16 ? 12 : 4;
    int sw = 4;
    if (layout == 2) {
        const size_t mw = M / 4;
        for (int w = 12; w >= 8; w -= 4) {
            const size_t blk = 32u * (size_t)w, nb = (mw + blk - 1) / blk;
            if (w <= strided_wmax && mw * 10 >= nb * blk * 9) { sw = w; break; }
        }
        if (strided_wmax_env == 4 || strided_wmax_env == 8 || strided_wmax_env == 12) sw = strided_wmax_env;   // forced
        layout = sw == 12 ? 5 : sw == 8 ? 4 : 2;
    }
    // 16-byte chunks, GF(16)/GF(256): 4 per thread (128-chunk blocks) when they
    // cover >= 90% of the packet (NEXT-2 GF(256) 4.53 -> 4.70 TB/s, GF(16) 4.78
    // -> 4.85; GF(4) loses 14% at 200 registers; profiles/r01_stream_wide4_v36.txt).
    // (harness: GF_PATH_STREAM_WIDE2 turns it off, GF_PATH_STREAM_WIDE4 forces it)
    // With several coded packets the accumulators multiply: four chunks only for
    // K = 1 (GF(256) K = 2 too), and GF(16) with K >= 3 back to one chunk per
    // thread (N = 16, 4 KiB: GF(16) K = 2 2.22 -> 2.73 TB/s, K = 4 1.19 -> 1.37;
    // GF(256) K = 4 1.21 -> 1.40; profiles/r01_stream_k2to4_v47.txt).
    const int wide4 = force == GF_PATH_STREAM_WIDE2 ? 0 : force == GF_PATH_STREAM_WIDE4 ? 1 : -1;
    if (layout == 3 && wide4 != 0) {
        const size_t m16 = M / 16, nb = (m16 + 127) / 128;
        const bool few_k = K == 1 || (field == 256 && K == 2);
        if (wide4 == 1 || (field >= 16 && few_k && m16 * 10 >= nb * 128 * 9)) layout = 6;
    }
    if (layout == 3 && wide4 != 1 && field == 16 && K >= 3) layout = 0;
    p.A = A; p.C = C; p.B = B; p.N = N; p.K = K;
    p.M16 = wide ? M / 16 : M / 4;
    p.wblocks = layout == 6 ? (p.M16 + 127) / 128 : layout == 3 ? (p.M16 + 63) / 64 : (M / 4 + 32u * sw - 1) / (32u * sw);
    p.total = layout >= 2 ? batch * p.wblocks * 32 : batch * p.M16;
    p.qmask = (uint32_t)field - 1u;
    switch (field) {
    case 2: return launch_stream_f<StreamOp<2>>(p, layout, st);
    case 4: return launch_stream_f<StreamOp<4>>(p, layout, st);
    case 16: return launch_stream_f<StreamOp<16>>(p, layout, st);
    case 256: return launch_stream_f<StreamOp<256>>(p, layout, st);
    default: return GF_EFIELD;
    }
}

template <int F>
static int launch_lanek_kg(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M,
                           size_t batch, cudaStream_t st)
{
    // coded packets per CTA: 32 (3 CTAs/SM), 64 or 128 (one CTA/SM); larger
    // groups share each table build among more lanes
    const int kg = K > 64 ? 4 : K > 32 ? 2 : 1;
    if (kg == 4) return launch_lanek<F, 4>(A, C, B, N, K, M, batch, st);
    if (kg == 2) return launch_lanek<F, 2>(A, C, B, N, K, M, batch, st);
    return launch_lanek<F, 1>(A, C, B, N, K, M, batch, st);
}

// GF(2) split engine (encode_gf2.cuh): all NS source words of a span in
// registers, one generation per block
template <int NS, int T = 0>
static int launch_gf2(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M, size_t batch,
                      cudaStream_t st, const Gf2Params *vp = nullptr)
{
    Gf2Params p{};
    if (vp) p = *vp;                                           // verification fields (T > 0)
    const bool ft = T > 0 && (p.fault >> 63);                  // harness fault injection armed
    p.A = A; p.C = C; p.B = B; p.N = N; p.K = K;
    p.Mw = (uint32_t)(M / 4);
    p.spans = (p.Mw + kG2SpanWords - 1) / kG2SpanWords;
    // spans per warp: 4 for long packets (C5: 1 MiB packets = 2048 spans, 128
    // blocks per generation; 2 - 16 measured within 1%,
    // profiles/r02_gf2_spw.txt), fewer for short ones
    uint32_t spw = p.spans / 512;
    spw = spw < 1 ? 1 : spw > 4 ? 4 : spw;
    p.spw = (int)spw;
    const uint32_t bpg = (p.spans + 4 * spw - 1) / (4 * spw);
    const size_t smem = gf2_smem_bytes(K, NS, T);
    if (smem > 227 * 1024) return GF_EARG;
    for (size_t g0 = 0; g0 < batch; g0 += 65535) {           // grid.y <= 65535 generations per launch
        const unsigned gy = (unsigned)(batch - g0 < 65535 ? batch - g0 : 65535);
        if (ft && N == NS)
            encode_gf2_kernel<NS, true, T, true><<<dim3(bpg, gy), kG2Threads, smem, st>>>(p, (uint32_t)g0);
        else if (ft)
            encode_gf2_kernel<NS, false, T, true><<<dim3(bpg, gy), kG2Threads, smem, st>>>(p, (uint32_t)g0);
        else if (N == NS)
            encode_gf2_kernel<NS, true, T><<<dim3(bpg, gy), kG2Threads, smem, st>>>(p, (uint32_t)g0);
        else
            encode_gf2_kernel<NS, false, T><<<dim3(bpg, gy), kG2Threads, smem, st>>>(p, (uint32_t)g0);
        const int rc = launch_status();
        if (rc != GF_OK) return rc;
    }
    return GF_OK;
}

// TMEM lookup-table engine (encode_tmem.cuh): 4-bit groups of the basis words
// x^j a_i, their 16 XOR-subsets in tensor memory, one lookup per (group, k).
// Warps per CTA: 8 for GF(2) (C5: 2.81 TB/s against 2.69 at 12), 12 for the
// other fields (GF(4) C5: 1.85 TB/s against 1.46 at 16 -- register spills at
// 128 per thread -- and 1.66 at 8; GF(16), N = K = 32: 1.03 against 0.90 at
// 8; tools/exp_tmem.cu, profiles/r02_exp_tmem_v7.txt, r02_exp_tmem_v13.txt);
// tm_wpc2 when the per-warp shared memory (coefficient-address table,
// staging tile, source ring) does not fit.
template <int LOGW>
constexpr int tm_wpc() { return LOGW == 0 ? 8 : 12; }
template <int LOGW>
constexpr int tm_wpc2() { return LOGW == 0 ? 4 : 8; }

static int tm_groups(int logw, int N) { return ((((N << logw) + 3) / 4) + kTmGPB - 1) / kTmGPB * kTmGPB; }

static size_t tm_smem_w(int logw, int N, int K, int wpc, int T = 0)
{
    return (size_t)wpc * tm_warp_bytes(logw, tm_groups(logw, N), (K + kTmKB - 1) / kTmKB, T);
}

static constexpr int log2_field(int field) { return field == 2 ? 0 : field == 4 ? 1 : field == 16 ? 2 : 3; }

// warps per CTA for this shape: the preferred count, tm_wpc2, or 4; 0 if none fits
static int tm_pick_wpc(int logw, int N, int K, int T = 0)
{
    const int w0 = logw == 0 ? tm_wpc<0>() : tm_wpc<1>(), w1 = logw == 0 ? tm_wpc2<0>() : tm_wpc2<1>();
    if (tm_smem_w(logw, N, K, w0, T) <= 226 * 1024) return w0;
    if (tm_smem_w(logw, N, K, w1, T) <= 226 * 1024) return w1;
    if (T == 0 && tm_smem_w(logw, N, K, 4) <= 226 * 1024) return 4;
    return 0;
}

static bool tmem_ok(int field, int N, int K, size_t M, const void *A, const void *B)
{
    return M % 16 == 0 && M / 4 < 0xFFFFFFFFull && N > 0 && K > 0 &&
           ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0 &&
           tm_pick_wpc(log2_field(field), N, K) > 0;
}

template <int LOGW, int WPC, int T = 0, bool FT = false>
static int launch_tmem_w(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M, size_t batch,
                         cudaStream_t st, const TmParams *vp = nullptr)
{
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    // TMA row coordinates are 32-bit signed: at most 2^31 - 1 rows of A per launch
    const size_t gmax = (size_t)0x7FFFFFFF / (size_t)N;
    for (size_t g0 = 0; g0 < batch; g0 += gmax) {
        const size_t nb = batch - g0 < gmax ? batch - g0 : gmax;
        TmParams p{};
        if (vp) {                                              // check fields (T > 0)
            p = *vp;
            p.U = vp->U + g0 * 2 * (size_t)N;
            p.RB = vp->RB + g0 * 2 * (size_t)vp->kw;
            p.mismatch = vp->mismatch + g0;
            const uint64_t fg = (vp->fault >> 32) & 0x7FFFFFFFu;
            p.fault = (fg >= g0 && fg < g0 + nb) ? (vp->fault & 0xFFFFFFFFull) | ((fg - g0) << 32)
                                                 : 0x7FFFFFFFull << 32;           // (no generation matches)
        }
        p.A = A + g0 * N * M; p.C = C + g0 * N * K; p.B = B + g0 * K * M; p.N = N; p.K = K;
        p.Mw = (uint32_t)(M / 4);
        p.spans = (p.Mw + tm_span_words(2) - 1) / tm_span_words(2);
        p.NG = tm_groups(LOGW, N);
        p.passes = (K + kTmKB - 1) / kTmKB;
        p.units = (uint64_t)nb * p.spans;
        const uint64_t warps = (uint64_t)(g_sm_count[dev] > 0 ? g_sm_count[dev] : 148) * WPC;
        p.upw = (p.units + warps - 1) / warps;
        const uint64_t blocks = (p.units + WPC * p.upw - 1) / (WPC * p.upw);
        const size_t smem = tm_smem_w(LOGW, N, K, WPC, T);
        CUtensorMap map;
        CUtensorMap mapb;
        if (!tm_make_map(&map, p.A, (uint64_t)nb * N, M, LOGW) || !tm_make_map_b(&mapb, p.B, nb, K, M))
            return GF_ECUDA;
        encode_tmem_kernel<LOGW, WPC, T, FT><<<(unsigned)blocks, WPC * 32, smem, st>>>(p, map, mapb);
        const int rc = launch_status();
        if (rc != GF_OK) return rc;
    }
    return GF_OK;
}

template <int LOGW>
static int launch_tmem(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M, size_t batch,
                       cudaStream_t st)
{
    constexpr int W0 = tm_wpc<LOGW>(), W1 = tm_wpc2<LOGW>();
    const int wpc = tm_pick_wpc(LOGW, N, K);
    if (wpc == W0) return launch_tmem_w<LOGW, W0>(A, C, B, N, K, M, batch, st);
    if (wpc == W1) return launch_tmem_w<LOGW, W1>(A, C, B, N, K, M, batch, st);
    if constexpr (W1 != 4)
        if (wpc == 4) return launch_tmem_w<LOGW, 4>(A, C, B, N, K, M, batch, st);
    return GF_EARG;
}

// the TMEM engine with the check fused (GF(2) / GF(4) / GF(16), K <= 64): the
// encode's warps per CTA (tm_wpc, tm_wpc2 when the shared memory does not fit)
template <int LOGW, int T>
static int launch_tmem_check(const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K, size_t M, size_t batch,
                             cudaStream_t st, const TmParams *vp)
{
    constexpr int W0 = tm_wpc<LOGW>(), W1 = tm_wpc2<LOGW>();
    const bool ft = (vp->fault >> 63) != 0;
    if (tm_smem_w(LOGW, N, K, W0, T) <= 226 * 1024)
        return ft ? launch_tmem_w<LOGW, W0, T, true>(A, C, B, N, K, M, batch, st, vp)
                  : launch_tmem_w<LOGW, W0, T>(A, C, B, N, K, M, batch, st, vp);
    if (tm_smem_w(LOGW, N, K, W1, T) <= 226 * 1024)
        return ft ? launch_tmem_w<LOGW, W1, T, true>(A, C, B, N, K, M, batch, st, vp)
                  : launch_tmem_w<LOGW, W1, T>(A, C, B, N, K, M, batch, st, vp);
    return GF_EARG;
}

// Harness override of the encode kernel (gf_set_encode_path, thread-local).
// Stream sub-layout codes force the streaming kernel.
static int encode_path_override()
{
    const int t = tls_path;
    return t >= GF_PATH_STREAM_STRIDED4 && t <= GF_PATH_STREAM_WIDE4 ? GF_PATH_STREAM : t;
}

// returned codes (include/gfrlnc.h, gf_encode_path): 0 column (words), 1 column
// (bytes), 2 / 3 lane-k with 32 / 64 (or 128) coded packets per CTA, 6 / 9 / 10
// product-row with 64 / 32 / 16 coded packets per CTA, 8 streaming (K <= 4),
// 11 GF(2) split engine (N <= 32, 16-byte aligned packets, K >= 24; any K when forced),
// 12 GF(16) product-row with nibble-indexed tables (K > 32), 13 GF(256)
// product-row with 32 coded packets per CTA on 768-word tiles (K > 32, long packets),
// 14 TMEM lookup-table engine (GF(2) K >= 9, GF(4) K >= 5, GF(16) K >= 5 but not 13..16 on
// packets >= 8 KiB, N <= 32 when K > 32; packets >= 256 B, M % 16 == 0, 16-byte aligned)
static bool gf2_split_ok(int field, int N, int K, size_t M, const void *A, const void *B)
{
    return field == 2 && N <= 32 && K >= 1 && M % 16 == 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0 &&
           (reinterpret_cast<uintptr_t>(B) & 15u) == 0 && gf2_smem_bytes(K, 32) <= 227 * 1024;
}

static int encode_path(int field, int N, int K, size_t M, const void *A, const void *B, bool tmem = true)
{
    const bool aligned = M % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 3u) == 0 &&
                         (reinterpret_cast<uintptr_t>(B) & 3u) == 0 && M / 4 < 0xFFFFFFFFull;
    const int ov = encode_path_override();
    if (!aligned) return 1;
    if (K <= 4 && (ov == GF_PATH_STREAM || ov == 0)) return 8;  // streaming (16- or 4-byte chunks)
    // The TMEM lookup-table engine on 16-byte aligned packets of >= 256 bytes:
    // GF(2) with K >= 9 and GF(4) with K >= 5 (C5: GF(2) 2.29 -> 2.9 TB/s
    // against the split engine, GF(4) 1.13 -> 2.06 against lane-k; K = 5-20:
    // 1.3-2.4x the column / product-row kernels; GF(2) K <= 8: the column
    // kernel is 0-10% faster; profiles/r02_exp_tmem_route_v6.txt), GF(16) with K >= 5 and N <= 32 for
    // K > 32 (1.1-3x the column / product-row kernels), except 13 <= K <= 16 on
    // packets >= 8 KiB where the 16-packet product-row kernel is 5-14% faster
    // (profiles/r02_exp_tmem_route_v5.txt).  Forced: any field and shape it takes.
    if (tmem && ov == GF_PATH_TMEM && tmem_ok(field, N, K, M, A, B)) return 14;
    const bool tm_gf16 = field == 16 && K >= 5 && (K <= 32 || N <= 32) && !(K >= 13 && K <= 16 && M >= 8192);
    if (tmem && ov == 0 && M >= 256 && ((field == 2 && K >= 9) || (field == 4 && K >= 5) || tm_gf16) &&
        tmem_ok(field, N, K, M, A, B))
        return 14;
    // GF(2): the split engine (encode_gf2.cuh) where the lane-k kernel ran
    // before, K >= 24 (C5 N = K = 32, 1 MiB: 2.21 vs 1.66 TB/s)
    if (ov == GF_PATH_GF2 && gf2_split_ok(field, N, K, M, A, B)) return 11;
    if (ov == 0 && K >= 24 && gf2_split_ok(field, N, K, M, A, B)) return 11;
    // GF(4), 9 <= K < 24: product rows beat the column kernel when the 384-word
    // tiles cover the packet well (>= 85%) and either K > 16 (where the column
    // kernel halves) or packets are >= 4 KiB (profiles/r01_gf4_prow_routing.txt)
    const size_t mw = M / 4, tiles = (mw + 383) / 384;
    const bool gf4_prow = field == 4 && K > 8 && K < 24 && mw * 100 >= tiles * 384 * 85 && (K > 16 || M >= 4096);
    if (ov == GF_PATH_COLUMN || (ov == 0 && K < 24 && !(field >= 16 && K > 8) && !gf4_prow)) return 0;
    const int kg2 = K > 32 ? 1 : 0;      // (K > 64 uses 128 coded packets per CTA)
    // product rows for GF(16)/GF(256) from K = 9 on (measured: tools/exp_shapes.py),
    // with 16, 32 or 64 coded packets per CTA so that few lanes idle
    // (GF(16) with 64 coded packets per CTA: the nibble-table kernel, path 12;
    // GF(256), K > 32, long packets whose 768-word tiles cover >= 90%: 32 coded
    // packets per CTA on 768-word tiles, half the table-build share, path 13:
    // C4 112.9 -> 115.8 GB/s, profiles/r02_c4_768.txt)
    const size_t tiles768 = (mw + 767) / 768;
    const bool long768 = field == 256 && K > 32 && mw >= 8 * 768 && mw * 10 >= tiles768 * 768 * 9;
    const int prow = K <= 16 ? 10 : K <= 32 ? 9 : field == 16 ? 12 : long768 ? 13 : 6;
    if (ov == GF_PATH_PROW || (ov == 0 && ((field >= 16 && K > 8) || gf4_prow))) return prow;
    return 2 + kg2;
}

static int encode_on_stream(int field, int fi, const uint8_t *A, const uint8_t *C, uint8_t *B,
                            int N, int K, size_t M, size_t batch, cudaStream_t st)
{
    {
        const int path = encode_path(field, N, K, M, A, B);
        if (path == 8) return launch_stream(field, fi, A, C, B, N, K, M, batch, st);
        if (path == 12) return launch_prow16(A, C, B, N, K, M, batch, st);
        if (path == 14) {
            switch (field) {
            case 2: return launch_tmem<0>(A, C, B, N, K, M, batch, st);
            case 4: return launch_tmem<1>(A, C, B, N, K, M, batch, st);
            case 16: return launch_tmem<2>(A, C, B, N, K, M, batch, st);
            default: return launch_tmem<3>(A, C, B, N, K, M, batch, st);
            }
        }
        if (path == 11) return N <= 16 ? launch_gf2<16>(A, C, B, N, K, M, batch, st)
                                       : launch_gf2<32>(A, C, B, N, K, M, batch, st);
        if (path == 6 || path == 9 || path == 10 || path == 13) {
            switch (field) {
            case 256: return launch_prow_kc<256>(path, A, C, B, N, K, M, batch, st);
            case 16: return launch_prow_kc<16>(path, A, C, B, N, K, M, batch, st);
            case 4: return launch_prow_kc<4>(path, A, C, B, N, K, M, batch, st);
            case 2: return launch_prow_kc<2>(path, A, C, B, N, K, M, batch, st);
            default: return GF_EFIELD;
            }
        }
        if (path >= 2) {
            switch (field) {
            case 256: return launch_lanek_kg<256>(A, C, B, N, K, M, batch, st);
            case 16: return launch_lanek_kg<16>(A, C, B, N, K, M, batch, st);
            case 4: return launch_lanek_kg<4>(A, C, B, N, K, M, batch, st);
            case 2: return launch_lanek_kg<2>(A, C, B, N, K, M, batch, st);
            default: return GF_EFIELD;
            }
        }
    }
    EncodeParams p;
    std::memset(&p, 0, sizeof(p));
    p.A = A; p.C = C; p.B = B;
    void *tabs = nullptr;
    if (symbol_address(0, &tabs) != GF_OK) return GF_ECUDA;
    p.tabs = reinterpret_cast<const uint32_t *>(tabs) + (size_t)fi * 256 * kTableWords;
    p.M = M; p.batch = batch; p.N = N; p.K = K; p.qmask = field - 1;
    const bool bytewise = (M % 4) != 0 || (reinterpret_cast<uintptr_t>(A) & 3u) ||
                          (reinterpret_cast<uintptr_t>(B) & 3u);
    p.Mw = bytewise ? M : M / 4;
    return bytewise ? launch_encode_field<true>(field, p, st) : launch_encode_field<false>(field, p, st);
}

static int validate_encode(int field, const uint8_t *A, const uint8_t *C, const uint8_t *B,
                           int N, int K, size_t M, size_t batch, size_t *a_bytes, size_t *b_bytes,
                           size_t *c_bytes)
{
    if (field_index(field) < 0) return GF_EFIELD;
    if (N < 1 || K < 1) return GF_EARG;
    size_t nm, km;
    if (__builtin_mul_overflow((size_t)N, M, &nm) || __builtin_mul_overflow(nm, batch, a_bytes) ||
        __builtin_mul_overflow((size_t)K, M, &km) || __builtin_mul_overflow(km, batch, b_bytes) ||
        __builtin_mul_overflow((size_t)N * (size_t)K, batch, c_bytes) || *a_bytes > (SIZE_MAX >> 1) ||
        *b_bytes > (SIZE_MAX >> 1))
        return GF_EARG;
    if (M == 0 || batch == 0) return GF_OK;
    if (!A || !C || !B) return GF_EARG;
    if (overlaps(B, *b_bytes, A, *a_bytes) || overlaps(B, *b_bytes, C, *c_bytes)) return GF_EOVERLAP;
    return GF_OK;
}

// ------------------------------------------------------------ host pipeline

constexpr int kPipeBufs = 3;     // chunks in flight: H2D(j+2) | kernel(j+1) | D2H(j)

struct HostPipe {
    bool ready = false;
    cudaStream_t s_h2d = nullptr, s_cmp = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_entry = nullptr;                 // the caller's stream at entry (workspace handed over)
    cudaEvent_t ev_in[kPipeBufs], ev_cmp[kPipeBufs], ev_free[kPipeBufs];
};
static HostPipe g_pipes[kMaxDevices];

static int pipe_for(int dev, HostPipe **out)
{
    HostPipe &P = g_pipes[dev];
    if (__atomic_load_n(&P.ready, __ATOMIC_ACQUIRE)) {
        *out = &P;
        return GF_OK;
    }
    std::lock_guard<std::mutex> g(g_lock);
    if (!P.ready) {
        if (cudaStreamCreateWithFlags(&P.s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&P.s_cmp, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&P.s_d2h, cudaStreamNonBlocking) != cudaSuccess)
            return GF_ECUDA;
        for (int b = 0; b < kPipeBufs; b++)
            if (cudaEventCreateWithFlags(&P.ev_in[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&P.ev_cmp[b], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&P.ev_free[b], cudaEventDisableTiming) != cudaSuccess)
                return GF_ECUDA;
        if (cudaEventCreateWithFlags(&P.ev_entry, cudaEventDisableTiming) != cudaSuccess) return GF_ECUDA;
        __atomic_store_n(&P.ready, true, __ATOMIC_RELEASE);
    }
    *out = &P;
    return GF_OK;
}


// harness fault injection for the unfused verify path: one wrong byte of B
__global__ void fault_byte_kernel(uint8_t *b) { *b ^= 0x5Au; }

// ------------------------------------------------------- one-time kernel setup
// Everything a launch needs besides its arguments is prepared here, once per
// (device, field), by gf_init: the dynamic shared-memory opt-in of every kernel
// instantiation the router can pick (so no launch calls cudaFuncSetAttribute)
// and, per device, the product-row kernel's shared-window probe.

template <class Kern>
static int allow_smem(Kern *k, int bytes)
{
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k) != cudaSuccess) return GF_ECUDA;
    // static + dynamic shared memory must fit the per-block opt-in maximum
    int cap = bytes - (int)fa.sharedSizeBytes;
    if (cap < 0) cap = 0;
    return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) == cudaSuccess ? GF_OK
                                                                                                     : GF_ECUDA;
}

template <int F, int W, int KT>
static int configure_column_t(int optin)
{
    constexpr int S = enc_stages<F>();
    int rc = allow_smem(encode_kernel<F, W, KT, S, false>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_kernel<F, W, KT, S, true>, optin);
    return rc;
}

template <int F, int W, int KTMAX>
static int configure_column(int optin)
{
    int rc = GF_OK;
    if (rc == GF_OK) rc = configure_column_t<F, W, 1>(optin);
    if (rc == GF_OK) rc = configure_column_t<F, W, 2>(optin);
    if (rc == GF_OK) rc = configure_column_t<F, W, 4>(optin);
    if (rc == GF_OK) rc = configure_column_t<F, W, 8>(optin);
    if (rc == GF_OK) rc = configure_column_t<F, W, 16>(optin);
    if constexpr (KTMAX >= 32)
        if (rc == GF_OK) rc = configure_column_t<F, W, 32>(optin);
    return rc;
}

template <int F>
static int configure_field(int optin, uint32_t smem_base)
{
    int rc = GF_OK;
    if constexpr (F >= 16) {
        rc = configure_column<F, 4, 16>(optin);
    } else {
        rc = configure_column<F, 4, 16>(optin);
        if (rc == GF_OK) rc = configure_column<F, 2, 32>(optin);
    }
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 1>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 2>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 4>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 1, 1>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 1, 2>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 2, 1>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 2, 2>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 1, 1, true>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 1, 2, true>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 2, 1, true>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_lanek_kernel<F, 2, 2, true>, optin);
    const int prow = (int)(kPrSmemEnd - smem_base);
    if (rc == GF_OK) rc = allow_smem(encode_prow_kernel<F, 16>, prow);
    if (rc == GF_OK) rc = allow_smem(encode_prow_kernel<F, 32>, prow);
    if (rc == GF_OK) rc = allow_smem(encode_prow_kernel<F, 64>, prow);
    if (rc == GF_OK) rc = allow_smem(encode_prow_kernel<F, 32, 768>, prow);
    if constexpr (F == 16)
        if (rc == GF_OK) rc = allow_smem(encode_prow16_kernel, (int)(kNbSmemEnd - smem_base));
    if constexpr (F == 2) {
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, false>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, false>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, true, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, false, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, true, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, false, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, true, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, false, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, true, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, false, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, true, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, false, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, true, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, false, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, true, 2, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<16, false, 2, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, true, 2, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_gf2_kernel<32, false, 2, true>, optin);
    }
    if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<log2_field(F), tm_wpc<log2_field(F)>()>, optin);
    if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<log2_field(F), tm_wpc2<log2_field(F)>()>, optin);
    if constexpr (tm_wpc2<log2_field(F)>() != 4)
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<log2_field(F), 4>, optin);
    if constexpr (F <= 16) {
        constexpr int L = log2_field(F), W0 = tm_wpc<L>(), W1 = tm_wpc2<L>();
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W0, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W0, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W0, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W0, 2, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W1, 1>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W1, 2>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W1, 1, true>, optin);
        if (rc == GF_OK) rc = allow_smem(encode_tmem_kernel<L, W1, 2, true>, optin);
    }
    if (rc == GF_OK) rc = allow_smem(invert_warp_kernel, optin);
    if (rc == GF_OK) rc = allow_smem(invert_kernel, optin);
    return rc;
}

static int configure_kernels(int field, int dev)
{
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
        return GF_ECUDA;
    const uint32_t base = g_smem_base[dev];
    switch (field) {
    case 2: return configure_field<2>(optin, base);
    case 4: return configure_field<4>(optin, base);
    case 16: return configure_field<16>(optin, base);
    case 256: return configure_field<256>(optin, base);
    default: return GF_EFIELD;
    }
}

}  // namespace gfr

using namespace gfr;

extern "C" {

int gf_version(void) { return kVersion; }

int gf_encode_path(int field, int N, int K, size_t M, size_t a_align, size_t b_align)
{
    if (field_index(field) < 0) return GF_EFIELD;
    if (N < 1 || K < 1) return GF_EARG;
    return encode_path(field, N, K, M, reinterpret_cast<const void *>(a_align & 15u),
                       reinterpret_cast<const void *>(b_align & 15u));
}

const char *gf_strerror(int status)
{
    switch (status) {
    case GF_OK: return "ok";
    case GF_EFIELD: return "unsupported field (expected 2, 4, 16 or 256)";
    case GF_ECOEFF: return "coefficient >= field size";
    case GF_EARG: return "invalid argument (NULL pointer, N/K < 1, size overflow or workspace too small)";
    case GF_EOVERLAP: return "overlapping buffers";
    case GF_ENOINIT: return "gf_init(field) not called on the current device";
    case GF_ECUDA: return "CUDA launch or runtime failure";
    default: return "unknown status";
    }
}

int gf_set_encode_path(int path)
{
    if (path < 0 || path > GF_PATH_TMEM || path == 3 || path == 5) return GF_EARG;
    tls_path = path;
    return GF_OK;
}

int gf_set_stream(void *cuda_stream)
{
    tls_stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    return GF_OK;
}

int gf_host_tables(int field, uint32_t *out, size_t cap_words)
{
    if (field_index(field) < 0) return GF_EFIELD;
    if (!out) return GF_EARG;
    const int rc = build_tables(field, out, cap_words);
    return rc == 0 ? GF_OK : (rc == -1 ? GF_EFIELD : GF_EARG);
}

int gf_init(int field)
{
    const int fi = field_index(field);
    if (fi < 0) return GF_EFIELD;
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    std::lock_guard<std::mutex> g(g_lock);
    if (!g_host_ready[fi]) {
        std::memset(g_host_tabs[fi], 0, sizeof(g_host_tabs[fi]));
        if (build_tables(field, g_host_tabs[fi], 256 * kTableWords) != 0) return GF_EFIELD;
        if (build_inverses(field, g_host_inv[fi]) != 0) return GF_EFIELD;
        if (build_products(field, g_host_mul[fi]) != 0) return GF_EFIELD;
        g_host_ready[fi] = true;
    }
    if (!(g_dev_ready[dev] >> fi & 1u)) {
        if (cudaMemcpyToSymbol(g_dev_tabs, g_host_tabs[fi], sizeof(g_host_tabs[fi]),
                               (size_t)fi * sizeof(g_host_tabs[fi]), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpyToSymbol(g_dev_inv, g_host_inv[fi], 256, (size_t)fi * 256, cudaMemcpyHostToDevice) !=
                cudaSuccess ||
            cudaMemcpyToSymbol(g_dev_mul, g_host_mul[fi], 65536, (size_t)fi * 65536, cudaMemcpyHostToDevice) !=
                cudaSuccess)
            return GF_ECUDA;
        if (g_sm_count[dev] == 0) {
            int sms = 0;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
                return GF_ECUDA;
            // the product-row kernel's tables sit at fixed shared-window addresses
            // above the dynamic window's base, which must start at <= 0x400
            if (probe_smem_base(dev) != GF_OK || g_smem_base[dev] > kPrBar) return GF_ECUDA;
            g_sm_count[dev] = sms;
        }
        if (configure_kernels(field, dev) != GF_OK) return GF_ECUDA;
        if (!tm_resolve_encoder()) return GF_ECUDA;   // the TMEM engine's tensor-map encoder
        void *sym;                               // cache the table addresses (no symbol lookups at launch)
        if (symbol_address(0, &sym) != GF_OK || symbol_address(1, &sym) != GF_OK ||
            symbol_address(2, &sym) != GF_OK)
            return GF_ECUDA;
        __atomic_or_fetch(&g_dev_ready[dev], 1u << fi, __ATOMIC_RELEASE);
    }
    return GF_OK;
}

int gf_maddrc(int field, uint8_t *dst, const uint8_t *src, uint8_t coeff, size_t bytes)
{
    int fi, dev;
    const int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    if (coeff >= (unsigned)field) return GF_ECOEFF;
    if (bytes == 0) return GF_OK;
    if (!dst || !src || bytes > (SIZE_MAX >> 1)) return GF_EARG;
    if (dst != src && overlaps(dst, bytes, src, bytes)) return GF_EOVERLAP;
    if (coeff == 0) return GF_OK;                            // Alg. 1: c == 0 returns
    const cudaStream_t st = tls_stream;
    const RegionParams p = region_params(fi, coeff);
    if (coeff == 1) return launch_region<OP_XOR>(dev, dst, src, bytes, p, st);   // xorr
    if (field == 4) return launch_region<OP_MADD_GF4>(dev, dst, src, bytes, p, st);
    return launch_region<OP_MADD_PRMT>(dev, dst, src, bytes, p, st);
}

int gf_mulrc(int field, uint8_t *dst, uint8_t coeff, size_t bytes)
{
    int fi, dev;
    const int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    if (coeff >= (unsigned)field) return GF_ECOEFF;
    if (bytes == 0) return GF_OK;
    if (!dst || bytes > (SIZE_MAX >> 1)) return GF_EARG;
    if (coeff == 1) return GF_OK;
    const cudaStream_t st = tls_stream;
    const RegionParams p = region_params(fi, coeff);
    if (coeff == 0) return launch_region<OP_ZERO>(dev, dst, nullptr, bytes, p, st);
    if (field == 4) return launch_region<OP_MUL_GF4>(dev, dst, nullptr, bytes, p, st);
    return launch_region<OP_MUL_PRMT>(dev, dst, nullptr, bytes, p, st);
}

int gf_encode_batch(int field, const uint8_t *A, const uint8_t *C, uint8_t *B, int N, int K,
                    size_t M, size_t batch)
{
    int fi, dev;
    int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    size_t ab, bb, cb;
    rc = validate_encode(field, A, C, B, N, K, M, batch, &ab, &bb, &cb);
    if (rc != GF_OK || M == 0 || batch == 0) return rc;
    return encode_on_stream(field, fi, A, C, B, N, K, M, batch, tls_stream);
}

int gf_encode_batch_host(int field, const uint8_t *A_host, const uint8_t *C_host, uint8_t *B_host,
                         int N, int K, size_t M, size_t batch, void *dev_ws, size_t ws_bytes)
{
    int fi, dev;
    int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    size_t ab, bb, cb;
    rc = validate_encode(field, A_host, C_host, B_host, N, K, M, batch, &ab, &bb, &cb);
    if (rc != GF_OK || M == 0 || batch == 0) return rc;
    if (!dev_ws) return GF_EARG;
    const size_t per_gen_a = (size_t)N * M, per_gen_c = (size_t)N * K, per_gen_b = (size_t)K * M;
    // keep every chunk 16-B aligned inside the workspace
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t chunk = ws_bytes / (kPipeBufs * (per_gen_a + per_gen_c + per_gen_b) + 144);
    if (chunk < 1) return GF_EARG;
    if (chunk > batch) chunk = batch;
    HostPipe *P;
    if ((rc = pipe_for(dev, &P)) != GF_OK) return rc;
    uint8_t *ws = static_cast<uint8_t *>(dev_ws);
    uint8_t *bufA[kPipeBufs], *bufC[kPipeBufs], *bufB[kPipeBufs];
    size_t off = 0;
    for (int b = 0; b < kPipeBufs; b++) {
        bufA[b] = ws + off; off = al(off + chunk * per_gen_a);
        bufC[b] = ws + off; off = al(off + chunk * per_gen_c);
        bufB[b] = ws + off; off = al(off + chunk * per_gen_b);
    }
    if (off > ws_bytes) return GF_EARG;
    // the workspace may still be in use by work queued on the caller's stream
    // (e.g. a stream-ordered allocator just handed it out): the pipeline's
    // first copy waits for everything queued there so far
    if (cudaEventRecord(P->ev_entry, tls_stream) != cudaSuccess ||
        cudaStreamWaitEvent(P->s_h2d, P->ev_entry, 0) != cudaSuccess)
        return GF_ECUDA;
    // on any failure after the first enqueue, drain all three streams before
    // returning, so no copy touches the caller's buffers after the call
    auto fail = [&](int code) {
        cudaStreamSynchronize(P->s_h2d);
        cudaStreamSynchronize(P->s_cmp);
        cudaStreamSynchronize(P->s_d2h);
        return code;
    };
    const size_t nchunks = (batch + chunk - 1) / chunk;
    for (size_t j = 0; j < nchunks; j++) {
        const int b = (int)(j % kPipeBufs);
        const size_t g0 = j * chunk, gn = (g0 + chunk <= batch) ? chunk : batch - g0;
        if (j >= kPipeBufs && cudaStreamWaitEvent(P->s_h2d, P->ev_free[b], 0) != cudaSuccess) return fail(GF_ECUDA);
        if (cudaMemcpyAsync(bufA[b], A_host + g0 * per_gen_a, gn * per_gen_a, cudaMemcpyHostToDevice,
                            P->s_h2d) != cudaSuccess ||
            cudaMemcpyAsync(bufC[b], C_host + g0 * per_gen_c, gn * per_gen_c, cudaMemcpyHostToDevice,
                            P->s_h2d) != cudaSuccess ||
            cudaEventRecord(P->ev_in[b], P->s_h2d) != cudaSuccess)
            return fail(GF_ECUDA);
        if (cudaStreamWaitEvent(P->s_cmp, P->ev_in[b], 0) != cudaSuccess) return fail(GF_ECUDA);
        if (j >= kPipeBufs && cudaStreamWaitEvent(P->s_cmp, P->ev_free[b], 0) != cudaSuccess) return fail(GF_ECUDA);
        if ((rc = encode_on_stream(field, fi, bufA[b], bufC[b], bufB[b], N, K, M, gn, P->s_cmp)) != GF_OK)
            return fail(rc);
        if (cudaEventRecord(P->ev_cmp[b], P->s_cmp) != cudaSuccess ||
            cudaStreamWaitEvent(P->s_d2h, P->ev_cmp[b], 0) != cudaSuccess ||
            cudaMemcpyAsync(B_host + g0 * per_gen_b, bufB[b], gn * per_gen_b, cudaMemcpyDeviceToHost,
                            P->s_d2h) != cudaSuccess ||
            cudaEventRecord(P->ev_free[b], P->s_d2h) != cudaSuccess)
            return fail(GF_ECUDA);
    }
    if (cudaStreamSynchronize(P->s_d2h) != cudaSuccess) return fail(GF_ECUDA);
    return GF_OK;
}

int gf_invert_batch(int field, const uint8_t *C, uint8_t *D, int *rank, int N, size_t batch)
{
    int fi, dev;
    const int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    if (N < 1 || N > 256) return GF_EARG;
    if (batch == 0) return GF_OK;
    if (!C || !D) return GF_EARG;
    size_t cb;
    if (__builtin_mul_overflow((size_t)N * (size_t)N, batch, &cb) || batch > 0x7FFFFFFFu) return GF_EARG;
    if (overlaps(C, cb, D, cb)) return GF_EOVERLAP;
    void *tabs = nullptr, *inv = nullptr;
    if (symbol_address(0, &tabs) != GF_OK || symbol_address(1, &inv) != GF_OK)
        return GF_ECUDA;
    InvertParams p;
    p.C = C; p.D = D; p.rank = rank; p.batch = batch; p.N = N; p.qmask = field - 1;
    p.tabs = reinterpret_cast<const uint32_t *>(tabs) + (size_t)fi * 256 * kTableWords;
    p.inv = reinterpret_cast<const uint8_t *>(inv) + (size_t)fi * 256;
    const size_t rw = (2 * (size_t)N + 3) / 4;
    if (field == 2 && N <= 64) {                              // bit-sliced, warp per matrix
        invert_gf2_kernel<<<(unsigned)((batch + kInvG2Warps - 1) / kInvG2Warps), 32 * kInvG2Warps, 0,
                            tls_stream>>>(p);
        return launch_status();
    }
    if (N <= 64) {                                            // warp per matrix (no CTA barriers)
        const size_t smem_w = (256 * 5 + 64 + kInvWarps * 32 * 4) * 4 + (size_t)kInvWarps * N * (rw + 1) * 4;
        invert_warp_kernel<<<(unsigned)((batch + kInvWarps - 1) / kInvWarps), 32 * kInvWarps, smem_w,
                             tls_stream>>>(p);
        return launch_status();
    }
    const size_t smem = (size_t)N * rw * 4 + 256 * 8 * 4 + 256;
    invert_kernel<<<(unsigned)batch, 256, smem, tls_stream>>>(p);
    return launch_status();
}

int gf_decode_batch(int field, const uint8_t *B, const uint8_t *C, uint8_t *A, int *rank, int N, size_t M,
                    size_t batch, void *dev_ws, size_t ws_bytes)
{
    int fi, dev;
    int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    size_t ab, bb, cb;
    rc = validate_encode(field, B, C, A, N, N, M, batch, &bb, &ab, &cb);
    if (rc != GF_OK || M == 0 || batch == 0) return rc;
    if (!dev_ws || ws_bytes < cb) return GF_EARG;
    uint8_t *D = static_cast<uint8_t *>(dev_ws);
    if (overlaps(D, cb, A, ab) || overlaps(D, cb, B, bb) || overlaps(D, cb, C, cb)) return GF_EOVERLAP;
    if ((rc = gf_invert_batch(field, C, D, rank, N, batch)) != GF_OK) return rc;
    return encode_on_stream(field, fi, B, D, A, N, N, M, batch, tls_stream);
}

int gf_verify_batch(int field, const uint8_t *A, const uint8_t *C, const uint8_t *B, const uint8_t *R, int t,
                    int N, int K, size_t M, size_t batch, unsigned long long *mismatch, void *dev_ws,
                    size_t ws_bytes)
{
    int fi, dev;
    int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    size_t ab, bb, cb;
    rc = validate_encode(field, A, C, B, N, K, M, batch, &ab, &bb, &cb);
    if (rc != GF_OK || M == 0 || batch == 0) return rc;
    if (t < 1 || t > 32 || !R || !mismatch || !dev_ws) return GF_EARG;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t u_bytes = al(batch * (size_t)N * t), y_bytes = al(batch * (size_t)t * M);
    if (ws_bytes < u_bytes + 2 * y_bytes) return GF_EARG;
    uint8_t *U = static_cast<uint8_t *>(dev_ws), *Y1 = U + u_bytes, *Y2 = Y1 + y_bytes;
    void *mul = nullptr;
    if (symbol_address(2, &mul) != GF_OK) return GF_ECUDA;
    const cudaStream_t st = tls_stream;
    const size_t nu = batch * (size_t)N * t;
    project_coeffs_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, st>>>(
        C, R, U, reinterpret_cast<const uint8_t *>(mul) + (size_t)fi * 65536, N, K, t, batch, field - 1);
    if ((rc = launch_status()) != GF_OK) return rc;
    if ((rc = encode_on_stream(field, fi, A, U, Y1, N, t, M, batch, st)) != GF_OK) return rc;   // sum_i u_i a_i
    if ((rc = encode_on_stream(field, fi, B, R, Y2, K, t, M, batch, st)) != GF_OK) return rc;   // sum_k r_k b_k
    if (cudaMemsetAsync(mismatch, 0, batch * sizeof(unsigned long long), st) != cudaSuccess) return GF_ECUDA;
    const size_t len = (size_t)t * M;
    unsigned gx = (unsigned)((len + 255) / 256);
    if (gx > 64) gx = 64;
    if (batch > 65535) {
        for (size_t g0 = 0; g0 < batch; g0 += 65535) {
            const size_t gn = batch - g0 < 65535 ? batch - g0 : 65535;
            count_mismatch_kernel<<<dim3(gx, (unsigned)gn), 256, 0, st>>>(Y1 + g0 * len, Y2 + g0 * len, len,
                                                                         mismatch + g0);
        }
    } else {
        count_mismatch_kernel<<<dim3(gx, (unsigned)batch), 256, 0, st>>>(Y1, Y2, len, mismatch);
    }
    return launch_status();
}

int gf_set_verify_fault(int enable, size_t g, int k, size_t word)
{
    if (!enable) {
        tls_fault = 0;
        return GF_OK;
    }
    if (k < 0 || k > 0xFFF || word > 0xFFFFF || g > 0x7FFFFFFF) return GF_EARG;
    tls_fault = (1ull << 63) | ((uint64_t)g << 32) | ((uint64_t)k << 20) | (uint64_t)word;
    return GF_OK;
}

int gf_encode_verify_batch(int field, const uint8_t *A, const uint8_t *C, uint8_t *B, const uint8_t *R, int t,
                           int N, int K, size_t M, size_t batch, unsigned long long *mismatch, void *dev_ws,
                           size_t ws_bytes)
{
    int fi, dev;
    int rc = check_ready(field, &fi, &dev);
    if (rc != GF_OK) return rc;
    size_t ab, bb, cb;
    rc = validate_encode(field, A, C, B, N, K, M, batch, &ab, &bb, &cb);
    if (rc != GF_OK || M == 0 || batch == 0) return rc;
    if (t < 1 || t > 2 || !R || !mismatch || !dev_ws || (reinterpret_cast<uintptr_t>(dev_ws) & 15u)) return GF_EARG;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const int kblocks = (K + 63) / 64, kw = (K + 31) / 32;
    const size_t u_bytes = al(batch * (size_t)kblocks * 2 * N), rb_bytes = batch * 2 * (size_t)kw * 4;
    if (ws_bytes < u_bytes + rb_bytes) return GF_EARG;
    uint8_t *U = static_cast<uint8_t *>(dev_ws);
    uint32_t *RB = reinterpret_cast<uint32_t *>(U + u_bytes);
    if (overlaps(U, u_bytes + rb_bytes, A, ab) || overlaps(U, u_bytes + rb_bytes, B, bb) ||
        overlaps(U, u_bytes + rb_bytes, C, cb))
        return GF_EOVERLAP;
    const cudaStream_t st = tls_stream;
    if (cudaMemsetAsync(mismatch, 0, batch * sizeof(unsigned long long), st) != cudaSuccess) return GF_ECUDA;
    if (batch > 0x7FFFFFFFu || 8 * (size_t)kw > 48 * 1024) return GF_EARG;
    verify_prep_kernel<<<(unsigned)batch, 128, 8 * (size_t)kw, st>>>(C, R, U, RB, N, K, t, kblocks, kw, batch,
                                                                      field - 1);
    if ((rc = launch_status()) != GF_OK) return rc;
    const int path = encode_path(field, N, K, M, A, B);
    if (path == 14 && field <= 16 && K <= 64 && tm_pick_wpc(log2_field(field), N, K, t) > 0) {   // fused: TMEM engine
        TmParams vp{};
        vp.U = U; vp.RB = RB; vp.kw = kw; vp.mismatch = mismatch; vp.fault = tls_fault;
        if (field == 2)
            return t == 1 ? launch_tmem_check<0, 1>(A, C, B, N, K, M, batch, st, &vp)
                          : launch_tmem_check<0, 2>(A, C, B, N, K, M, batch, st, &vp);
        if (field == 16)
            return t == 1 ? launch_tmem_check<2, 1>(A, C, B, N, K, M, batch, st, &vp)
                          : launch_tmem_check<2, 2>(A, C, B, N, K, M, batch, st, &vp);
        return t == 1 ? launch_tmem_check<1, 1>(A, C, B, N, K, M, batch, st, &vp)
                      : launch_tmem_check<1, 2>(A, C, B, N, K, M, batch, st, &vp);
    }
    // The GF(2) split engine (HBM-bound: a second pass over A and B would double
    // its traffic) checks inside the encode.  Every other kernel -- the
    // shared-memory-bound product-row kernels among them, which leave most of
    // the HBM bandwidth unused -- runs the encode and then one streaming pass
    // over A and B (verify_words_kernel; C3 GF(256): +17.9% at t = 2 against
    // +51% for the product-row kernel with the check fused into it, which was
    // removed).
    if (path == 11 && K <= 64) {                               // fused: GF(2) split engine
        Gf2Params vp;
        std::memset(&vp, 0, sizeof(vp));
        vp.U = U; vp.RB = RB; vp.kw = kw; vp.t = t; vp.mismatch = mismatch; vp.fault = tls_fault;
        if (t == 1)                                            // one projection: 12 warps / SM as the encode
            return N <= 16 ? launch_gf2<16, 1>(A, C, B, N, K, M, batch, st, &vp)
                           : launch_gf2<32, 1>(A, C, B, N, K, M, batch, st, &vp);
        return N <= 16 ? launch_gf2<16, 2>(A, C, B, N, K, M, batch, st, &vp)
                       : launch_gf2<32, 2>(A, C, B, N, K, M, batch, st, &vp);
    }
    if ((path == 2 || path == 3) && K <= 64) {                 // fused: lane-k, one block per CTA
        LanekParams vp{};
        vp.U = U; vp.RB = RB; vp.kw = kw; vp.mismatch = mismatch; vp.fault = tls_fault;
        const bool kg2 = K > 32;
        switch (field) {
        case 256: return kg2 ? (t == 1 ? launch_lanek<256, 2, 1>(A, C, B, N, K, M, batch, st, &vp)
                                       : launch_lanek<256, 2, 2>(A, C, B, N, K, M, batch, st, &vp))
                             : (t == 1 ? launch_lanek<256, 1, 1>(A, C, B, N, K, M, batch, st, &vp)
                                       : launch_lanek<256, 1, 2>(A, C, B, N, K, M, batch, st, &vp));
        case 16: return kg2 ? (t == 1 ? launch_lanek<16, 2, 1>(A, C, B, N, K, M, batch, st, &vp)
                                      : launch_lanek<16, 2, 2>(A, C, B, N, K, M, batch, st, &vp))
                            : (t == 1 ? launch_lanek<16, 1, 1>(A, C, B, N, K, M, batch, st, &vp)
                                      : launch_lanek<16, 1, 2>(A, C, B, N, K, M, batch, st, &vp));
        case 4: return kg2 ? (t == 1 ? launch_lanek<4, 2, 1>(A, C, B, N, K, M, batch, st, &vp)
                                     : launch_lanek<4, 2, 2>(A, C, B, N, K, M, batch, st, &vp))
                           : (t == 1 ? launch_lanek<4, 1, 1>(A, C, B, N, K, M, batch, st, &vp)
                                     : launch_lanek<4, 1, 2>(A, C, B, N, K, M, batch, st, &vp));
        default: return kg2 ? (t == 1 ? launch_lanek<2, 2, 1>(A, C, B, N, K, M, batch, st, &vp)
                                      : launch_lanek<2, 2, 2>(A, C, B, N, K, M, batch, st, &vp))
                            : (t == 1 ? launch_lanek<2, 1, 1>(A, C, B, N, K, M, batch, st, &vp)
                                      : launch_lanek<2, 1, 2>(A, C, B, N, K, M, batch, st, &vp));
        }
    }
    // every other kernel: the encode, then the same check in a streaming pass
    if ((rc = encode_on_stream(field, fi, A, C, B, N, K, M, batch, st)) != GF_OK) return rc;
    if (tls_fault >> 63) {
        const size_t fg = (tls_fault >> 32) & 0x7FFFFFFFu, fk = (tls_fault >> 20) & 0xFFFu, fw = tls_fault & 0xFFFFFu;
        if (fg < batch && fk < (size_t)K && 4 * fw < M) fault_byte_kernel<<<1, 1, 0, st>>>(B + (fg * K + fk) * M + 4 * fw);
    }
    void *tabs = nullptr;
    if (symbol_address(0, &tabs) != GF_OK) return GF_ECUDA;
    const uint32_t *ftabs = reinterpret_cast<const uint32_t *>(tabs) + (size_t)fi * 256 * kTableWords;
    if (M % 4 == 0 && ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 3u) == 0) {
        const size_t units = batch * ((M / 4 + 32 * kVwW - 1) / (32 * kVwW));   // (generation, 128-word chunk)
        if (units > 0x7FFFFFFFu) return GF_EARG;
        // blocks of 64 coded packets per pass over A: all of them up to four
        const int kb = kblocks >= 4 ? 4 : kblocks;
        auto go = [&](auto kern) {
            kern<<<(unsigned)units, 32, 0, st>>>(A, B, U, RB, ftabs, N, K, kblocks, kw, M, batch, mismatch);
        };
        if (t == 1) {
            if (kb == 1) go(verify_words_kernel<1, 1>);
            else if (kb == 2) go(verify_words_kernel<1, 2>);
            else if (kb == 3) go(verify_words_kernel<1, 3>);
            else go(verify_words_kernel<1, 4>);
        } else {
            if (kb == 1) go(verify_words_kernel<2, 1>);
            else if (kb == 2) go(verify_words_kernel<2, 2>);
            else if (kb == 3) go(verify_words_kernel<2, 3>);
            else go(verify_words_kernel<2, 4>);
        }
        return launch_status();
    }
    unsigned gx = (unsigned)((M + 255) / 256);
    if (gx > 64) gx = 64;
    for (size_t g0 = 0; g0 < batch; g0 += 65535) {
        const size_t gn = batch - g0 < 65535 ? batch - g0 : 65535;
        verify_plain_kernel<<<dim3(gx, (unsigned)gn), 256, 0, st>>>(
            A + g0 * (size_t)N * M, B + g0 * (size_t)K * M, U + g0 * (size_t)kblocks * 2 * N, RB + g0 * 2 * (size_t)kw,
            reinterpret_cast<const uint32_t *>(tabs) + (size_t)fi * 256 * kTableWords, N, K, kblocks, kw, M, gn,
            mismatch + g0);
        if ((rc = launch_status()) != GF_OK) return rc;
    }
    return GF_OK;
}

int gf_fill_random2d(uint8_t *dst, size_t rows, size_t cols, uint64_t seed, uint64_t stream,
                     uint64_t base, uint64_t row_stride, uint8_t mask)
{
    if (rows == 0 || cols == 0) return GF_OK;
    if (!dst) return GF_EARG;
    int dev;
    if (current_device(&dev) != GF_OK) return GF_ECUDA;
    const uint64_t key = seed ^ (stream * kStreamMul);
    const bool words = cols % 8 == 0 && base % 8 == 0 && row_stride % 8 == 0 &&
                       (reinterpret_cast<uintptr_t>(dst) & 7u) == 0;
    const size_t total = words ? rows * (cols / 8) : rows * cols;
    size_t blocks = (total + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (words)
        fill_random_kernel<true><<<(unsigned)blocks, 256, 0, tls_stream>>>(dst, rows, cols, key, base,
                                                                            row_stride, mask);
    else
        fill_random_kernel<false><<<(unsigned)blocks, 256, 0, tls_stream>>>(dst, rows, cols, key, base,
                                                                             row_stride, mask);
    return launch_status();
}

int gf_fill_random(uint8_t *dst, size_t bytes, uint64_t seed, uint64_t stream, uint64_t offset,
                   uint8_t mask)
{
    if (bytes == 0) return GF_OK;
    // a 1-D range is a single row (64-bit stores when offset, dst, bytes allow)
    return gf_fill_random2d(dst, 1, bytes, seed, stream, offset, bytes, mask);
}

}  // extern "C"
