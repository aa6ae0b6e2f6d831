// tcgen05 weight-streaming GEMM for the ragged forward (sm_100a): the batched
// draft / verify projections of BASS (ref:model.py:160-164 `_linear`,
// :214-245; the dense layers stay batched).
//
//   Y[m, n] = sum_k X[m, k] W[n, k]      (W output-major [N, K] bf16, X [M, K] bf16)
//
// Swap-AB: weight rows are the MMA's M side (NB sub-tiles of 128 rows per
// CTA), the token block the N side (TT = 16..256 tokens), so a skinny
// verify/draft GEMM (M = 8..264 rows) issues full 128-row UMMAs and the kernel
// is a pure HBM weight stream.  Per CTA a ring of shared-memory stages
// {W NB x [128 x 64], X [TT x 64]} is filled by one producer thread — W as
// contiguous 16 KB blocks of the packed tile layout (one 1-D bulk copy each,
// whole DRAM pages; common.cuh packed_index), X through a 2-D TMA map — and
// one elected thread issues tcgen05.mma (kind::f16, fp32 accumulators in
// TMEM, one per sub-tile).  With NB = 2 the two sub-tiles share every X tile,
// halving the L2 -> SM activation traffic that bounds the verify shapes
// (M ~ 88-264).  After the last k block four warps drain TMEM (tcgen05.ld
// 32x32b) through the fused epilogue (QKV + KV-append, residual add, exact
// GELU, fp32 logits).
// Split-K over a fixed split count S(N, K) — never a function of M, so a
// row's bits do not depend on the batch (batched == solo, verify ==
// sequential decode): the S CTAs of a tile are one thread-block cluster; each
// writes its fp32 partial to an L2-resident workspace and after a cluster
// barrier reduces 1/S of the tile in split order (deterministic, no atomics).
// Many CTAs (2 per SM when they fit) let the hardware scheduler balance the
// tail and let the next kernel (PDL) prefetch its weights beside this one.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <tuple>

#include "runtime.h"
#include "quant.cuh"

namespace bass {
namespace tc {

constexpr int BN = 128;          // weight rows per sub-tile (UMMA M)
constexpr int BK = 64;           // k per stage (one 128-byte swizzle row of bf16)
constexpr int UK = 16;           // k per tcgen05.mma for 16-bit inputs
constexpr int EH = 2;               // epilogue row groups: warps w, w + 4 share TMEM lane quarter w (EH = 3 with 80 registers measured slower)
constexpr int THREADS = 128 * EH;   // 8 warps: 0 producer, 1 MMA, 2 TMEM alloc / folded-LN stats; all drain

// STG > 0: a fixed ring depth (a GEMM whose every split fits in STG stages
// takes less shared memory, so its CTAs can start beside the kernel before it)
template <int TT, int NB, int STG = 0>
struct Cfg {
    static constexpr int W_BYTES = NB * BN * BK * 2;
    static constexpr int X_BYTES = TT * BK * 2;
    static constexpr int STAGE = W_BYTES + X_BYTES;
    // two CTAs per SM (110 KB) when that still leaves >= 2 stages, else one
    static constexpr int BUDGET = (110 * 1024 - 2048) / STAGE >= 2 ? 110 * 1024 - 2048 : 200 * 1024;
    static constexpr int STAGES_RAW = BUDGET / STAGE;
    static constexpr int STAGES = STG > 0 ? STG : STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
    static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/ + 2 * TT * 4 /*XN row stats*/;
    static constexpr int COLS = NB * TT;
    static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try(bar, parity)) {
    }
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint32_t dst, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
// 1-D bulk copy global -> shared (one packed 16 KB weight tile)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// L2 policy for data read once per forward (weights, K/V history): evict first,
// so the stream does not push activations and kernel code out of L2
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B
// apart (SBO = 64 x 16 B), LBO = 1 (unused for swizzled K-major), version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
// instruction descriptor: bf16 x bf16 -> f32, K-major A and B, M = 128, N = tt
__host__ __device__ constexpr uint32_t idesc(int tt) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(tt >> 3) << 17) | ((uint32_t)(BN >> 4) << 24);
}
// kind::i8: signed int8 x signed int8 -> s32 (D format 2, A / B format 1 = signed)
__host__ __device__ constexpr uint32_t idesc_i8(int tt) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(tt >> 3) << 17) | ((uint32_t)(BN >> 4) << 24);
}
// one kind::i8 MMA consumes 32 int8 of k (32 bytes, the same step as 16 bf16)
__device__ __forceinline__ void umma_i8(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(
            dtmem),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
            dtmem),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

struct Split {
    int S;             // number of K splits
    int k_iters;       // K / BK (int8: K / 128 — a stage is always 128 bytes of k)
    float* ws;         // per (tile, token group): [S][TT][NB*BN] fp32 partials (S > 1; int8: s32 bits)
    int evict_first;   // weights streamed with an L2 evict-first policy
    const double* sx;  // int8 (W8A8): per-token activation scales [M]
    const double* sw;  // int8 (W8A8): per-channel weight scales [N]
    const int32_t* m_dev;   // device-planned forward: rows beyond *m_dev are not live
};

// LayerNorm folded into the GEMM (XN):  LN(x) W^T = rstd * ((x*g) W^T - mean * c) + e
// with c = W g and e = W b per output column (precomputed), X = bf16(x * g)
// written by the previous residual epilogue, and the row mean / rstd from
// the per-(tile, row) sums that epilogue emitted (`stats`, `stat_tiles`).
struct XNorm {
    const float* stats;    // [stat_tiles][M] {sum, sum of squares} of c = x - K (K: the producer's row shift)
    const float* c;        // [N] sum_k g_k W[n, k]
    const float* e;        // [N] sum_k b_k W[n, k]
    float* kmean;          // [M] row shift K on entry; the tile-0 / split-0 CTA leaves K + mean(c) = mean(x)
    int stat_tiles;
};

// Split-K reduction of U consecutive partial rows: all S x U loads are issued
// before the first add, then summed in split order s = 0..S-1 (the fixed
// order every path uses, so the bits do not depend on the path or on M).
constexpr int MAX_S = 8;
template <int U, bool INT = false>
__device__ __forceinline__ void dsmem_sum(uint32_t addr0, uint32_t row_stride, int S, float* acc) {
    float p[MAX_S][U];
#pragma unroll
    for (int s = 0; s < MAX_S; ++s)
        if (s < S) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr0 + u * row_stride), "r"(s));
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(p[s][u]) : "r"(ra));
            }
        }
    if constexpr (INT) {   // s32 partials (kind::i8): exact integer sum, bits returned in a float
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int a = 0;
#pragma unroll
            for (int s = 0; s < MAX_S; ++s)
                if (s < S) a += __float_as_int(p[s][u]);
            acc[u] = __int_as_float(a);
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;
#pragma unroll
    for (int s = 0; s < MAX_S; ++s)
        if (s < S) {
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] += p[s][u];
        }
}
template <int U, bool INT = false>
__device__ __forceinline__ void l2_sum(const float* p0, int64_t split_stride, int64_t row_stride, int S, float* acc) {
    float p[MAX_S][U];
#pragma unroll
    for (int s = 0; s < MAX_S; ++s)
        if (s < S) {
#pragma unroll
            for (int u = 0; u < U; ++u) p[s][u] = __ldcg(p0 + s * split_stride + u * row_stride);
        }
    if constexpr (INT) {   // s32 partials (kind::i8): exact integer sum, bits returned in a float
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int a = 0;
#pragma unroll
            for (int s = 0; s < MAX_S; ++s)
                if (s < S) a += __float_as_int(p[s][u]);
            acc[u] = __int_as_float(a);
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;
#pragma unroll
    for (int s = 0; s < MAX_S; ++s)
        if (s < S) {
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] += p[s][u];
        }
}

#ifdef BASS_GEMM_PROBE
// debug build only: globaltimer stamps of one GEMM shape's pipeline events
// (first 16 CTAs of every launch with N == g_gp_n, K == g_gp_k; the last such
// launch wins)
__device__ unsigned long long* g_gp;
__device__ int g_gp_n, g_gp_k;
#define GPROBE(i)                                      \
    do {                                               \
        if (gp_on) g_gp[gp_cta * 16 + (i)] = gtimer(); \
    } while (0)
#else
#define GPROBE(i) \
    do {          \
    } while (0)
#endif

// PACKED: W in the packed tile layout (1-D bulk copies); else W [N, K] via `tw`.
// LNF: 0 plain; 1 (consumer) the LayerNorm preceding this GEMM is folded in
// (see XNorm); 2 (residual producer) the epilogue also emits the next
// LayerNorm's row sums and X = bf16(x * g_next).  Compile-time, so the plain
// kernels carry none of it.
// I8: W8A8 — int8 packed weights and int8 activations (kind::i8, s32
// accumulators), dequantized in the epilogue: acc * sx[m] * sw[n] in fp64
// (ref:quant.py:98-123 int_gemm_dequant).  LNF must be 0.
// SER: serial split-K for prefill-sized M — one CTA per (token group, tile)
// runs the S splits one after another, each into its own TMEM accumulator
// (S x TT <= 512 columns), and the epilogue sums the S partials in split
// order exactly as the cluster reduction does (same K partition, same
// accumulation and summation order: bit-identical rows, no cluster
// barriers, no partial exchange).
template <int TT, int MODE, int NB, bool PACKED, int LNF, bool I8 = false, bool SER = false, int STG = 0>
__global__ void __launch_bounds__(THREADS, EH > 2 ? 2 : 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tw,
                                                             const __grid_constant__ CUtensorMap tx,
                                                             const __nv_bfloat16* __restrict__ wpk, int M, int N,
                                                             Split sp, Epi e, XNorm xn, TraceArg tr) {
    constexpr bool XN = LNF == 1;
    static_assert(!I8 || (LNF == 0 && PACKED), "W8A8 GEMMs take packed weights and no folded LayerNorm");
    constexpr int XK = I8 ? 128 : BK;   // k elements of X per stage (128 bytes either way)
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
#ifdef BASS_GEMM_PROBE
    const int gp_cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const bool gp_on = g_gp && N == g_gp_n && sp.k_iters * BK == g_gp_k && gp_cta < 16;
#endif
    if (threadIdx.x == 0) GPROBE(0);
    using C = Cfg<TT, NB, STG>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = su32(smem_raw);
    const uint32_t base = (raw + 1023) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
    // bars[0..S) full, [S..2S) empty, [2S] done; tmem base address after
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 1);
    static_assert(!SER || NB == 1, "serial split-K: one 128-row sub-tile");
    // SER: one accumulator per split (the host keeps S x TT <= 512)
    const uint32_t tcols = SER ? (sp.S * TT <= 256 ? 256u : 512u) : (uint32_t)C::TMEM_COLS;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wq = warp & 3, half = warp >> 2;   // epilogue: TMEM lane quarter, row half
    // grid (token groups, splits, tiles): the token groups of one weight tile are
    // adjacent in launch order, so for large M (prefill) the tile is read from
    // HBM once and re-served from L2 to the other groups
    const int tile = blockIdx.z, split = blockIdx.y, group = blockIdx.x;
    const int n0 = tile * NB * BN, m0 = group * TT;
    // device-planned forward (decode-loop graph): the live rows are known only
    // on the device; a token group past them exits before touching anything
    // (all CTAs of a split-K cluster share the group)
    const int Mv = sp.m_dev ? min(M, __ldg(sp.m_dev)) : M;
    if (m0 >= Mv) return;
    const int it0 = SER ? 0 : (int)((int64_t)split * sp.k_iters / sp.S);
    const int it1 = SER ? sp.k_iters : (int)((int64_t)(split + 1) * sp.k_iters / sp.S);
    const int nit = it1 - it0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(su32(&bars[s]), 1);
            mbar_init(su32(&bars[C::STAGES + s]), 1);
        }
        mbar_init(su32(&bars[2 * C::STAGES]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (!PACKED) asm volatile("prefetch.tensormap [%0];" ::"l"(&tw) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tx) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(tcols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // PDL: let the next kernel's CTAs start their own prologue / weight
    // prefetch as soon as SMs free up
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t wpol = sp.evict_first ? policy_evict_first() : 0ull;
    auto load_w = [&](uint32_t dst, uint32_t bar, int kb) {
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            if constexpr (PACKED) {
                const int nt = tile * NB + sub;   // 128-row packed tile
                if (wpol)
                    bulk_g2s_hint(dst + sub * BN * BK * 2, wpk + ((int64_t)nt * sp.k_iters + kb) * (BN * BK),
                                  BN * BK * 2, bar, wpol);
                else
                    bulk_g2s(dst + sub * BN * BK * 2, wpk + ((int64_t)nt * sp.k_iters + kb) * (BN * BK), BN * BK * 2, bar);
            } else {
                tma_2d(&tw, dst + sub * BN * BK * 2, bar, kb * BK, n0 + sub * BN);
            }
        }
    };
    if (warp == 0) {
        if (lane == 0) {   // ---- producer
            // Weights do not depend on the previous kernel: fill the ring with
            // W tiles first, then wait for the producer of X (griddepcontrol)
            const int pre = nit < C::STAGES ? nit : C::STAGES;
            for (int i = 0; i < pre; ++i) {
                const uint32_t full = su32(&bars[i]);
                mbar_expect_tx(full, C::STAGE);
                load_w(base + i * C::STAGE, full, it0 + i);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            GPROBE(1);
            for (int i = 0; i < pre; ++i)
                tma_2d(&tx, base + i * C::STAGE + C::W_BYTES, su32(&bars[i]), (it0 + i) * XK, m0);
            for (int i = pre; i < nit; ++i) {
                const int s = i % C::STAGES;
                mbar_wait(su32(&bars[C::STAGES + s]), ((i / C::STAGES) - 1) & 1);
                const uint32_t full = su32(&bars[s]);
                const uint32_t st = base + s * C::STAGE;
                mbar_expect_tx(full, C::STAGE);
                load_w(st, full, it0 + i);
                tma_2d(&tx, st + C::W_BYTES, full, (it0 + i) * XK, m0);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {   // ---- MMA issuer: one accumulator (TT columns) per sub-tile
            constexpr uint32_t ID = I8 ? idesc_i8(TT) : idesc(TT);
            int ps = 0;                                                  // SER: current split
            int pb0 = 0, pb1 = SER ? (int)((int64_t)sp.k_iters / sp.S) : nit;   // its k-block range
            for (int i = 0; i < nit; ++i) {
                const int s = i % C::STAGES;
                const bool first = i == pb0;
                mbar_wait(su32(&bars[s]), (i / C::STAGES) & 1);
                if (i == 0) GPROBE(2);
                fence_after();
                const uint32_t st = base + s * C::STAGE;
                const uint64_t b = sdesc(st + C::W_BYTES);
                const uint32_t dacc = tmem + (SER ? (uint32_t)(ps * TT) : 0u);
#pragma unroll
                for (int sub = 0; sub < NB; ++sub) {
                    const uint64_t a = sdesc(st + sub * BN * BK * 2);
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk) {   // +32 bytes per UMMA_K step inside the swizzle row
                        if constexpr (I8)
                            umma_i8(dacc + sub * TT, a + (uint64_t)(kk * 2), b + (uint64_t)(kk * 2), ID,
                                    (!first || kk > 0) ? 1u : 0u);
                        else
                            umma(dacc + sub * TT, a + (uint64_t)(kk * 2), b + (uint64_t)(kk * 2), ID,
                                 (!first || kk > 0) ? 1u : 0u);
                    }
                }
                umma_commit(su32(&bars[C::STAGES + s]));
                if (SER && i == pb1 - 1) {   // split ps complete: the next one starts a fresh accumulator
                    ++ps;
                    pb0 = pb1;
                    pb1 = (int)((int64_t)(ps + 1) * sp.k_iters / sp.S);
                }
            }
            umma_commit(su32(&bars[2 * C::STAGES]));
            GPROBE(3);
        }
        __syncwarp();
    } else if (XN && warp == 2) {
        // ---- folded LayerNorm (warp 2, idle during the main loop): row mean /
        // rstd of this CTA's token rows from the per-(tile, row) sums
        const int K = sp.k_iters * BK;
        float* s_mean = reinterpret_cast<float*>(tmem_slot + 4);   // [TT]
        float* s_rstd = s_mean + TT;                                // [TT]
        asm volatile("griddepcontrol.wait;" ::: "memory");        // the sums are complete
        for (int r = lane; r < TT; r += 32) {
            const int m = m0 + r;
            float mean = 0.f, rstd = 0.f;
            if (m < M) {
                float sm = 0.f, sq = 0.f;
                for (int t0 = 0; t0 < xn.stat_tiles; t0 += 8) {   // 8 loads in flight, summed in tile order
                    float2 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (t0 + u < xn.stat_tiles)
                            v[u] = __ldcg(reinterpret_cast<const float2*>(xn.stats) + (int64_t)(t0 + u) * M + m);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (t0 + u < xn.stat_tiles) {
                            sm += v[u].x;
                            sq += v[u].y;
                        }
                }
                    // sums are of c = x - K (K = the producer's row shift ~ mean):
                // `mean` is mean(c) = mean(x) - K, var(x) = E[c^2] - mean(c)^2
                mean = sm / (float)K;
                const float var = fmaxf(sq / (float)K - mean * mean, 0.f);
                rstd = 1.0f / sqrtf(var + 1e-5f);
            }
            s_mean[r] = mean;
            s_rstd[r] = rstd;
            // the row's exact mean for the next residual producer's shift (one
            // writer per row; it is the only CTA of this launch touching kmean)
            if (xn.kmean && tile == 0 && split == 0 && m < M) xn.kmean[m] = __ldcg(xn.kmean + m) + mean;
        }
    } else if (LNF == 2 && warp == 2) {
        // ---- residual producer (warp 2, idle during the main loop): each row's
        // shift K = the mean of the stream this GEMM adds into (left in kmean by
        // the LayerNorm consumer before it); the epilogue centres on it
        float* s_shift = reinterpret_cast<float*>(tmem_slot + 4);   // [TT]
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int r = lane; r < TT; r += 32) {
            const int m = m0 + r;
            s_shift[r] = m < M ? __ldcg(e.shift + m) : 0.f;
        }
    }
    __syncwarp();

    // ---- epilogue: TMEM lane = weight row n0 + sub*128 + 32*warp + lane; columns = tokens
    asm volatile("griddepcontrol.wait;" ::: "memory");   // previous kernel's writes visible
    if (threadIdx.x == 64) GPROBE(4);
    if constexpr (LNF != 0) __syncthreads();              // row mean / rstd or shift (warp 2) visible
    mbar_wait(su32(&bars[2 * C::STAGES]), 0);
    if (threadIdx.x == 64) GPROBE(5);
    fence_after();
    const uint32_t trow = tmem + ((uint32_t)(wq * 32) << 16);
    const int rows = min(TT, Mv - m0);
    // the finished accumulator chunk of token columns [c0, c0 + 16): TMEM, or
    // for SER the S per-split accumulators summed in split order (the cluster
    // reduction's order: 0 + p0 + p1 + ...; s32 partials as integers)
    auto acc_chunk = [&](int sub, int c0, float* v) {
        if constexpr (SER) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            for (int s2 = 0; s2 < sp.S; ++s2) {
                float p[16];
                tmem_ld16(trow + (uint32_t)(s2 * TT) + c0, p);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    v[j] = I8 ? __int_as_float(__float_as_int(v[j]) + __float_as_int(p[j])) : v[j] + p[j];
            }
        } else {
            tmem_ld16(trow + sub * TT + c0, v);
        }
    };
    const bool direct = SER || sp.S == 1;   // no cross-CTA reduction in the epilogue
    // W8A8: s32 accumulator bits -> acc * s_token * s_channel (fp64, ref:quant.py:119)
    auto deq = [&](int m, int n, float bits) -> float {
        if constexpr (I8) return (float)((double)__float_as_int(bits) * __ldg(sp.sx + m) * __ldg(sp.sw + n));
        else return bits;
    };
    // W8A8 FC epilogue (its output is quantized per token next, ref:model.py:243-244):
    // the exact GELU, an fp32 store and the row's running max |value| — lanes
    // hold consecutive columns, so a warp shuffle reduction and one
    // uint-ordered atomicMax (|v| >= 0) per warp: order-free, deterministic.
    auto emit = [&](int m, int n, float bits) {
        const float v0 = deq(m, n, bits);
        if constexpr (I8 && MODE == EPI_GELU) {
            const float v = gelu_erf(v0);
            reinterpret_cast<float*>(e.out)[(int64_t)m * N + n] = v;
            float a = fabsf(v);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
            if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(e.amax) + m, __float_as_uint(a));
        } else {
            epilogue<MODE, __nv_bfloat16>(e, m, n, N, v0);
        }
    };
    // W8A8 QKV: q / k / v fake-quantized per (token, head) right here
    // (ref:model.py:219-222, quant.py:126-129) and written as bf16 to q and
    // the KV cache — no fp32 round trip, no separate quantizer kernel.  A
    // head's columns are one warp (d_head <= 32) or 2-4 warps of the same
    // row half: their maxima meet in a 512-byte exchange at the end of the
    // (idle) stage ring behind a 128-thread named barrier per half.
    constexpr bool QQ = I8 && MODE == EPI_QKV;
    float* qx = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE - 512) + half * 64;   // [16 rows][4 warps]
    auto qgrp = [&](auto& w, int m_first, int count, int n) {
        constexpr int U = sizeof(w) / sizeof(float);
        const int dh = e.dh, g = dh < 32 ? dh : 32;
        float a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u] = u < count ? fabsf(w[u]) : 0.f;
            for (int o = 1; o < g; o <<= 1) a[u] = fmaxf(a[u], __shfl_xor_sync(0xffffffffu, a[u], o));
        }
        if (dh > 32) {
            if (lane == 0)
#pragma unroll
                for (int u = 0; u < U; ++u) qx[u * 4 + wq] = a[u];
            asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
            const int wpg = dh / 32, w0 = (wq / wpg) * wpg;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float mx = 0.f;
                for (int t = 0; t < wpg; ++t) mx = fmaxf(mx, qx[u * 4 + w0 + t]);
                a[u] = mx;
            }
            asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
        }
        const int part = n / e.d, nn = n - part * e.d, hh = nn / dh, c = nn - hh * dh;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u >= count) break;
            const int m = m_first + u;
            const double sc = group_scale(a[u]);
            const __nv_bfloat16 val = __float2bfloat16_rn((float)((double)quant_round((double)w[u] / sc) * sc));
            if (part == 0)
                reinterpret_cast<__nv_bfloat16*>(e.out)[(int64_t)m * e.d + nn] = val;
            else
                reinterpret_cast<__nv_bfloat16*>(part == 1 ? e.kc : e.vc)
                    [(((int64_t)__ldg(e.row_slot + m) * e.H + hh) * e.cap + __ldg(e.row_pos + m)) * dh + c] = val;
        }
    };
    if constexpr (LNF == 0) {
    if (direct) {
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int n = n0 + sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                acc_chunk(sub, c0, v);
                if (n < N) {
                    if constexpr (QQ) {
                        float w[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) w[j] = c0 + j < rows ? deq(m0 + c0 + j, n, v[j]) : 0.f;
                        qgrp(w, m0 + c0, min(16, rows - c0), n);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < rows) emit(m0 + c0 + j, n, v[j]);
                    }
                }
            }
        }
    } else if ((size_t)rows * NB * BN * 4 + (QQ ? 512 : 0) <= (size_t)C::STAGES * C::STAGE) {
        // split-K through distributed shared memory: the S CTAs of this tile
        // are one cluster.  Each parks its fp32 partial [token][row] in its own
        // (now idle) stage ring, the cluster barrier publishes it, and CTA
        // `split` reduces token rows [split*R/S, (split+1)*R/S) reading every
        // rank's partial over DSMEM, in fixed split order (same arithmetic as
        // the L2 path below).
        constexpr int WR = NB * BN;
        float* part = reinterpret_cast<float*>(smem);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                tmem_ld16(trow + sub * TT + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < rows) part[(c0 + j) * WR + nn] = v[j];
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int r0 = split * rows / sp.S, r1 = (split + 1) * rows / sp.S;
        // the EH warp groups take consecutive 4-row-aligned slices of [r0, r1)
        const int rper = ((r1 - r0 + 4 * EH - 1) / (4 * EH)) * 4;
        const int rb = r0 + min(r1 - r0, half * rper), re = r0 + min(r1 - r0, (half + 1) * rper);
        const uint32_t part_s = su32(part);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane, n = n0 + nn;
            if (n < N) {
                int r = rb;
                for (; r + 4 <= re; r += 4) {   // 4 rows x S partials in flight
                    float acc[4];
                    dsmem_sum<4, I8>(part_s + (uint32_t)((r * WR + nn) * 4), WR * 4, sp.S, acc);
                    if constexpr (QQ) {
                        float w[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) w[u] = deq(m0 + r + u, n, acc[u]);
                        qgrp(w, m0 + r, 4, n);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) emit(m0 + r + u, n, acc[u]);
                    }
                }
                for (; r < re; ++r) {
                    float acc;
                    dsmem_sum<1, I8>(part_s + (uint32_t)((r * WR + nn) * 4), WR * 4, sp.S, &acc);
                    if constexpr (QQ) {
                        float w[1] = {deq(m0 + r, n, acc)};
                        qgrp(w, m0 + r, 1, n);
                    } else {
                        emit(m0 + r, n, acc);
                    }
                }
            }
        }
        // no CTA may leave (and free its shared memory) while others still read it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        // split-K through L2: the S CTAs of this tile are one thread-block
        // cluster.  Each writes its fp32 partial tile (L2-resident scratch),
        // the cluster barrier publishes them, and CTA `split` reduces token
        // rows [split*R/S, (split+1)*R/S) of the tile in fixed split order.
        constexpr int WR = NB * BN;   // partial row width
        float* blk = sp.ws + (int64_t)(tile * gridDim.x + group) * sp.S * TT * WR;
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                tmem_ld16(trow + sub * TT + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < rows) __stcg(&blk[((int64_t)split * TT + c0 + j) * WR + nn], v[j]);
            }
        }
        __threadfence();
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int r0 = split * rows / sp.S, r1 = (split + 1) * rows / sp.S;
        // the EH warp groups take consecutive 4-row-aligned slices of [r0, r1)
        const int rper = ((r1 - r0 + 4 * EH - 1) / (4 * EH)) * 4;
        const int rb = r0 + min(r1 - r0, half * rper), re = r0 + min(r1 - r0, (half + 1) * rper);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane, n = n0 + nn;
            if (n < N) {
                int r = rb;
                for (; r + 4 <= re; r += 4) {   // 4 rows x S partials in flight
                    float acc[4];
                    l2_sum<4, I8>(blk + (int64_t)r * WR + nn, (int64_t)TT * WR, WR, sp.S, acc);
                    if constexpr (QQ) {
                        float w[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) w[u] = deq(m0 + r + u, n, acc[u]);
                        qgrp(w, m0 + r, 4, n);
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) emit(m0 + r + u, n, acc[u]);
                    }
                }
                for (; r < re; ++r) {
                    float acc;
                    l2_sum<1, I8>(blk + (int64_t)r * WR + nn, (int64_t)TT * WR, WR, sp.S, &acc);
                    if constexpr (QQ) {
                        float w[1] = {deq(m0 + r, n, acc)};
                        qgrp(w, m0 + r, 1, n);
                    } else {
                        emit(m0 + r, n, acc);
                    }
                }
            }
        }
    }
    } else {
    // RESID with row statistics for the next LayerNorm: x += acc, and the
    // 128 columns' {sum, sum of squares} of the new x per row, reduced in a
    // fixed order (warp shuffle, then warps 0..3) — see XNorm
    constexpr bool stats = MODE == EPI_RESID && LNF == 2;
    float2* red = nullptr;        // [local row][warp] per-warp row sums (idle stage ring)
    const float* s_mean = reinterpret_cast<const float*>(tmem_slot + 4);
    const float* s_rstd = s_mean + TT;
    // per-thread column constants (NB == 1: one weight row n per thread)
    const int n_t = n0 + wq * 32 + lane;
    float g_n = 0.f, c_n = 0.f, e_n = 0.f;
    if (n_t < N) {
        if constexpr (stats) g_n = __ldg(e.xg + n_t);
        if constexpr (XN) {
            c_n = __ldg(xn.c + n_t);
            e_n = __ldg(xn.e + n_t);
        }
    }
    // QKV: this thread's column is a fixed destination — q [M, d] (column nn)
    // or the K / V cache of head h at dim c (row (slot, pos) per token row)
    __nv_bfloat16* qkv_base = nullptr;
    bool qkv_cache = false;
    if constexpr (MODE == EPI_QKV) {
        if (n_t < N) {
            const int part = n_t / e.d, nn = n_t - part * e.d;
            if (part == 0) {
                qkv_base = reinterpret_cast<__nv_bfloat16*>(e.out) + nn;
            } else {
                const int h = nn / e.dh, c = nn - h * e.dh;
                qkv_base = reinterpret_cast<__nv_bfloat16*>(part == 1 ? e.kc : e.vc) + (int64_t)h * e.cap * e.dh + c;
                qkv_cache = true;
            }
        }
    }
    // returns the new x (stats) — the row reduction is done 4 rows at a time by stat4
    // row-dependent epilogue inputs (old residual / KV-cache row offset), loaded
    // before the split-K reduction so their latency overlaps it
    struct RowIn {
        float x;
        int64_t off;
    };
    auto pre = [&](int m, int n) -> RowIn {
        RowIn ri{0.f, 0};
        if (n < N) {
            if constexpr (stats) ri.x = e.x[(int64_t)m * N + n];
            if constexpr (MODE == EPI_QKV)
                ri.off = qkv_cache ? ((int64_t)__ldg(e.row_slot + m) * e.H * e.cap + __ldg(e.row_pos + m)) * e.dh
                                   : (int64_t)m * e.d;
        }
        return ri;
    };
    auto put = [&](int m, int n, float acc, const RowIn& ri) -> float {
        float nv = 0.f;
        if (n < N) {
            if constexpr (stats) {
                const float xnew = ri.x + acc;
                e.x[(int64_t)m * N + n] = xnew;
                // X of the next GEMM (its LayerNorm folded): bf16((x - K) * g_next);
                // the statistics are of the centred value too
                nv = xnew - s_mean[m - m0];
                e.xb[(int64_t)m * N + n] = __float2bfloat16_rn(nv * g_n);
            } else {
                if constexpr (XN) {
                    const int r = m - m0;
                    acc = s_rstd[r] * (acc - s_mean[r] * c_n) + e_n;
                }
                if constexpr (MODE == EPI_QKV) qkv_base[ri.off] = __float2bfloat16_rn(acc);   // KV append (ref:kv_cache.py:63-84)
                else epilogue<MODE, __nv_bfloat16>(e, m, n, N, acc);
            }
        }
        return nv;
    };
    // {sum, sum^2} over the warp's 32 columns for 4 rows at once (transpose-
    // reduce: 9 shuffles), lane (4 i + 0) ends with value i = 2 * row + stat
    auto stat4 = [&](int r_local0, int count, float n0v, float n1v, float n2v, float n3v) {
        if constexpr (stats) {
            float a[8] = {n0v, n0v * n0v, n1v, n1v * n1v, n2v, n2v * n2v, n3v, n3v * n3v};
            {
                const bool up = lane & 16;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float snd = up ? a[i] : a[i + 4], kp = up ? a[i + 4] : a[i];
                    a[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 16);
                }
            }
            {
                const bool up = lane & 8;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float snd = up ? a[i] : a[i + 2], kp = up ? a[i + 2] : a[i];
                    a[i] = kp + __shfl_xor_sync(0xffffffffu, snd, 8);
                }
            }
            {
                const bool up = lane & 4;
                const float snd = up ? a[0] : a[1], kp = up ? a[1] : a[0];
                a[0] = kp + __shfl_xor_sync(0xffffffffu, snd, 4);
            }
            a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
            a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
            const int idx = (lane >> 2) & 7, row = idx >> 1;
            if ((lane & 3) == 0 && row < count) {
                float* dst = reinterpret_cast<float*>(&red[(r_local0 + row) * 4 + wq]);
                dst[idx & 1] = a[0];
            }
        }
    };
    auto flush_stats = [&](int r_first, int nrows) {
        if constexpr (!stats) return;
        __syncthreads();
        for (int t = threadIdx.x; t < nrows; t += THREADS) {
            const float2 a = red[t * 4], b = red[t * 4 + 1], c2 = red[t * 4 + 2], d = red[t * 4 + 3];
            reinterpret_cast<float2*>(e.stats)[(int64_t)tile * M + m0 + r_first + t] =
                make_float2((a.x + b.x) + (c2.x + d.x), (a.y + b.y) + (c2.y + d.y));
        }
    };
    if (direct) {
        red = reinterpret_cast<float2*>(smem);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int n = n0 + sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                acc_chunk(sub, c0, v);
#pragma unroll
                for (int j0 = 0; j0 < 16; j0 += 4) {
                    float nv[4] = {0.f, 0.f, 0.f, 0.f};
                    RowIn ri[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) ri[j] = pre(m0 + c0 + j0 + j, c0 + j0 + j < rows ? n : N);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (c0 + j0 + j < rows) nv[j] = put(m0 + c0 + j0 + j, n, v[j0 + j], ri[j]);
                    if (c0 + j0 < rows) stat4(c0 + j0, min(4, rows - c0 - j0), nv[0], nv[1], nv[2], nv[3]);
                }
            }
        }
        flush_stats(0, rows);
    } else if ((size_t)rows * (NB * BN * 4 + (stats ? 32 : 0)) <= (size_t)C::STAGES * C::STAGE) {
        // split-K through distributed shared memory: the S CTAs of this tile
        // are one cluster.  Each parks its fp32 partial [token][row] in its own
        // (now idle) stage ring, the cluster barrier publishes it, and CTA
        // `split` reduces token rows [split*R/S, (split+1)*R/S) reading every
        // rank's partial over DSMEM, in fixed split order (same arithmetic as
        // the L2 path below).
        constexpr int WR = NB * BN;
        float* part = reinterpret_cast<float*>(smem);
        red = reinterpret_cast<float2*>(smem + (size_t)rows * WR * 4);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                tmem_ld16(trow + sub * TT + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < rows) part[(c0 + j) * WR + nn] = v[j];
            }
        }
        if (threadIdx.x == 64) GPROBE(6);
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 64) GPROBE(7);
        const int r0 = split * rows / sp.S, r1 = (split + 1) * rows / sp.S;
        // the EH warp groups take consecutive 4-row-aligned slices of [r0, r1)
        const int rper = ((r1 - r0 + 4 * EH - 1) / (4 * EH)) * 4;
        const int rb = r0 + min(r1 - r0, half * rper), re = r0 + min(r1 - r0, (half + 1) * rper);
        const uint32_t part_s = su32(part);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane, n = n0 + nn;
            int r = rb;
            for (; r + 4 <= re; r += 4) {   // 4 rows x S partials in flight
                RowIn ri[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ri[u] = pre(m0 + r + u, n);
                float acc[4];
                dsmem_sum<4>(part_s + (uint32_t)((r * WR + nn) * 4), WR * 4, sp.S, acc);
                float nv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) nv[u] = put(m0 + r + u, n, acc[u], ri[u]);
                stat4(r - r0, 4, nv[0], nv[1], nv[2], nv[3]);
            }
            for (; r < re; ++r) {
                const RowIn ri = pre(m0 + r, n);
                float acc;
                dsmem_sum<1>(part_s + (uint32_t)((r * WR + nn) * 4), WR * 4, sp.S, &acc);
                stat4(r - r0, 1, put(m0 + r, n, acc, ri), 0.f, 0.f, 0.f);
            }
        }
        if (threadIdx.x == 64) GPROBE(8);
        flush_stats(r0, r1 - r0);
        if (threadIdx.x == 64) GPROBE(9);
        // no CTA may leave (and free its shared memory) while others still read it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (threadIdx.x == 64) GPROBE(10);
    } else {
        // split-K through L2: the S CTAs of this tile are one thread-block
        // cluster.  Each writes its fp32 partial tile (L2-resident scratch),
        // the cluster barrier publishes them, and CTA `split` reduces token
        // rows [split*R/S, (split+1)*R/S) of the tile in fixed split order.
        constexpr int WR = NB * BN;   // partial row width
        float* blk = sp.ws + (int64_t)(tile * gridDim.x + group) * sp.S * TT * WR;
        red = reinterpret_cast<float2*>(smem);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane;
#pragma unroll 1
            for (int c0 = half * 16; c0 < TT; c0 += 16 * EH) {
                if (c0 >= rows) break;
                float v[16];
                tmem_ld16(trow + sub * TT + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < rows) __stcg(&blk[((int64_t)split * TT + c0 + j) * WR + nn], v[j]);
            }
        }
        __threadfence();
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int r0 = split * rows / sp.S, r1 = (split + 1) * rows / sp.S;
        // the EH warp groups take consecutive 4-row-aligned slices of [r0, r1)
        const int rper = ((r1 - r0 + 4 * EH - 1) / (4 * EH)) * 4;
        const int rb = r0 + min(r1 - r0, half * rper), re = r0 + min(r1 - r0, (half + 1) * rper);
#pragma unroll
        for (int sub = 0; sub < NB; ++sub) {
            const int nn = sub * BN + wq * 32 + lane, n = n0 + nn;
            int r = rb;
            for (; r + 4 <= re; r += 4) {   // 4 rows x S partials in flight
                RowIn ri[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ri[u] = pre(m0 + r + u, n);
                float acc[4];
                l2_sum<4>(blk + (int64_t)r * WR + nn, (int64_t)TT * WR, WR, sp.S, acc);
                float nv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) nv[u] = put(m0 + r + u, n, acc[u], ri[u]);
                stat4(r - r0, 4, nv[0], nv[1], nv[2], nv[3]);
            }
            for (; r < re; ++r) {
                const RowIn ri = pre(m0 + r, n);
                float acc;
                l2_sum<1>(blk + (int64_t)r * WR + nn, (int64_t)TT * WR, WR, sp.S, &acc);
                stat4(r - r0, 1, put(m0 + r, n, acc, ri), 0.f, 0.f, 0.f);
            }
        }
        flush_stats(r0, r1 - r0);
    }
    }
    fence_before();
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols)
                     : "memory");
    if (threadIdx.x == 64) GPROBE(11);
    if (tr.buf && threadIdx.x == 0) {   // trace record index: linear block id
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        const long long id = tr.base + blockIdx.x + (long long)gridDim.x * (blockIdx.y + (long long)gridDim.y * blockIdx.z);
        unsigned long long* rec = tr.buf + 4 * id;
        rec[0] = t_start;
        rec[1] = gtimer();
        rec[2] = sm;
        rec[3] = (unsigned long long)tr.tag;
    }
}

// ------------------------------------------------------------------ host
#ifdef BASS_GEMM_PROBE
void gemm_probe_set(void* p, int n, int k) {
    BASS_CUDA(cudaMemcpyToSymbol(g_gp, &p, sizeof(p)));
    BASS_CUDA(cudaMemcpyToSymbol(g_gp_n, &n, sizeof(n)));
    BASS_CUDA(cudaMemcpyToSymbol(g_gp_k, &k, sizeof(k)));
}
#endif

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        BASS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeFn)p;
    }
    return fn;
}

// 2D row-major [rows, cols] map with a box of {128 bytes of cols, box_rows}, 128B swizzle
// (bf16: 64 columns; int8: 128 columns)
static CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int box_rows, bool i8 = false) {
    CUtensorMap m;
    const int es = i8 ? 1 : 2;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * es};
    cuuint32_t box[2] = {(cuuint32_t)(128 / es), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encoder()(&m, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

struct State {
    std::map<std::tuple<const void*, int, int>, CUtensorMap> wmaps;
    std::map<std::tuple<const void*, int, int, int>, CUtensorMap> xmaps;   // (X, M, K, TT); int8 X: K < 0
    std::map<std::pair<int, int>, int> splits;
    DevBuf ws;
};

static State& state(bass_model& m) {
    if (!m.tc_state) m.tc_state = new State();
    return *static_cast<State*>(m.tc_state);
}

// Split count from (N, K) and the SM count only — never from M — so a row's
// reduction order (and hence its bits) does not depend on how many rows share
// the launch.  Rule (fit to the in-chain sweeps of profiles/r1_gemm_nb_split_sweep.txt,
// profiles/r1_split_chain_final.txt): the largest S <= 8 that divides the k
// blocks evenly, leaves >= 4 k blocks per CTA and keeps the 128-row tiles x S
// within 1.75 CTAs per SM; S = 2 may fill the two-CTA-per-SM wave (<= 2 per SM)
// when each CTA still streams >= 32 k blocks.  At every C2 shape this gives the
// measured optimum (qkv 2, o 6, fc 2, proj 6, head 1; draft 4 / 8 / 4 / 8 / 1).
// int8 (W8A8) GEMMs pass K / 2 (a k block is 128 bytes either way) and a
// 16-block floor for the two-CTA wave: their per-CTA stream is half as long
// for the same split, and the C2 FC projection measured best at S = 2
// (1.494 -> 1.457 ms/token; profiles/r2/int8_split_sweep.txt).
static int choose_splits(int sm_count, int N, int K, int wave_blocks = 32) {
    const int n_tiles = (N + BN - 1) / BN, k_iters = K / BK;
    int best = 1;
    for (int s = 2; s <= MAX_S; ++s) {
        if (k_iters % s != 0 || k_iters / s < 4) continue;
        const int ctas = n_tiles * s;
        if (ctas * 4 <= sm_count * 7 || (s == 2 && ctas <= 2 * sm_count && k_iters / s >= wave_blocks)) best = s;
    }
    return best;
}

struct LaunchArgs {
    const CUtensorMap* wm;
    const CUtensorMap* xm;
    const void* W;
    int M, N;
    Split sp;
    XNorm xn;
    bool lite;
};

template <int TT, int MODE, bool PACKED, int LNF, bool I8 = false, bool SER = false, int STG = 0>
static void launch_k(bass_model& m, const LaunchArgs& a, const Epi& e) {
    constexpr int NB = 1;   // (NB = 2 measured slower at every benchmark shape: profiles/r1_gemm_nb_split_sweep.txt)
    // serial split-K at 256-token tiles: 512 TMEM columns hold one CTA per
    // SM, so its ring takes four 48 KB stages instead of the two-CTA budget
    constexpr int STG_ = (SER && TT == 256) ? 4 : STG;
    using C = Cfg<TT, NB, STG_>;
    static unsigned attr = 0;
    once_per_device(attr, [] {
        BASS_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<TT, MODE, NB, PACKED, LNF, I8, SER, STG_>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    });
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a.M + TT - 1) / TT, SER ? 1 : a.sp.S, (a.N + NB * BN - 1) / (NB * BN));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = m.ctx->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;   // split-K CTAs of a tile = one cluster
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = a.sp.S;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = (a.sp.S > 1 && !SER) ? 2 : 1;
    const int nblk = (int)(cfg.gridDim.x * cfg.gridDim.y * cfg.gridDim.z);
    BASS_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TT, MODE, NB, PACKED, LNF, I8, SER, STG_>, *a.wm, *a.xm,
                                 (const __nv_bfloat16*)a.W, a.M, a.N, a.sp, e, a.xn,
                                 m.ctx->trace(nblk, BASS_TR_GEMM)));
}

template <int TT, bool SER = false>
static void launch_mode(bass_model& m, int mode, bool packed, bool xn, const LaunchArgs& a, const Epi& e) {
    if (a.sp.sx) {   // W8A8 (packed int8 weights): plain epilogues after the dequantization
        if (!packed || xn) throw Error(BASS_ERR_STATE, "int8 GEMM: packed weights, no folded LayerNorm");
        if ((mode == EPI_QKV || mode == EPI_GELU) && (a.N % 128 != 0 || (mode == EPI_GELU && !e.amax)))
            throw Error(BASS_ERR_STATE, "int8 QKV / GELU epilogues: N % 128 == 0 (GELU: with its amax buffer)");
        if (mode == EPI_RESID) launch_k<TT, EPI_RESID, true, 0, true, SER>(m, a, e);
        else if (mode == EPI_STORE) launch_k<TT, EPI_STORE, true, 0, true, SER>(m, a, e);
        else if (mode == EPI_QKV) launch_k<TT, EPI_QKV, true, 0, true, SER>(m, a, e);
        else launch_k<TT, EPI_GELU, true, 0, true, SER>(m, a, e);
        return;
    }
    if (!packed) {   // raw [N, K] pointers (bass_gemm): plain fp32 store
        if (mode != EPI_STORE || xn) throw Error(BASS_ERR_STATE, "tcgen05 GEMM: fused epilogues need packed weights");
        launch_k<TT, EPI_STORE, false, 0, false, SER>(m, a, e);
        return;
    }
    if (xn) {   // LayerNorm folded in: the two projections that follow a LayerNorm
        if (mode == EPI_QKV) launch_k<TT, EPI_QKV, true, 1, false, SER>(m, a, e);
        else if (mode == EPI_GELU) launch_k<TT, EPI_GELU, true, 1, false, SER>(m, a, e);
        else if (mode == EPI_STORE) launch_k<TT, EPI_STORE, true, 1, false, SER>(m, a, e);   // head (final LayerNorm)
        else throw Error(BASS_ERR_STATE, "tcgen05 GEMM: folded LayerNorm only for QKV / FC / head");
        return;
    }
    switch (mode) {
        case EPI_QKV: launch_k<TT, EPI_QKV, true, 0, false, SER>(m, a, e); break;
        case EPI_RESID:
            if constexpr (TT == 16 && !SER) {
                if (e.stats && a.lite) {   // every split in 4 stages (74 KB): starts beside the attention kernel
                    launch_k<16, EPI_RESID, true, 2, false, false, 4>(m, a, e);
                    break;
                }
            }
            if (e.stats) launch_k<TT, EPI_RESID, true, 2, false, SER>(m, a, e);   // emits the next LayerNorm's inputs
            else launch_k<TT, EPI_RESID, true, 0, false, SER>(m, a, e);
            break;
        case EPI_GELU: launch_k<TT, EPI_GELU, true, 0, false, SER>(m, a, e); break;
        default: launch_k<TT, EPI_STORE, true, 0, false, SER>(m, a, e); break;
    }
}

}  // namespace tc

bool tc_gemm_supported(const bass_model& m, int N, int K) {
    if (m.dtype == BASS_INT8) return K % 128 == 0 && N >= tc::BN;
    return m.dtype == BASS_BF16 && K % tc::BK == 0 && K >= tc::BK && N >= tc::BN;
}

void tc_gemm(bass_model& m, int mode, const void* X, const void* W, int M, int N, int K, const Epi& e, bool packed,
             const TcNorm* norm, const double* sx, const double* sw) {
    const bool i8 = sx != nullptr;
    using namespace tc;
    State& S = state(m);
    // token tile: smallest of 16/32/64/128/160/192/256 covering M; beyond
    // 256 rows, the tile in {256, 192, 160, 128} with the least padding over
    // the token groups (larger on ties): M = 1100 -> 7 x 160 (1120 rows)
    // instead of 5 x 256 (1280), 6-9 % faster per prefill GEMM.  Row bits do
    // not depend on the tile (tested for every tile size).
    int TT = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : M <= 160 ? 160 : M <= 192 ? 192 : 256;
    if (M > 256) {
        int best = 0x7fffffff;
        for (int t : {256, 192, 160, 128}) {
            const int padded = (M + t - 1) / t * t;
            if (padded < best) {
                best = padded;
                TT = t;
            }
        }
    }
    constexpr int NB = 1;
    static CUtensorMap dummy{};
    const CUtensorMap* wm = &dummy;
    if (!packed) {
        auto key = std::make_tuple(W, N, K);
        auto it = S.wmaps.find(key);
        if (it == S.wmaps.end()) it = S.wmaps.emplace(key, make_map(W, N, K, BN)).first;
        wm = &it->second;
    }
    XNorm xn{};
    if (norm) xn = XNorm{norm->stats, norm->c, norm->e, norm->kmean, norm->stat_tiles};   // X = bf16(x * g) (caller)
    auto xkey = std::make_tuple(X, M, i8 ? -K : K, TT);
    auto xit = S.xmaps.find(xkey);
    if (xit == S.xmaps.end()) xit = S.xmaps.emplace(xkey, make_map(X, M, K, TT, i8)).first;
    const CUtensorMap* xm = &xit->second;
    auto sk = std::make_pair(N, K);
    auto si = S.splits.find(sk);
    // int8: a k block is 128 elements, so the split rule sees K / 2 bf16-equivalent columns
    if (si == S.splits.end())
        si = S.splits.emplace(sk, choose_splits(m.ctx->sm_count, N, i8 ? K / 2 : K, i8 ? 16 : 32)).first;
    // one token group: every weight byte is read once (prefill re-reads it per group from L2)
    Split sp{si->second, i8 ? K / 128 : K / BK, nullptr, (packed && M <= TT) ? 1 : 0, sx, sw, m.dev_rows};
    // reduction loops and cluster size hold <= 8; every split owns >= 1 k block
    sp.S = std::max(1, std::min(std::min(MAX_S, sp.S), sp.k_iters));
    // prefill-sized M (more than two 128-row token groups): serial split-K —
    // the same K partition and summation order, so the rows' bits do not
    // change, without the split clusters (whose per-CTA tails dominate there)
    const bool ser = sp.S > 1 && sp.S <= 4 && M > 256 && packed;
    if (ser) {
        TT = sp.S <= 4 ? 128 : 64;   // S accumulators of TT columns in 512 TMEM columns
        // two splits, at least two 256-row token groups and no more padding
        // than 128-row groups: 256-token tiles (two 256-column accumulators,
        // one CTA per SM, a 4-stage 192 KB ring) read each weight tile half
        // as often from L2 (prefill QKV; prompt prefill 8 x 128 20.7 -> 20.3 ms)
        if (sp.S <= 2 && !i8 && M >= 512 && (M + 255) / 256 * 256 <= (M + 127) / 128 * 128) TT = 256;
        const auto xk2 = std::make_tuple(X, M, i8 ? -K : K, TT);
        auto x2 = S.xmaps.find(xk2);
        if (x2 == S.xmaps.end()) x2 = S.xmaps.emplace(xk2, make_map(X, M, K, TT, i8)).first;
        xm = &x2->second;
    }
    if (sp.S > 1 && !ser) {
        const size_t blocks = (size_t)((N + NB * BN - 1) / (NB * BN)) * ((M + TT - 1) / TT);
        sp.ws = (float*)S.ws.need(blocks * sp.S * TT * NB * BN * 4, m.ctx->stream);
    }
    // decode-sized residual projection whose splits hold <= 4 k blocks (the
    // draft's O-projection): a 4-stage ring (74 KB) fits beside the
    // attention kernel (146 KB), so its CTAs launch during the attention and
    // have their whole weight slice in shared memory when it ends (C2
    // 1.263 -> 1.254 ms/token; the same arithmetic, only the ring depth)
    const bool lite = TT == 16 && !ser && sp.S > 1 && sp.k_iters <= 4 * sp.S && mode == EPI_RESID && packed && !i8;
    LaunchArgs a{wm, xm, W, M, N, sp, xn, lite};
    const bool xnb = norm != nullptr;
    if (ser) {
        if (TT == 128) launch_mode<128, true>(m, mode, packed, xnb, a, e);
        else if (TT == 256) launch_mode<256, true>(m, mode, packed, xnb, a, e);
        else launch_mode<64, true>(m, mode, packed, xnb, a, e);
    } else switch (TT) {
        case 16: launch_mode<16>(m, mode, packed, xnb, a, e); break;
        case 32: launch_mode<32>(m, mode, packed, xnb, a, e); break;
        case 64: launch_mode<64>(m, mode, packed, xnb, a, e); break;
        case 128: launch_mode<128>(m, mode, packed, xnb, a, e); break;
        case 160: launch_mode<160>(m, mode, packed, xnb, a, e); break;
        case 192: launch_mode<192>(m, mode, packed, xnb, a, e); break;
        default: launch_mode<256>(m, mode, packed, xnb, a, e); break;
    }
    m.ctx->launches++;
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("tcgen05 gemm launch: ") + cudaGetErrorString(err));
}

void tc_set_split(bass_model& m, int N, int K, int splits) {
    tc::State& S = tc::state(m);
    const auto key = std::make_pair(N, K);
    if (splits > 0) S.splits[key] = splits;
    else S.splits.erase(key);
}

void tc_release(bass_model& m) {
    if (!m.tc_state) return;
    tc::State* s = static_cast<tc::State*>(m.tc_state);
    s->ws.release();
    delete s;
    m.tc_state = nullptr;
}

}  // namespace bass
