// Persistent stream-K tcgen05 weight-streaming GEMM for the ragged forward
// (sm_100a) — the batched draft / verify projections of BASS
// (ref:model.py:160-164 `_linear`, :214-245; dense layers stay batched,
// PAPER.md:142).
//
//   Y[m, n] = sum_k X[m, k] W[n, k]      (W output-major [N, K] bf16, X [M, K] bf16)
//
// Swap-AB: 128 weight rows are the UMMA M side, a token tile of TT rows the N
// side.  The weight stream is cut into units (128-row tile, 64-wide k block),
// k fastest; the grid is persistent (one CTA per SM) and CTA b owns the
// contiguous unit range [b U / G, (b+1) U / G) — every SM streams the same
// number of weight bytes, with no wave quantisation and no tail.  A tile cut
// by a range boundary is finished by its *owner* (the CTA holding k block 0,
// which reaches it last): the other pieces (each a CTA's first segment, done
// first) leave fp32 partials in an L2-resident workspace and raise a flag;
// the owner adds them in k order and runs the fused epilogue.  The partition
// depends only on (N, K, G), never on M, so a row's bits do not depend on the
// batch (batched == solo, verify == sequential decode).
//
// Warp roles (192 threads): warp 0 TMA producer (ring of W + X stages),
// warp 1 MMA issuer (accumulator double-buffered in TMEM so the next segment
// overlaps this one's epilogue), warps 2-5 epilogue (TMEM lane = weight row).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>

#include "runtime.h"

namespace bass {
namespace sk {

constexpr int BN = 128;          // weight rows per tile (UMMA M)
constexpr int BK = 64;           // k per unit (one 128-byte swizzle row of bf16)
constexpr int UK = 16;           // k per tcgen05.mma (16-bit inputs)
constexpr int THREADS = 192;
#ifndef SK_SMEM_KB
#define SK_SMEM_KB 100   // two CTAs per SM: the next kernel (PDL) prefetches its weights beside this one
#endif
constexpr int SMEM_BUDGET = SK_SMEM_KB * 1024;

template <int TT>
struct Cfg {
    static constexpr int W_BYTES = BN * BK * 2;
    static constexpr int X_BYTES = TT * BK * 2;
    static constexpr int STAGE = W_BYTES + X_BYTES;
    // TT <= 128: <= 100 KB smem and <= 256 TMEM columns, so two CTAs share an
    // SM without blocking each other's TMEM allocation (the owner of a split
    // tile spins on other CTAs of the grid); larger tiles take a whole SM
    static constexpr int BUDGET = TT <= 128 ? SMEM_BUDGET : 200 * 1024;
    static constexpr int STAGES_RAW = BUDGET / STAGE;
    static constexpr int STAGES = STAGES_RAW > 16 ? 16 : STAGES_RAW;
    static constexpr int NBAR = 2 * STAGES + 4;   // full[S] empty[S] acc_full[2] acc_empty[2]
    static constexpr int SMEM = STAGES * STAGE + 1024 + NBAR * 8 + 16;
    static constexpr int TMEM_COLS = 2 * TT <= 32 ? 32 : 2 * TT <= 64 ? 64 : 2 * TT <= 128 ? 128 : 2 * TT <= 256 ? 256 : 512;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
}
// 1-D bulk copy global -> shared (packed weight tiles: one contiguous 16 KB block)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint32_t dst, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
// K-major, 128-byte swizzle, 8-row groups 1024 B apart, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
// bf16 x bf16 -> f32, K-major A and B, M = 128, N = tt
__host__ __device__ constexpr uint32_t idesc(int tt) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(tt >> 3) << 17) | ((uint32_t)(BN >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
            dtmem),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {
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
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Unit partition: CTA b owns [start(b), start(b+1)).
struct Part {
    int64_t U;      // units = n_tiles * k_iters
    int G, k_iters;
    __host__ __device__ int64_t start(int b) const { return (int64_t)b * U / G; }
    __device__ int cta_of(int64_t u) const {
        int b = (int)((u * G) / U);
        while (b + 1 < G && start(b + 1) <= u) ++b;
        while (b > 0 && start(b) > u) --b;
        return b;
    }
};

// One segment = the part of one (token group, weight tile) inside this CTA's range.
struct Seg {
    int g, tile, kb0, kb1;   // k blocks [kb0, kb1)
};
// Walks this CTA's segments (identically in every role).
struct SegIter {
    Part p;
    int groups, b;
    int64_t u0, u1, u;
    int g;
    __device__ SegIter(const Part& p_, int groups_, int b_) : p(p_), groups(groups_), b(b_) {
        u0 = p.start(b);
        u1 = p.start(b + 1);
        u = u0;
        g = 0;
    }
    __device__ bool next(Seg& s) {
        if (u >= u1) {
            if (++g >= groups || u0 >= u1) return false;
            u = u0;
        }
        s.g = g;
        s.tile = (int)(u / p.k_iters);
        s.kb0 = (int)(u - (int64_t)s.tile * p.k_iters);
        const int64_t tile_end = (int64_t)(s.tile + 1) * p.k_iters;
        const int64_t e = u1 < tile_end ? u1 : tile_end;
        s.kb1 = (int)(e - (int64_t)s.tile * p.k_iters);
        u = e;
        return true;
    }
};

// PACKED: W in the packed tile layout (common.cuh packed_index) -> one 1-D
// bulk copy per unit; otherwise W [N, K] row-major through the 2-D map `tw`.
template <int TT, int MODE, bool PACKED>
__global__ void __launch_bounds__(THREADS, 1) gemm_sk_kernel(const __grid_constant__ CUtensorMap tw,
                                                             const __grid_constant__ CUtensorMap tx,
                                                             const __nv_bfloat16* __restrict__ wpk, int M, int N,
                                                             Part part, int groups, float* __restrict__ ws,
                                                             int* __restrict__ flags, int epoch, Epi e,
                                                             TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    using C = Cfg<TT>;
    constexpr int ST = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = su32(smem_raw);
    const uint32_t base = (raw + 1023) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * C::STAGE);
    uint64_t* full = bars;
    uint64_t* empty = bars + ST;
    uint64_t* acc_full = bars + 2 * ST;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::NBAR; ++i) mbar_init(su32(&bars[i]), 1);
        for (int i = 0; i < 2; ++i) mbar_init(su32(&acc_empty[i]), 4);   // one arrival per epilogue warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (!PACKED) asm volatile("prefetch.tensormap [%0];" ::"l"(&tw) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tx) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(C::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            // weights do not depend on the previous kernel: fill the ring with
            // W tiles first, then wait for the producer of X (griddepcontrol)
            SegIter it(part, groups, b);
            Seg s;
            int i = 0;
            bool waited = false;
            int pending[ST];   // stages whose X load is deferred until griddepcontrol.wait
            int pk[ST], pg[ST];
            int npend = 0;
            while (it.next(s)) {
                for (int kb = s.kb0; kb < s.kb1; ++kb, ++i) {
                    const int st = i % ST;
                    if (i >= ST) {
                        if (!waited) {
                            asm volatile("griddepcontrol.wait;" ::: "memory");
                            for (int q = 0; q < npend; ++q)
                                tma_2d(&tx, base + pending[q] * C::STAGE + C::W_BYTES, su32(&full[pending[q]]), pk[q],
                                       pg[q]);
                            waited = true;
                        }
                        mbar_wait(su32(&empty[st]), ((i / ST) - 1) & 1);
                    }
                    const uint32_t stg = base + st * C::STAGE;
                    mbar_expect_tx(su32(&full[st]), C::STAGE);
                    if constexpr (PACKED)
                        bulk_g2s(stg, wpk + ((int64_t)s.tile * part.k_iters + kb) * (BN * BK), C::W_BYTES,
                                 su32(&full[st]));
                    else
                        tma_2d(&tw, stg, su32(&full[st]), kb * BK, s.tile * BN);
                    if (waited) {
                        tma_2d(&tx, stg + C::W_BYTES, su32(&full[st]), kb * BK, s.g * TT);
                    } else {
                        pending[npend] = st;
                        pk[npend] = kb * BK;
                        pg[npend] = s.g * TT;
                        ++npend;
                    }
                }
            }
            if (!waited) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                for (int q = 0; q < npend; ++q)
                    tma_2d(&tx, base + pending[q] * C::STAGE + C::W_BYTES, su32(&full[pending[q]]), pk[q], pg[q]);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t ID = idesc(TT);
            SegIter it(part, groups, b);
            Seg s;
            int i = 0, j = 0;
            while (it.next(s)) {
                const int buf = j & 1;
                if (j >= 2) mbar_wait(su32(&acc_empty[buf]), ((j >> 1) - 1) & 1);
                fence_after();
                const uint32_t d = tmem + buf * TT;
                for (int kb = s.kb0; kb < s.kb1; ++kb, ++i) {
                    const int st = i % ST;
                    mbar_wait(su32(&full[st]), (i / ST) & 1);
                    fence_after();
                    const uint32_t stg = base + st * C::STAGE;
                    const uint64_t a = sdesc(stg), bd = sdesc(stg + C::W_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / UK; ++kk)   // +32 bytes per UMMA_K step inside the swizzle row
                        umma(d, a + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), ID,
                             (kb > s.kb0 || kk > 0) ? 1u : 0u);
                    commit(su32(&empty[st]));
                }
                commit(su32(&acc_full[buf]));
                ++j;
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 2-5): TMEM lane = weight row, columns = tokens
        asm volatile("griddepcontrol.wait;" ::: "memory");   // previous kernel's writes visible
        const int wq = warp & 3;
        const int nn = wq * 32 + lane;                        // row within the tile
        const int tid = threadIdx.x - 64;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        SegIter it(part, groups, b);
        Seg s;
        int j = 0;
        while (it.next(s)) {
            const int buf = j & 1;
            const uint32_t tacc = tmem + lane_off + buf * TT;
            const int n = s.tile * BN + nn, m0 = s.g * TT;
            const int rows = min(TT, M - m0);
            const bool whole = s.kb0 == 0 && s.kb1 == part.k_iters;
            // workspace slot of CTA c for group g: [BN rows][TT tokens] fp32, row-contiguous
            auto slot = [&](int c) { return ws + (((int64_t)s.g * part.G + c) * BN + nn) * TT; };
            if (s.kb0 != 0) {
                // non-owner piece (this CTA's first segment): partial -> workspace, raise the flag
                mbar_wait(su32(&acc_full[buf]), (j >> 1) & 1);
                fence_after();
                float4* dst = reinterpret_cast<float4*>(slot(b));
#pragma unroll
                for (int c0 = 0; c0 < TT; c0 += 16) {
                    if (c0 < rows) {
                        float v[16];
                        ld16(tacc + c0, v);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            __stcg(dst + c0 / 4 + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(su32(&acc_empty[buf]));
                __threadfence();
                epi_bar();
                if (tid == 0) st_release(flags + (int64_t)s.g * part.G + b, epoch);
            } else {
                // owner (or whole tile).  The other pieces were finished early by
                // the next CTAs: sum them (k order) into registers while this
                // segment is still streaming, then add the accumulator and run
                // the fused epilogue.
                int npieces = 1;
                constexpr int PS = TT < 128 ? TT : 128;   // tokens whose partial sums are prefetched
                float4 ps[PS / 4];
                if (!whole) {
                    const int64_t last_u = (int64_t)(s.tile + 1) * part.k_iters - 1;
                    npieces = part.cta_of(last_u) - b + 1;
                    if (tid == 0)
                        for (int p = 1; p < npieces; ++p)
                            while (ld_acquire(flags + (int64_t)s.g * part.G + b + p) != epoch) {
                            }
                    epi_bar();
                    for (int p = 1; p < npieces; ++p) {
                        const float4* src = reinterpret_cast<const float4*>(slot(b + p));
#pragma unroll
                        for (int q = 0; q < PS / 4; ++q) {
                            const float4 w = 4 * q < rows ? __ldcg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                            if (p == 1) {
                                ps[q] = w;
                            } else {
                                ps[q].x += w.x;
                                ps[q].y += w.y;
                                ps[q].z += w.z;
                                ps[q].w += w.w;
                            }
                        }
                    }
                }
                mbar_wait(su32(&acc_full[buf]), (j >> 1) & 1);
                fence_after();
#pragma unroll
                for (int c0 = 0; c0 < TT; c0 += 16) {
                    if (c0 < rows) {
                        float v[16];
                        ld16(tacc + c0, v);
                        if (npieces > 1) {
                            if (c0 < PS) {
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const float4 a = ps[(c0 < PS ? c0 : 0) / 4 + q];
                                    v[4 * q] += a.x;
                                    v[4 * q + 1] += a.y;
                                    v[4 * q + 2] += a.z;
                                    v[4 * q + 3] += a.w;
                                }
                            } else {   // tokens beyond the prefetched range: same k order, read now
                                float t[16];
#pragma unroll
                                for (int q = 0; q < 16; ++q) t[q] = 0.f;
                                for (int p = 1; p < npieces; ++p) {
                                    const float4* src = reinterpret_cast<const float4*>(slot(b + p)) + c0 / 4;
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        const float4 w = __ldcg(src + q);
                                        if (p == 1) {
                                            t[4 * q] = w.x; t[4 * q + 1] = w.y; t[4 * q + 2] = w.z; t[4 * q + 3] = w.w;
                                        } else {
                                            t[4 * q] += w.x; t[4 * q + 1] += w.y; t[4 * q + 2] += w.z; t[4 * q + 3] += w.w;
                                        }
                                    }
                                }
#pragma unroll
                                for (int q = 0; q < 16; ++q) v[q] += t[q];
                            }
                        }
                        if (n < N) {
#pragma unroll
                            for (int q = 0; q < 16; ++q)
                                if (c0 + q < rows) epilogue<MODE, __nv_bfloat16>(e, m0 + c0 + q, n, N, v[q]);
                        }
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(su32(&acc_empty[buf]));
            }
            ++j;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS)
                     : "memory");
    trace_end(tr, t_start);
}

// ------------------------------------------------------------------ host
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

// 2D bf16 row-major [rows, cols] map with a box of {64 cols, box_rows}, 128B swizzle
static CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

struct State {
    std::map<std::tuple<const void*, int, int>, CUtensorMap> wmaps;
    std::map<std::tuple<const void*, int, int, int>, CUtensorMap> xmaps;   // (X, M, K, TT)
    DevBuf ws, flags;
    size_t flags_n = 0;
    int epoch = 0;
};

static State& state(bass_model& m) {
    if (!m.sk_state) m.sk_state = new State();
    return *static_cast<State*>(m.sk_state);
}

struct Args {
    const CUtensorMap* wm;
    const CUtensorMap* xm;
    const void* W;
    int M, N;
    Part p;
    int groups;
    float* ws;
    int* flags;
    int epoch;
};

template <int TT, int MODE, bool PACKED>
static void launch(bass_model& m, const Args& a, const Epi& e) {
    using C = Cfg<TT>;
    static bool attr = false;
    if (!attr) {
        BASS_CUDA(cudaFuncSetAttribute(gemm_sk_kernel<TT, MODE, PACKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM));
        attr = true;
    }
    BASS_CUDA(launch_pdl(gemm_sk_kernel<TT, MODE, PACKED>, dim3(a.p.G), dim3(THREADS), (size_t)C::SMEM, m.ctx->stream,
                         *a.wm, *a.xm, (const __nv_bfloat16*)a.W, a.M, a.N, a.p, a.groups, a.ws, a.flags, a.epoch, e,
                         m.ctx->trace(a.p.G, BASS_TR_GEMM)));
}

// packed (model) weights: every fused epilogue; raw [N, K] pointers: plain store
template <int TT>
static void launch_mode(bass_model& m, int mode, bool packed, const Args& a, const Epi& e) {
    if (!packed) {
        if (mode != EPI_STORE) throw Error(BASS_ERR_STATE, "stream-K GEMM: fused epilogues need packed weights");
        launch<TT, EPI_STORE, false>(m, a, e);
        return;
    }
    switch (mode) {
        case EPI_QKV: launch<TT, EPI_QKV, true>(m, a, e); break;
        case EPI_RESID: launch<TT, EPI_RESID, true>(m, a, e); break;
        case EPI_GELU: launch<TT, EPI_GELU, true>(m, a, e); break;
        default: launch<TT, EPI_STORE, true>(m, a, e); break;
    }
}

}  // namespace sk

void sk_gemm(bass_model& m, int mode, const void* X, const void* W, int M, int N, int K, const Epi& e, bool packed) {
    using namespace sk;
    State& S = state(m);
    // token tile: smallest multiple of 32 (16 for tiny blocks) covering M, groups of 256 beyond
    const int TT = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 96 ? 96 : M <= 128 ? 128 : M <= 160 ? 160
                 : M <= 192 ? 192 : 256;
    const int groups = (M + TT - 1) / TT;
    static CUtensorMap dummy{};
    const CUtensorMap* wm = &dummy;
    if (!packed) {
        auto key = std::make_tuple(W, N, K);
        auto it = S.wmaps.find(key);
        if (it == S.wmaps.end()) it = S.wmaps.emplace(key, make_map(W, N, K, BN)).first;
        wm = &it->second;
    }
    auto xkey = std::make_tuple(X, M, K, TT);
    auto xit = S.xmaps.find(xkey);
    if (xit == S.xmaps.end()) xit = S.xmaps.emplace(xkey, make_map(X, M, K, TT)).first;
    Part p;
    p.k_iters = K / BK;
    p.U = (int64_t)((N + BN - 1) / BN) * p.k_iters;
    // a function of (N, K) only: one CTA per SM, but at least `min_units` k blocks each
    static const int min_units = getenv("BASS_SK_MIN_UNITS") ? std::max(1, atoi(getenv("BASS_SK_MIN_UNITS"))) : 1;
    p.G = (int)std::max<int64_t>(1, std::min<int64_t>(m.ctx->sm_count, p.U / min_units));
    float* ws = (float*)S.ws.need((size_t)groups * p.G * TT * BN * 4, m.ctx->stream);
    const size_t nflags = (size_t)groups * p.G;
    if (nflags > S.flags_n) {
        int* f = (int*)S.flags.need(nflags * 4, m.ctx->stream);
        BASS_CUDA(cudaMemsetAsync(f, 0, nflags * 4, m.ctx->stream));
        S.flags_n = nflags;
        S.epoch = 0;
    }
    Args a{wm, &xit->second, W, M, N, p, groups, ws, (int*)S.flags.p, ++S.epoch};
    switch (TT) {
        case 16: launch_mode<16>(m, mode, packed, a, e); break;
        case 32: launch_mode<32>(m, mode, packed, a, e); break;
        case 64: launch_mode<64>(m, mode, packed, a, e); break;
        case 96: launch_mode<96>(m, mode, packed, a, e); break;
        case 128: launch_mode<128>(m, mode, packed, a, e); break;
        case 160: launch_mode<160>(m, mode, packed, a, e); break;
        case 192: launch_mode<192>(m, mode, packed, a, e); break;
        default: launch_mode<256>(m, mode, packed, a, e); break;
    }
    m.ctx->launches++;
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("stream-K gemm launch: ") + cudaGetErrorString(err));
}

void sk_release(bass_model& m) {
    if (!m.sk_state) return;
    sk::State* s = static_cast<sk::State*>(m.sk_state);
    s->ws.release();
    s->flags.release();
    delete s;
    m.sk_state = nullptr;
}

}  // namespace bass
