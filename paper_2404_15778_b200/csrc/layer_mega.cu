// Persistent "layer megakernel" (sm_100a): one launch runs the dense part of
// a transformer layer of the BASS forward (ref:model.py:214-245) as a chain
// of phases —
//     O-proj (+ residual)  ->  LN2  ->  FC (+ exact GELU)  ->  proj (+ residual)
//     ->  LN1 of the next layer  ->  QKV of the next layer (+ KV append)
// (or any prefix / suffix of it: first layer [LN1, QKV], last layer
// [O, LN2, FC, proj, LN_f(gather), head]) — with a grid-wide barrier between
// phases.  Attention stays a separate launch (attn_stream.cu).
//
// Why: a verify / draft layer is a handful of weight streams (42-170 MB each
// at 7.8B scale, 8-34 MB for the draft) separated by tiny LayerNorms.  As
// separate kernels every boundary drains the HBM pipe (launch, prologue,
// first-byte latency, split-K tail); profiles/r1_trace_* showed a layer at
// ~2x its weight-streaming time.  Here the weight stream never stops: the
// producer warp keeps filling the shared-memory ring with the NEXT phase's
// weights (which depend on nothing) while the current phase finishes and the
// grid barrier resolves; only the activation (X) loads wait for the barrier.
//
// GEMM phases are stream-K over units (128 weight rows x 64 k) with a static
// partition that depends only on (N, K, grid): every CTA streams the same
// number of weight bytes; a tile cut by a range boundary is finished by its
// owner (k block 0), which adds the other pieces' fp32 partials in k order
// (deterministic; a row's bits do not depend on the batch).  All CTAs are
// resident for the whole launch (one per SM), which the owner waits and the
// grid barriers rely on.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (TMEM
// accumulators double-buffered across segments and phases), warps 2-5
// epilogue / LayerNorm / grid barrier.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>

#include "runtime.h"
#include "tcgen05.cuh"

namespace bass {
namespace mg {

using namespace t5;

constexpr int BN = 128, BK = 64, UK = 16, THREADS = 192;
constexpr int SMEM_BUDGET = 200 * 1024;
constexpr int LN_V4 = 16;   // d <= 4 * 128 * 16 = 8192

enum { PH_GEMM = 0, PH_LN = 1 };

// One phase of a launch (device array, built on the host per forward).
struct alignas(64) Phase {
    CUtensorMap tx;                  // GEMM: X [M, K] bf16, box {64, TT}
    const __nv_bfloat16* w;          // GEMM: packed weights [Npad, K]
    Epi e;                           // GEMM: fused epilogue
    int64_t U;                       // GEMM: units = n_tiles * k_iters
    int type, mode, M, N, K, k_iters, groups;
    // LN: out[r] = LN(x[gather ? gather[r] : r]) * g + b, r < rows
    const float* x;
    const int32_t* gather;
    const float* g;
    const float* b;
    __nv_bfloat16* out;
    int rows, d;
};

template <int TT>
struct Cfg {
    static constexpr int W_BYTES = BN * BK * 2;
    static constexpr int X_BYTES = TT * BK * 2;
    static constexpr int STAGE = W_BYTES + X_BYTES;
    static constexpr int STAGES_RAW = SMEM_BUDGET / STAGE;
    static constexpr int STAGES = STAGES_RAW > 12 ? 12 : STAGES_RAW;
    // full[S] empty[S] acc_full[2] acc_empty[2] xready
    static constexpr int NBAR = 2 * STAGES + 5;
    static constexpr int SMEM = STAGES * STAGE + 1024 + NBAR * 8 + 16 + 64 * 4 + 32 * 8;
    static constexpr int TMEM_COLS = 2 * TT <= 32 ? 32 : 2 * TT <= 64 ? 64 : 2 * TT <= 128 ? 128 : 2 * TT <= 256 ? 256 : 512;
};

// stream-K partition of one GEMM phase: CTA b owns units [start(b), start(b+1))
struct Part {
    int64_t U;
    int G, k_iters;
    __device__ int64_t start(int b) const { return (int64_t)b * U / G; }
    __device__ int cta_of(int64_t u) const {
        int b = (int)((u * G) / U);
        while (b + 1 < G && start(b + 1) <= u) ++b;
        while (b > 0 && start(b) > u) --b;
        return b;
    }
};
struct Seg {
    int g, tile, kb0, kb1;
};
struct SegIter {
    Part p;
    int groups;
    int64_t u0, u1, u;
    int g;
    __device__ SegIter(const Part& p_, int groups_, int b) : p(p_), groups(groups_) {
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

// grid-wide barrier (one thread per CTA, after a CTA-level barrier): the
// arrival counter only grows — barrier number `gen` completes when it reaches
// (gen + 1) * G — so one release-add per CTA and acquire polling suffice
// (no reset, no last-arriver flag round trip).
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned G, unsigned gen) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = (gen + 1) * G;
    while ((int)(ld_acquire_u(bar) - target) < 0) {
    }
}

template <int TT>
__global__ void __launch_bounds__(THREADS, 1) mega_kernel(const Phase* __restrict__ phases, int n_phases,
                                                           float* __restrict__ ws, int* __restrict__ flags, int epoch,
                                                           unsigned* __restrict__ gbar, unsigned gen0, TraceArg tr) {
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
    uint64_t* xready = acc_empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
    float* red = reinterpret_cast<float*>(tmem_slot + 4);   // LN block reductions [2][4]
    unsigned long long* t_ready = reinterpret_cast<unsigned long long*>(red + 8);   // [16] producer X-ready times
    unsigned long long* t_wait = t_ready + 16;                                        // [16] producer starts waiting
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x, G = gridDim.x;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::NBAR; ++i) mbar_init(su32(&bars[i]), 1);
        for (int i = 0; i < 2; ++i) mbar_init(su32(&acc_empty[i]), 4);   // one arrival per epilogue warp
        for (int i = 0; i < 32; ++i) t_ready[i] = 0ull;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(su32(tmem_slot), C::TMEM_COLS);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {   // ---------------- producer
            int i = 0, nx = 0;   // ring slot counter; X-ready signals consumed
            for (int p = 0; p < n_phases; ++p) {
                const Phase* ph = phases + p;
                if (ph->type != PH_GEMM) continue;
                asm volatile("prefetch.tensormap [%0];" ::"l"(&ph->tx) : "memory");
                const Part part{ph->U, G, ph->k_iters};
                SegIter it(part, ph->groups, b);
                Seg s;
                bool ready = false;
                int pend_st[16], pend_kb[16], pend_g[16], npend = 0;
                // X of this phase may be read once the previous phase is complete
                // everywhere: the previous kernel (p == 0) or this launch's grid barrier
                auto make_ready = [&]() {
                    if (tr.buf) t_wait[p] = gtimer();
                    if (p == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
                    else mbar_wait(su32(xready), (nx++) & 1);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    for (int q = 0; q < npend; ++q)
                        tma_2d(&ph->tx, base + pend_st[q] * C::STAGE + C::W_BYTES, su32(&full[pend_st[q]]),
                               pend_kb[q] * BK, pend_g[q] * TT);
                    npend = 0;
                    ready = true;
                    if (tr.buf) t_ready[p] = gtimer();
                };
                while (it.next(s)) {
                    for (int kb = s.kb0; kb < s.kb1; ++kb, ++i) {
                        const int st = i % ST;
                        if (i >= ST) {
                            if (!ready && npend >= ST) make_ready();   // ring full of this phase's stages
                            mbar_wait(su32(&empty[st]), ((i / ST) - 1) & 1);
                        }
                        const uint32_t stg = base + st * C::STAGE;
                        mbar_expect_tx(su32(&full[st]), C::STAGE);
                        bulk_g2s(stg, ph->w + ((int64_t)s.tile * ph->k_iters + kb) * (BN * BK), C::W_BYTES,
                                 su32(&full[st]));
                        if (ready) {
                            tma_2d(&ph->tx, stg + C::W_BYTES, su32(&full[st]), kb * BK, s.g * TT);
                        } else {
                            pend_st[npend] = st;
                            pend_kb[npend] = kb;
                            pend_g[npend] = s.g;
                            ++npend;
                        }
                    }
                }
                if (!ready) make_ready();
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t ID = idesc_bf16(TT);
            int i = 0, j = 0;
            for (int p = 0; p < n_phases; ++p) {
                const Phase* ph = phases + p;
                if (ph->type != PH_GEMM) continue;
                const Part part{ph->U, G, ph->k_iters};
                SegIter it(part, ph->groups, b);
                Seg s;
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
                        const uint64_t a = sdesc_k128(stg), bd = sdesc_k128(stg + C::W_BYTES);
#pragma unroll
                        for (int kk = 0; kk < BK / UK; ++kk)
                            umma(d, a + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), ID, (kb > s.kb0 || kk > 0) ? 1u : 0u);
                        commit(su32(&empty[st]));
                    }
                    commit(su32(&acc_full[buf]));
                    ++j;
                }
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue / LayerNorm / barriers (warps 2-5)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int wq = warp & 3;
        const int nn = wq * 32 + lane;
        const int tid = threadIdx.x - 64;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        int j = 0;
        unsigned gen = gen0;
        for (int p = 0; p < n_phases; ++p) {
            const Phase* ph = phases + p;
            const int ep = epoch + p;
            if (ph->type == PH_GEMM) {
                const Part part{ph->U, G, ph->k_iters};
                const int M = ph->M, N = ph->N, MODE = ph->mode;
                const Epi e = ph->e;
                SegIter it(part, ph->groups, b);
                Seg s;
                while (it.next(s)) {
                    const int buf = j & 1;
                    const uint32_t tacc = tmem + lane_off + buf * TT;
                    const int n = s.tile * BN + nn, m0 = s.g * TT;
                    const int rows = min(TT, M - m0);
                    const bool whole = s.kb0 == 0 && s.kb1 == part.k_iters;
                    auto slot = [&](int c) { return ws + (((int64_t)s.g * G + c) * BN + nn) * TT; };
                    if (s.kb0 != 0) {
                        // non-owner piece (this CTA's first segment): partial -> workspace, flag
                        mbar_wait(su32(&acc_full[buf]), (j >> 1) & 1);
                        fence_after();
                        float4* dst = reinterpret_cast<float4*>(slot(b));
#pragma unroll
                        for (int c0 = 0; c0 < TT; c0 += 16) {
                            if (c0 < rows) {
                                float v[16];
                                tmem_ld16(tacc + c0, v);
#pragma unroll
                                for (int q = 0; q < 4; ++q)
                                    __stcg(dst + c0 / 4 + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                            }
                        }
                        fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(su32(&acc_empty[buf]));
                        __threadfence();
                        named_bar(1, 128);
                        if (tid == 0) st_release(flags + (int64_t)s.g * G + b, ep);
                    } else {
                        // owner (or whole tile): other pieces summed in k order into
                        // registers while this segment streams, then the epilogue
                        int npieces = 1;
                        constexpr int PS = TT < 128 ? TT : 128;
                        float4 ps[PS / 4];
                        if (!whole) {
                            npieces = part.cta_of((int64_t)(s.tile + 1) * part.k_iters - 1) - b + 1;
                            if (tid == 0)
                                for (int q = 1; q < npieces; ++q)
                                    while (ld_acquire(flags + (int64_t)s.g * G + b + q) != ep) {
                                    }
                            named_bar(1, 128);
                            for (int q = 1; q < npieces; ++q) {
                                const float4* src = reinterpret_cast<const float4*>(slot(b + q));
#pragma unroll
                                for (int u = 0; u < PS / 4; ++u) {
                                    const float4 w = 4 * u < rows ? __ldcg(src + u) : make_float4(0.f, 0.f, 0.f, 0.f);
                                    if (q == 1) {
                                        ps[u] = w;
                                    } else {
                                        ps[u].x += w.x;
                                        ps[u].y += w.y;
                                        ps[u].z += w.z;
                                        ps[u].w += w.w;
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
                                tmem_ld16(tacc + c0, v);
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
                                    } else {
                                        float t[16];
#pragma unroll
                                        for (int q = 0; q < 16; ++q) t[q] = 0.f;
                                        for (int q = 1; q < npieces; ++q) {
                                            const float4* src = reinterpret_cast<const float4*>(slot(b + q)) + c0 / 4;
#pragma unroll
                                            for (int u = 0; u < 4; ++u) {
                                                const float4 w = __ldcg(src + u);
                                                t[4 * u] += w.x;
                                                t[4 * u + 1] += w.y;
                                                t[4 * u + 2] += w.z;
                                                t[4 * u + 3] += w.w;
                                            }
                                        }
#pragma unroll
                                        for (int q = 0; q < 16; ++q) v[q] += t[q];
                                    }
                                }
                                if (n < N) {
#pragma unroll
                                    for (int q = 0; q < 16; ++q) {
                                        if (c0 + q < rows) {
                                            const int m = m0 + c0 + q;
                                            switch (MODE) {
                                                case EPI_QKV: epilogue<EPI_QKV, __nv_bfloat16>(e, m, n, N, v[q]); break;
                                                case EPI_RESID: epilogue<EPI_RESID, __nv_bfloat16>(e, m, n, N, v[q]); break;
                                                case EPI_GELU: epilogue<EPI_GELU, __nv_bfloat16>(e, m, n, N, v[q]); break;
                                                default: epilogue<EPI_STORE, __nv_bfloat16>(e, m, n, N, v[q]); break;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                        fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(su32(&acc_empty[buf]));
                    }
                    ++j;
                }
            } else {
                // LayerNorm rows b, b + G, ... (fp32 stats, population variance)
                const int d = ph->d, n4 = d >> 2;
                for (int r = b; r < ph->rows; r += G) {
                    const int src = ph->gather ? ph->gather[r] : r;
                    const float4* xr = reinterpret_cast<const float4*>(ph->x + (int64_t)src * d);
                    float4 v[LN_V4];
                    float sum = 0.f;
#pragma unroll
                    for (int i = 0; i < LN_V4; ++i) {
                        const int c = tid + i * 128;
                        v[i] = c < n4 ? __ldcg(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                        sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    if (lane == 0) red[wq] = sum;
                    named_bar(1, 128);
                    const float mean = ((red[0] + red[1]) + (red[2] + red[3])) / (float)d;
                    float sq = 0.f;
#pragma unroll
                    for (int i = 0; i < LN_V4; ++i) {
                        const int c = tid + i * 128;
                        if (c < n4) {
                            const float a = v[i].x - mean, bb = v[i].y - mean, cc = v[i].z - mean, dd = v[i].w - mean;
                            sq += (a * a + bb * bb) + (cc * cc + dd * dd);
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                    if (lane == 0) red[4 + wq] = sq;
                    named_bar(1, 128);
                    const float var = ((red[4] + red[5]) + (red[6] + red[7])) / (float)d;
                    const float rstd = 1.0f / sqrtf(var + 1e-5f);
                    const float4* g4 = reinterpret_cast<const float4*>(ph->g);
                    const float4* b4 = reinterpret_cast<const float4*>(ph->b);
#pragma unroll
                    for (int i = 0; i < LN_V4; ++i) {
                        const int c = tid + i * 128;
                        if (c < n4) {
                            const float4 gg = g4[c], bv = b4[c];
                            __nv_bfloat162 lo = __floats2bfloat162_rn((v[i].x - mean) * rstd * gg.x + bv.x,
                                                                      (v[i].y - mean) * rstd * gg.y + bv.y);
                            __nv_bfloat162 hi = __floats2bfloat162_rn((v[i].z - mean) * rstd * gg.z + bv.z,
                                                                      (v[i].w - mean) * rstd * gg.w + bv.w);
                            uint2 pk;
                            pk.x = *reinterpret_cast<uint32_t*>(&lo);
                            pk.y = *reinterpret_cast<uint32_t*>(&hi);
                            *reinterpret_cast<uint2*>(ph->out + (int64_t)r * d + 4 * c) = pk;
                        }
                    }
                    named_bar(1, 128);   // red[] reused by the next row
                }
            }
            const unsigned long long t_done = tr.buf ? gtimer() : 0ull;
            if (p + 1 < n_phases) {
                // phase boundary: every CTA's writes of this phase are visible
                // (to generic loads and to the TMA reads of the next GEMM phase):
                // CTA barrier, then tid 0's gpu-scope release covers them
                fence_proxy_async_global();
                named_bar(1, 128);
                if (tid == 0) grid_sync(gbar, (unsigned)G, gen);
                ++gen;
                named_bar(1, 128);
                if (tid == 0 && phases[p + 1].type == PH_GEMM) mbar_arrive(su32(xready));
            }
            if (tr.buf && tid == 0) {   // per-phase record after the kernel record: {done, released, x_ready, tag}
                unsigned long long* rec = tr.buf + 4 * (tr.base + (long long)(p + 1) * G + b);
                rec[0] = t_done;
                rec[1] = gtimer();
                rec[2] = 0;
                rec[3] = (unsigned long long)(tr.tag | (1 << 3)) | ((unsigned long long)p << 40);
                // second record of the phase: {producer wait start, 0, 0, tag | p}
                unsigned long long* rec2 = tr.buf + 4 * (tr.base + (long long)(n_phases + 1 + p) * G + b);
                rec2[0] = 0;
                rec2[1] = 0;
                rec2[2] = 0;
                rec2[3] = (unsigned long long)(tr.tag | (1 << 3)) | ((unsigned long long)p << 40) | (1ull << 62);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
    if (tr.buf && threadIdx.x == 0)
        for (int p = 0; p < n_phases; ++p) {
            tr.buf[4 * (tr.base + (long long)(p + 1) * G + b) + 2] = t_ready[p];
            tr.buf[4 * (tr.base + (long long)(n_phases + 1 + p) * G + b)] = t_wait[p];
        }
    trace_end(tr, t_start);
}

// ------------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap x_map(const void* ptr, int64_t rows, int64_t cols, int box_rows) {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        BASS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeFn)p;
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled (mega) failed");
    return m;
}

struct State {
    DevBuf phases, ws, flags, gbar;
    size_t flags_n = 0;
    int epoch = 0;
    unsigned gen = 0;
    std::map<std::tuple<const void*, int, int, int>, CUtensorMap> xmaps;
    // prepared launches of the current forward
    struct L {
        size_t off;
        int n, TT, epoch;
        unsigned gen;
    };
    std::vector<L> launches;
    float* ws_p = nullptr;
    int G = 0;
};

static State& state(bass_model& m) {
    if (!m.mega_state) m.mega_state = new State();
    return *static_cast<State*>(m.mega_state);
}

template <int TT>
static void launch(bass_model& m, int G, const Phase* dph, int n, float* ws, int* flags, int epoch, unsigned* gbar,
                   unsigned gen) {
    using C = Cfg<TT>;
    static bool attr = false;
    if (!attr) {
        BASS_CUDA(cudaFuncSetAttribute(mega_kernel<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        attr = true;
    }
    BASS_CUDA(launch_pdl(mega_kernel<TT>, dim3(G), dim3(THREADS), (size_t)C::SMEM, m.ctx->stream, dph, n, ws, flags,
                         epoch, gbar, gen, m.ctx->trace(G * (2 * n + 1), BASS_TR_MEGA)));
}

}  // namespace mg

// bf16 packed weights, d <= 8192; opt-in with BASS_MEGA=1 (measured slower
// than one kernel per GEMM so far: profiles/r1_trace_mega.txt — grid barriers
// ~3 us each and skewed phase starts dominate at draft scale)
bool mega_supported(const bass_model& m) {
    static const bool on = getenv("BASS_MEGA") && atoi(getenv("BASS_MEGA")) == 1;
    return on && m.packed && m.g.d_model % 64 == 0 && m.g.d_model <= 8192;
}

int mega_token_tile(int M) {
    return M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 96 ? 96 : M <= 128 ? 128 : M <= 160 ? 160 : M <= 192 ? 192
                                                                                                                : 256;
}

// Build every launch of one forward (phase descriptors with their X tensor
// maps) and upload them with ONE copy before the forward's first kernel, so
// no copy sits between two kernels of the chain (that would break the PDL
// overlap the weight prefetch relies on).
void mega_prepare(bass_model& m, const std::vector<MegaLaunch>& launches) {
    using namespace mg;
    State& S = state(m);
    // grid: one CTA per SM, but no more CTAs than the smallest GEMM has units
    // (d x d O-projection) — a function of the model only, never of M
    int G = m.ctx->sm_count;
    for (const MegaLaunch& L : launches)
        for (const MegaPhase& s : L.phases)
            if (s.gemm) G = (int)std::min<int64_t>(G, (int64_t)((s.N + BN - 1) / BN) * (s.K / BK));
    S.G = G;
    cudaStream_t st = m.ctx->stream;
    std::vector<Phase> all;
    S.launches.clear();
    size_t ws_need = 16, flags_need = 0;
    int epoch = S.epoch;
    unsigned gen = S.gen;
    for (const MegaLaunch& L : launches) {
        const int TT = mega_token_tile(L.M_tile);
        const int n = (int)L.phases.size();
        BASS_REQUIRE(n >= 1, "mega: empty launch");
        S.launches.push_back({all.size(), n, TT, epoch + 1, gen});
        epoch += n;
        gen += (unsigned)(n - 1);
        for (const MegaPhase& s : L.phases) {
            Phase p;
            std::memset(&p, 0, sizeof(Phase));
            p.type = s.gemm ? PH_GEMM : PH_LN;
            if (s.gemm) {
                auto key = std::make_tuple(s.X, s.M, s.K, TT);
                auto it = S.xmaps.find(key);
                if (it == S.xmaps.end()) it = S.xmaps.emplace(key, x_map(s.X, s.M, s.K, TT)).first;
                p.tx = it->second;
                p.w = (const __nv_bfloat16*)s.W;
                p.e = s.e;
                p.mode = s.mode;
                p.M = s.M;
                p.N = s.N;
                p.K = s.K;
                p.k_iters = s.K / BK;
                p.U = (int64_t)((s.N + BN - 1) / BN) * p.k_iters;
                p.groups = (s.M + TT - 1) / TT;
                BASS_REQUIRE(s.K % BK == 0 && p.U >= G, "mega: GEMM shape unsupported");
                ws_need = std::max(ws_need, (size_t)p.groups * G * TT * BN * 4);
                flags_need = std::max(flags_need, (size_t)p.groups * G);
            } else {
                p.x = s.x;
                p.gather = s.gather;
                p.g = s.g;
                p.b = s.b;
                p.out = (__nv_bfloat16*)s.out;
                p.rows = s.rows;
                p.d = s.d;
                BASS_REQUIRE(s.d % 4 == 0 && s.d <= 4 * 128 * LN_V4, "mega: LayerNorm width");
            }
            all.push_back(p);
        }
    }
    S.ws_p = (float*)S.ws.need(ws_need, st);
    if (flags_need > S.flags_n) {
        int* f = (int*)S.flags.need(flags_need * 4, st);
        BASS_CUDA(cudaMemsetAsync(f, 0, flags_need * 4, st));
        S.flags_n = flags_need;
        // epochs restart above any value a flag may hold
        const int shift = 1 - S.launches.front().epoch;
        for (auto& l : S.launches) l.epoch += shift;
        epoch += shift;
    }
    if (!S.gbar.p) {
        S.gbar.need(256, st);
        BASS_CUDA(cudaMemsetAsync(S.gbar.p, 0, 256, st));
    }
    S.epoch = epoch;
    S.gen = gen;
    const size_t bytes = sizeof(Phase) * all.size();
    void* dst = S.phases.need(bytes, st);
    void* hst = m.ctx->staging.take(bytes + 64);
    if (!hst) {
        m.ctx->sync();
        hst = m.ctx->staging.take(bytes + 64);
    }
    BASS_REQUIRE(hst != nullptr, "mega: staging arena too small");
    char* h64 = (char*)(((uintptr_t)hst + 63) & ~(uintptr_t)63);
    std::memcpy(h64, all.data(), bytes);
    BASS_CUDA(cudaMemcpyAsync(dst, h64, bytes, cudaMemcpyHostToDevice, st));
    m.ctx->h2d_bytes += (int64_t)bytes;
}

void mega_launch(bass_model& m, int idx) {
    using namespace mg;
    State& S = state(m);
    const State::L& L = S.launches.at(idx);
    const Phase* dph = (const Phase*)S.phases.p + L.off;
    int* flags = (int*)S.flags.p;
    unsigned* gbar = (unsigned*)S.gbar.p;
    switch (L.TT) {
        case 16: launch<16>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 32: launch<32>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 64: launch<64>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 96: launch<96>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 128: launch<128>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 160: launch<160>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        case 192: launch<192>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
        default: launch<256>(m, S.G, dph, L.n, S.ws_p, flags, L.epoch, gbar, L.gen); break;
    }
    m.ctx->launches++;
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("mega launch: ") + cudaGetErrorString(err));
}

void mega_release(bass_model& m) {
    if (!m.mega_state) return;
    mg::State* s = static_cast<mg::State*>(m.mega_state);
    s->phases.release();
    s->ws.release();
    s->flags.release();
    s->gbar.release();
    delete s;
    m.mega_state = nullptr;
}

}  // namespace bass
