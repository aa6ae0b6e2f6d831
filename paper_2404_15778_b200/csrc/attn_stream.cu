// Streaming flash-decoding attention on tcgen05 (sm_100a), d_head = 128.
//
// One CTA = (sequence, query tile of NQ rows, head, 1024-key split).  Warp
// roles (256 threads):
//   warp 0  TMA producer: Q once, then K/V 128-key chunks into a 2-3 stage
//           ring (64 KB per stage) — the HBM stream;
//   warp 1  MMA issuer: S^T_c = K_c . Q^T into one of two TMEM buffers, one
//           chunk ahead of the softmax; O^T += V_c^T . P_c^T into TMEM;
//   warp 2  TMEM allocator;
//   warps 4-7 softmax / correction / epilogue (TMEM lane quarter = warp % 4):
//           online softmax per query column (causal s <= off + t, / sqrt(dh)),
//           O rescaled in TMEM when the running max moves, P (bf16) to smem.
// Split boundaries are absolute key positions (multiples of 1024) and every
// reduction is per column in a fixed order, so a row's bits do not depend on
// the batch, the tile or the strategy.  Rows whose history fits one split are
// written normalised (o / l) directly; longer rows leave (m, l, o) per split
// for attn_combine_kernel (same arithmetic as a one-split merge).
// ref:attention.py:85-137 (PAD / SPLIT per-sequence causal softmax).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <utility>

#include "runtime.h"

namespace bass {
namespace ast {

constexpr int DH = 128, CH = 128, SPLIT_CH = 8, SPLIT = CH * SPLIT_CH, THREADS = 256;

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
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint32_t dst, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n, int a_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
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
__device__ __forceinline__ void st16(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct Work {
    int32_t seq, t0, split, nch;   // nch: 128-key chunks of this split the tile's last row sees
};

template <int NQ>
struct Cfg {
    static constexpr int STAGES = 2;
    static constexpr int KV_TILE = CH * 128;     // one 64-wide swizzle sub-tile (bytes)
    static constexpr int STAGE = 4 * KV_TILE;    // K0 K1 V0 V1
    static constexpr int R_TILE = 128 * 128;     // 128 rows x 64 bf16: one sub-tile of Q or P
    static constexpr int OFF_Q = STAGES * STAGE, OFF_P = OFF_Q + 2 * R_TILE;
    static constexpr int OFF_BAR = OFF_P + 2 * R_TILE;
    static constexpr int NBAR = 2 * STAGES + 1 + 2 + 1 + 1;   // kv_full, kv_empty, q_full, s_full[2], p_full, o_done
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
    static constexpr int TMEM_COLS = 512;        // S0 [0,128) S1 [128,256) O [256,384)
};

// Query rows on TMEM lanes: S = Q . K^T (M = 128 query rows, N = 128 keys),
// so each softmax thread owns one row and the max / sum over keys are
// register-local; O = P . V (A = P from smem, B = V read MN-major).
template <int NQ>
__global__ void __launch_bounds__(THREADS, 1) attn_stream_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, Seqs seqs, const Work* __restrict__ work, int H, int cap, int pad_len,
    float* __restrict__ part_o, float* __restrict__ part_ml, int max_splits, __nv_bfloat16* __restrict__ out) {
    using Cf = Cfg<NQ>;
    constexpr int ST = Cf::STAGES;
    extern __shared__ uint8_t smem_raw[];
    pdl_trigger();
    const Work wk = work[blockIdx.x];
    const int h = blockIdx.y;
    const int slot = seqs.slot[wk.seq], qn = seqs.qn[wk.seq], off = seqs.off[wk.seq], q0row = seqs.q0[wk.seq];
    const int L = off + qn;
    const int s0 = wk.split * SPLIT;
    if (wk.t0 >= qn || wk.nch <= 0) return;   // idle CTA (uniform)
    const int nch = wk.nch;
    const int rows_valid = min(128, qn - wk.t0);

    const uint32_t raw = su32(smem_raw);
    const uint32_t base = (raw + 1023) & ~1023u;
    uint8_t* sm = smem_raw + (base - raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Cf::OFF_BAR);
    uint64_t* kv_full = bars;
    uint64_t* kv_empty = bars + ST;
    uint64_t* q_full = bars + 2 * ST;
    uint64_t* s_full = bars + 2 * ST + 1;   // [2]
    uint64_t* p_full = bars + 2 * ST + 3;
    uint64_t* o_done = bars + 2 * ST + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cf::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < Cf::NBAR; ++i) mbar_init(su32(&bars[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(Cf::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tO = tmem + 256;
    const int kv_row0 = (slot * H + h) * cap + s0;

    if (warp == 0) {
        if (lane == 0) {   // ---- producer
            asm volatile("griddepcontrol.wait;" ::: "memory");   // Q and this step's K/V rows come from the QKV GEMM
            mbar_expect_tx(su32(q_full), 2 * Cf::R_TILE);
            for (int s = 0; s < 2; ++s)
                tma_2d(&tq, base + Cf::OFF_Q + s * Cf::R_TILE, su32(q_full), h * DH + s * 64, q0row + wk.t0);
            for (int c = 0; c < nch; ++c) {
                const int s = c % ST;
                if (c >= ST) mbar_wait(su32(&kv_empty[s]), ((c / ST) - 1) & 1);
                const uint32_t b = su32(&kv_full[s]), st = base + s * Cf::STAGE;
                mbar_expect_tx(b, Cf::STAGE);
                for (int sub = 0; sub < 2; ++sub) {
                    tma_2d(&tk, st + sub * Cf::KV_TILE, b, sub * 64, kv_row0 + c * CH);
                    tma_2d(&tv, st + (2 + sub) * Cf::KV_TILE, b, sub * 64, kv_row0 + c * CH);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {   // ---- MMA issuer
            constexpr uint32_t ID1 = idesc(128, 0);                      // S = Q . K^T
            constexpr uint32_t ID2 = idesc(128, 0) | (1u << 16);          // O = P . V  (B = V, MN-major)
            auto mma1 = [&](int c) {
                const uint32_t st = base + (c % ST) * Cf::STAGE;
#pragma unroll
                for (int kk = 0; kk < DH / 16; ++kk) {
                    const uint32_t sub = kk >> 2, in = (kk & 3) * 32;
                    umma(tmem + (c & 1) * 128, sdesc(base + Cf::OFF_Q + sub * Cf::R_TILE + in, 16, 1024),
                         sdesc(st + sub * Cf::KV_TILE + in, 16, 1024), ID1, kk > 0);
                }
                commit(su32(&s_full[c & 1]));
            };
            mbar_wait(su32(q_full), 0);
            mbar_wait(su32(&kv_full[0]), 0);
            fence_after();
            mma1(0);
            for (int c = 0; c < nch; ++c) {
                if (c + 1 < nch) {
                    mbar_wait(su32(&kv_full[(c + 1) % ST]), ((c + 1) / ST) & 1);
                    fence_after();
                    mma1(c + 1);
                }
                mbar_wait(su32(p_full), c & 1);
                fence_after();
                const uint32_t st = base + (c % ST) * Cf::STAGE;
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk) {
                    const uint32_t sub = kk >> 2, in = (kk & 3) * 32;
                    umma(tO, sdesc(base + Cf::OFF_P + sub * Cf::R_TILE + in, 16, 1024),
                         sdesc(st + 2 * Cf::KV_TILE + kk * 2048, Cf::KV_TILE, 1024), ID2, (c > 0 || kk > 0) ? 1u : 0u);
                }
                commit(su32(o_done));
                commit(su32(&kv_empty[c % ST]));
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ---- softmax / correction / epilogue: thread r owns query row t0 + r (TMEM lane r)
        const int r = threadIdx.x - 128, t = wk.t0 + r;
        const bool warp_live = (warp - 4) * 32 < rows_valid;   // warp-uniform
        const bool live = r < rows_valid;
        const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
        const float scale = sqrtf((float)DH);
        uint8_t* Prow = sm + Cf::OFF_P + r * 128;
        float m_run = -INFINITY, l_run = 0.f;
        for (int c = 0; c < nch; ++c) {
            const int kbase = s0 + c * CH;
            const uint32_t tS = tmem + lane_off + (c & 1) * 128;
            mbar_wait(su32(&s_full[c & 1]), (c >> 1) & 1);
            fence_after();
            float mn = m_run, alpha = 1.f;
            if (warp_live) {
                float mc = -INFINITY;
#pragma unroll 1
                for (int j0 = 0; j0 < 128; j0 += 16) {
                    float v[16];
                    ld16(tS + j0, v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int kp = kbase + j0 + j;
                        if (live && kp <= off + t && kp < L) mc = fmaxf(mc, v[j] / scale);
                    }
                }
                mn = fmaxf(m_run, mc);
                alpha = mn == -INFINITY ? 1.f : expf(m_run - mn);   // m_run = -inf -> 0
            }
            if (c > 0) {   // previous PV landed: P buffer free, O may be rescaled
                mbar_wait(su32(o_done), (c - 1) & 1);
                fence_after();
                if (warp_live && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                    for (int j0 = 0; j0 < 128; j0 += 16) {
                        float v[16];
                        ld16(tO + lane_off + j0, v);
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] *= alpha;
                        st16(tO + lane_off + j0, v);
                    }
                }
            }
            float ls = 0.f;
            if (warp_live) {
#pragma unroll 1
                for (int j0 = 0; j0 < 128; j0 += 16) {
                    float v[16];
                    ld16(tS + j0, v);
                    uint32_t pk[8];
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        float p2[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int kp = kbase + j0 + j + u;
                            const bool ok = live && kp <= off + t && kp < L && mn != -INFINITY;
                            p2[u] = ok ? expf(v[j + u] / scale - mn) : 0.f;
                            ls += p2[u];
                        }
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(p2[0], p2[1]);
                        pk[j >> 1] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    // keys j0..j0+15 = two 16-byte chunks of the 128B-swizzled row
                    const int kb = j0 >> 6, ch = (j0 & 63) >> 3;
                    uint8_t* rowp = Prow + kb * Cf::R_TILE;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint32_t pc = (uint32_t)(ch + u) ^ (uint32_t)(r & 7);
                        *reinterpret_cast<uint4*>(rowp + pc * 16) =
                            make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
                    }
                }
            } else {
                // rows of an idle warp still hand the tensor core zeros
#pragma unroll
                for (int kb = 0; kb < 2; ++kb)
#pragma unroll
                    for (int ch = 0; ch < 8; ++ch)
                        *reinterpret_cast<uint4*>(Prow + kb * Cf::R_TILE + ch * 16) = make_uint4(0, 0, 0, 0);
            }
            l_run = l_run * alpha + ls;
            m_run = mn;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P -> tensor core
            fence_before();
            softmax_bar();
            if (r == 0) mbar_arrive(su32(p_full));
        }
        // ---- epilogue: row t, 128 head dims
        mbar_wait(su32(o_done), (nch - 1) & 1);
        fence_after();
        if (warp_live) {
            const bool sees = live && off + t >= s0;
            const int row = q0row + t;
            const bool direct = off + t < SPLIT;   // whole history in split 0
            const int64_t idx = ((int64_t)row * H + h) * max_splits + wk.split;
#pragma unroll 1
            for (int j0 = 0; j0 < 128; j0 += 16) {
                float v[16];
                ld16(tO + lane_off + j0, v);
                if (!sees) continue;
                if (direct) {
                    uint32_t pk[8];
#pragma unroll
                    for (int j = 0; j < 16; j += 2) {
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(v[j] / l_run, v[j + 1] / l_run);
                        pk[j >> 1] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    uint4* dst = reinterpret_cast<uint4*>(out + ((int64_t)row * H + h) * DH + j0);
                    dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                } else {
                    float4* dst = reinterpret_cast<float4*>(part_o + idx * DH + j0);
#pragma unroll
                    for (int u = 0; u < 4; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                }
            }
            if (sees && !direct) {
                part_ml[idx * 2] = m_run;
                part_ml[idx * 2 + 1] = l_run;
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::TMEM_COLS)
                     : "memory");
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap map2d(const void* ptr, int64_t rows, int64_t cols, int64_t row_stride_elems, int box_rows) {
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
    cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled (stream attention) failed");
    return m;
}

static const CUtensorMap& kv_map(const void* ptr, int64_t rows) {
    static std::map<std::pair<const void*, int64_t>, CUtensorMap> cache;
    auto key = std::make_pair(ptr, rows);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, map2d(ptr, rows, DH, DH, CH)).first;
    return it->second;
}

template <int NQ>
static void launch(bass_ctx* ctx, const AttnPlan& p, const CUtensorMap& tk, const CUtensorMap& tv, const Seqs& seqs,
                   const Work* wp, int nw, float* po, float* pml, __nv_bfloat16* out) {
    using Cf = Cfg<NQ>;
    static bool attr = false;
    if (!attr) {
        BASS_CUDA(cudaFuncSetAttribute(attn_stream_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
        attr = true;
    }
    BASS_CUDA(launch_pdl(attn_stream_kernel<NQ>, dim3(nw, p.H), dim3(THREADS), (size_t)Cf::SMEM, ctx->stream, p.tq,
                         tk, tv, seqs, wp, p.H, p.cap, p.pad_len, po, pml, p.mc, out));
}

}  // namespace ast

int stream_split_len() { return ast::SPLIT; }

// Plan: work items (seq, q tile, split, chunks seen) — RAGGED/SPLIT exact,
// PAD over the padded [max q] x [max L] grid (padded keys computed, masked).
void stream_attention_plan(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots,
                           const std::vector<int32_t>& qn, const std::vector<int32_t>& off, int H, int cap,
                           DevBuf& work_buf, AttnPlan& plan) {
    using namespace ast;
    const int n_seq = (int)qn.size();
    int max_qn = 0, max_L = 0;
    for (int i = 0; i < n_seq; ++i) {
        max_qn = std::max(max_qn, qn[i]);
        max_L = std::max(max_L, off[i] + qn[i]);
    }
    const int NQ = 128;   // query-row tile (TMEM lanes)
    std::vector<int32_t> w;
    std::vector<int> first(n_seq + 1, 0);
    bool multi = false;
    for (int i = 0; i < n_seq; ++i) {
        first[i] = (int)w.size() / 4;
        const int rows = strategy == BASS_PAD ? max_qn : qn[i];
        for (int t0 = 0; t0 < rows; t0 += NQ) {
            const int last = strategy == BASS_PAD ? max_L - 1 : off[i] + std::min(qn[i], t0 + NQ) - 1;
            const int n_chunks = last / CH + 1;
            for (int s = 0; s * SPLIT_CH < n_chunks; ++s) {
                w.insert(w.end(), {i, t0, s, std::min(SPLIT_CH, n_chunks - s * SPLIT_CH)});
                if (s > 0) multi = true;
            }
        }
    }
    first[n_seq] = (int)w.size() / 4;
    Work* wd = (Work*)work_buf.need(std::max<size_t>(w.size(), 4) * 4, ctx->stream);
    void* hst = ctx->staging.take(w.size() * 4);
    if (!hst) {
        ctx->sync();
        hst = ctx->staging.take(w.size() * 4);
    }
    std::memcpy(hst, w.data(), w.size() * 4);
    BASS_CUDA(cudaMemcpyAsync(wd, hst, w.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (int64_t)w.size() * 4;
    plan.tq = map2d(q, M, (int64_t)H * DH, (int64_t)H * DH, NQ);
    plan.NQ = NQ;
    plan.pad_len = strategy == BASS_PAD ? max_L : 0;
    plan.strategy = strategy;
    plan.H = H;
    plan.cap = cap;
    plan.n_slots = n_slots;
    plan.mc = (cap + SPLIT - 1) / SPLIT;   // splits per row (partial buffer stride)
    plan.fused = false;
    plan.stream = true;
    plan.needs_combine = multi;
    plan.first = std::move(first);
    plan.work = wd;
    plan.valid = true;
}

void stream_attention_run(bass_ctx* ctx, const AttnPlan& p, const void* kc, const void* vc, const Seqs& seqs_dev,
                          float* part_o, float* part_ml, void* out) {
    using namespace ast;
    const int64_t kv_rows = (int64_t)p.n_slots * p.H * p.cap;
    const CUtensorMap& tk = kv_map(kc, kv_rows);
    const CUtensorMap& tv = kv_map(vc, kv_rows);
    const Work* wd = static_cast<const Work*>(p.work);
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
    auto go = [&](const Work* wp, int nw) {
        if (nw == 0) return;
        switch (p.NQ) {
            case 16: launch<16>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
            case 32: launch<32>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
            case 64: launch<64>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
            default: launch<128>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
        }
        ctx->launches++;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(e));
    };
    const int n_seq = (int)p.first.size() - 1;
    if (p.strategy == BASS_SPLIT) {
        for (int i = 0; i < n_seq; ++i) go(wd + p.first[i], p.first[i + 1] - p.first[i]);
    } else {
        go(wd, p.first[n_seq]);
    }
}

}  // namespace bass
