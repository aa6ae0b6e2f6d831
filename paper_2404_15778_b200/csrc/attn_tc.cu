// Ragged verify / decode attention on tcgen05 (sm_100a), d_head = 128.
//
// One CTA = (sequence, query tile of NQ rows, head, 128-key chunk).
//   TMA:   K chunk [128 keys x 128] and V chunk (bf16, 128-byte swizzle)
//          straight from the KV cache rows, Q tile [NQ x 128] from the QKV
//          GEMM output.
//   MMA 1: S^T[key, q] = K . Q^T       (UMMA M = 128 keys, N = NQ, K = 128)
//   softmax over keys per query column (causal s <= off + t, / sqrt(dh)),
//          P (bf16) written to smem in the K-major 128B-swizzle layout
//   MMA 2: O^T[d, q] = V^T . P^T       (A = V read MN-major, M = 128 = dh)
//   epilogue: per-(row, chunk) partial (m, l, o[128]) -> combine kernel.
// Chunk boundaries are absolute key positions and every column's reductions
// are fixed-order, so a row's output does not depend on the tile it shares
// (PAD / SPLIT / RAGGED and prefill / verify / decode agree bitwise).
// ref:attention.py:85-137 (per-sequence causal softmax, PAD and SPLIT).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <utility>
#include <cstdlib>
#include <cstring>
#include <string>

#include "runtime.h"

namespace bass {
namespace atc {

constexpr int DH = 128, CH = 128, THREADS = 128;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
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
// shared-memory matrix descriptor, 128-byte swizzle, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, bf16 inputs, f32 accumulate, M = 128, N = n; a_mn: A is MN-major
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

struct Work {
    int32_t seq, t0, chunk, n;   // n: chunks walked by a fused CTA (0 in split mode)
};

constexpr int MAXC = 16;   // fused mode: at most 16 chunks (2048 keys) per CTA

template <int NQ>
struct Cfg {
    static constexpr int KV_TILE = CH * 128;            // one 64-wide swizzle sub-tile, bytes
    static constexpr int Q_TILE = NQ * 128;
    static constexpr int OFF_K = 0, OFF_V = 2 * KV_TILE, OFF_Q = 4 * KV_TILE, OFF_P = OFF_Q + 2 * Q_TILE;
    static constexpr int OFF_RED = OFF_P + 2 * Q_TILE;   // float red_max[4][NQ], red_sum[4][NQ], m[NQ]
    static constexpr int OFF_ML = OFF_RED + 9 * NQ * 4;   // fused: m, l per (chunk, column)
    static constexpr int OFF_BAR = OFF_ML + 2 * MAXC * NQ * 4;
    static constexpr int SMEM = OFF_BAR + 64 + 1024;
};

template <int NQ>
__global__ void __launch_bounds__(THREADS, 1) attn_tc_kernel(const __grid_constant__ CUtensorMap tq,
                                                             const __grid_constant__ CUtensorMap tk,
                                                             const __grid_constant__ CUtensorMap tv, Seqs seqs,
                                                             const Work* __restrict__ work, int H, int cap,
                                                             int pad_len, int tmem_cols, float* __restrict__ part_o,
                                                             float* __restrict__ part_ml, int max_chunks,
                                                             __nv_bfloat16* __restrict__ out) {
    // out == nullptr: split mode, one chunk per CTA, partial (m, l, o) out;
    // out != nullptr: fused mode, the CTA walks wk.n chunks and merges them
    // (same arithmetic as attn_combine_kernel) into ctx directly.
    using Cf = Cfg<NQ>;
    extern __shared__ uint8_t smem_raw[];
    pdl_trigger();
    const Work wk = work[blockIdx.x];
    const int h = blockIdx.y;
    const int slot = seqs.slot[wk.seq], qn = seqs.qn[wk.seq], off = seqs.off[wk.seq], q0row = seqs.q0[wk.seq];
    const int L = off + qn;
    const int kv_len = pad_len > 0 ? pad_len : L;
    const bool fused = out != nullptr;
    const int nch = fused ? wk.n : 1;
    const int cfirst = wk.chunk * CH;
    const int t_last = min(qn, wk.t0 + NQ) - 1;
    if (wk.t0 >= qn || nch <= 0 || cfirst >= kv_len || off + t_last < cfirst) return;   // idle CTA (uniform)

    const uint32_t raw = su32(smem_raw);
    const uint32_t base = (raw + 1023) & ~1023u;
    uint8_t* sm = smem_raw + (base - raw);
    float* red_max = reinterpret_cast<float*>(sm + Cf::OFF_RED);
    float* red_sum = red_max + 4 * NQ;
    float* m_col = red_sum + 4 * NQ;
    float* ml_m = reinterpret_cast<float*>(sm + Cf::OFF_ML);     // [MAXC][NQ] chunk maxima (fused)
    float* ml_l = ml_m + MAXC * NQ;                               // [MAXC][NQ] chunk sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Cf::OFF_BAR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) mbar_init(su32(&bars[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int key = warp * 32 + lane;
    const float scale = sqrtf((float)DH);
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    uint8_t* P = sm + Cf::OFF_P;
    const int psub = key >> 6, pin = key & 63;

    for (int ci = 0; ci < nch; ++ci) {
        const uint32_t ph = ci & 1;
        const int c0 = cfirst + ci * CH;
        if (threadIdx.x == 0) {   // loads: K, V chunk (2 sub-tiles each); Q tile once
            const uint32_t b = su32(&bars[0]);
            if (ci == 0) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                mbar_expect_tx(b, 4 * Cf::KV_TILE + 2 * Cf::Q_TILE);
            } else {
                mbar_expect_tx(b, 4 * Cf::KV_TILE);
            }
            const int kv_row = (slot * H + h) * cap + c0;
            for (int s = 0; s < 2; ++s) {
                tma_2d(&tk, base + Cf::OFF_K + s * Cf::KV_TILE, b, s * 64, kv_row);
                tma_2d(&tv, base + Cf::OFF_V + s * Cf::KV_TILE, b, s * 64, kv_row);
                if (ci == 0) tma_2d(&tq, base + Cf::OFF_Q + s * Cf::Q_TILE, b, h * DH + s * 64, q0row + wk.t0);
            }
            mbar_wait(b, ph);
            fence_after();
            // S^T = K . Q^T : A = K (K-major), B = Q (K-major), 8 k-steps of 16 over d
            constexpr uint32_t ID1 = idesc(NQ, 0);
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
                const uint32_t sub = kk >> 2, in = (kk & 3) * 32;
                const uint64_t a = sdesc(base + Cf::OFF_K + sub * Cf::KV_TILE + in, 16, 1024);
                const uint64_t bq = sdesc(base + Cf::OFF_Q + sub * Cf::Q_TILE + in, 16, 1024);
                umma(tmem, a, bq, ID1, kk > 0);
            }
            commit(su32(&bars[1]));
        }
        __syncwarp();
        mbar_wait(su32(&bars[1]), ph);
        fence_after();

        // ---- softmax over the 128 keys of this chunk, per query column
        const int kpos = c0 + key;
#pragma unroll 1
        for (int j0 = 0; j0 < NQ; j0 += 16) {
            float v[16];
            ld16(trow + j0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int t = wk.t0 + j0 + j;
                const bool ok = t < qn && kpos <= off + t && kpos < L;
                const float s = ok ? v[j] / scale : -INFINITY;
                const float mx = warp_max(s);
                if (lane == 0) red_max[warp * NQ + j0 + j] = mx;
            }
        }
        __syncthreads();
        if (threadIdx.x < NQ) {
            const int q = threadIdx.x;
            m_col[q] = fmaxf(fmaxf(red_max[q], red_max[NQ + q]), fmaxf(red_max[2 * NQ + q], red_max[3 * NQ + q]));
        }
        __syncthreads();
#pragma unroll 1
        for (int j0 = 0; j0 < NQ; j0 += 16) {
            float v[16];
            ld16(trow + j0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int q = j0 + j, t = wk.t0 + q;
                const bool ok = t < qn && kpos <= off + t && kpos < L;
                const float m = m_col[q];
                const float p = (ok && m != -INFINITY) ? expf(v[j] / scale - m) : 0.f;
                const float ps = warp_sum(p);
                if (lane == 0) red_sum[warp * NQ + q] = ps;
                // P[q][key] in the K-major 128B-swizzled sub-tile psub
                const uint32_t chunk = (uint32_t)(pin >> 3) ^ (uint32_t)(q & 7);
                __nv_bfloat16* dst =
                    reinterpret_cast<__nv_bfloat16*>(P + psub * Cf::Q_TILE + q * 128 + chunk * 16) + (pin & 7);
                *dst = __float2bfloat16_rn(p);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P visible to the tensor core
        fence_before();
        __syncthreads();
        const uint32_t ocol = fused ? (uint32_t)(NQ * (1 + ci)) : (uint32_t)NQ;
        if (threadIdx.x == 0) {
            fence_after();
            // O^T = V^T . P^T : A = V (MN-major: d contiguous), B = P (K-major over keys)
            constexpr uint32_t ID2 = idesc(NQ, 1);
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk) {
                const uint64_t a = sdesc(base + Cf::OFF_V + kk * 2048, Cf::KV_TILE, 1024);
                const uint32_t sub = kk >> 2, in = (kk & 3) * 32;
                const uint64_t bp = sdesc(base + Cf::OFF_P + sub * Cf::Q_TILE + in, 16, 1024);
                umma(tmem + ocol, a, bp, ID2, kk > 0);
            }
            commit(su32(&bars[2]));
        }
        // column max / sum of this chunk
        if (threadIdx.x < NQ) {
            const int q = threadIdx.x, t = wk.t0 + q;
            const float l = (red_sum[q] + red_sum[NQ + q]) + (red_sum[2 * NQ + q] + red_sum[3 * NQ + q]);
            if (fused) {
                ml_m[ci * NQ + q] = m_col[q];
                ml_l[ci * NQ + q] = l;
            } else if (t < qn && off + t >= c0) {
                const int64_t idx = ((int64_t)(q0row + t) * H + h) * max_chunks + wk.chunk;
                part_ml[idx * 2] = m_col[q];
                part_ml[idx * 2 + 1] = l;
            }
        }
        __syncwarp();
        mbar_wait(su32(&bars[2]), ph);   // V, P and the S^T columns are free again
        fence_after();
    }
    __syncthreads();

    if (!fused) {
        // O^T lane = d (0..127), columns = query rows -> partial o
#pragma unroll 1
        for (int j0 = 0; j0 < NQ; j0 += 16) {
            float v[16];
            ld16(trow + NQ + j0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int t = wk.t0 + j0 + j;
                if (t < qn && off + t >= cfirst) {
                    const int64_t idx = ((int64_t)(q0row + t) * H + h) * max_chunks + wk.chunk;
                    part_o[idx * DH + key] = v[j];
                }
            }
        }
    } else {
        // merge the chunks in order, exactly as attn_combine_kernel does
#pragma unroll 1
        for (int j0 = 0; j0 < NQ; j0 += 16) {
            float mx[16], num[16], den[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                mx[j] = -INFINITY;
                num[j] = 0.f;
                den[j] = 0.f;
            }
            for (int c = 0; c < nch; ++c)
#pragma unroll
                for (int j = 0; j < 16; ++j) mx[j] = fmaxf(mx[j], ml_m[c * NQ + j0 + j]);
            for (int c = 0; c < nch; ++c) {
                float v[16];
                ld16(trow + NQ * (1 + c) + j0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float m = ml_m[c * NQ + j0 + j];
                    if (m == -INFINITY) continue;
                    const float w = expf(m - mx[j]);
                    num[j] = fmaf(w, v[j], num[j]);
                    den[j] = fmaf(w, ml_l[c * NQ + j0 + j], den[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int t = wk.t0 + j0 + j;
                if (t < qn) out[((int64_t)(q0row + t) * H + h) * DH + key] = __float2bfloat16_rn(num[j] / den[j]);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols)
                     : "memory");
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

static CUtensorMap map2d(const void* ptr, int64_t rows, int64_t cols, int64_t row_stride_elems, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(BASS_ERR_CUDA, "cuTensorMapEncodeTiled (attention) failed");
    return m;
}

template <int NQ>
static void launch(bass_ctx* ctx, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                   const Seqs& seqs, const Work* work, int n_work, int H, int cap, int pad_len, int tmem_cols,
                   float* po, float* pml, int max_chunks, __nv_bfloat16* out) {
    using Cf = Cfg<NQ>;
    static bool attr = false;
    if (!attr) {
        BASS_CUDA(cudaFuncSetAttribute(attn_tc_kernel<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
        attr = true;
    }
    BASS_CUDA(launch_pdl(attn_tc_kernel<NQ>, dim3(n_work, H), dim3(THREADS), (size_t)Cf::SMEM, ctx->stream, tq, tk, tv,
                         seqs, work, H, cap, pad_len, tmem_cols, po, pml, max_chunks, out));
}

static int pow2_cols(int c) {
    int p = 32;
    while (p < c) p <<= 1;
    return p;
}

}  // namespace atc

bool tc_attention_supported(int dtype, int dh) {
    static const bool off = getenv("BASS_ATTN") && std::string(getenv("BASS_ATTN")) == "simt";
    return !off && dtype == BASS_BF16 && dh == atc::DH;
}

// One-shot (plan + run) used by the standalone bass_attention path (split mode).
void tc_attention(bass_ctx* ctx, int strategy, const void* q, int M, const void* kc, const void* vc, int n_slots,
                  const Seqs& seqs_dev, const std::vector<int32_t>& qn, const std::vector<int32_t>& off, int H, int cap,
                  DevBuf& work_buf, float* part_o, float* part_ml, int max_chunks, int* nq_out) {
    AttnPlan plan;
    tc_attention_plan(ctx, strategy, q, M, n_slots, qn, off, H, cap, work_buf, plan, /*allow_fused=*/false);
    *nq_out = plan.NQ;
    tc_attention_run(ctx, plan, kc, vc, seqs_dev, part_o, part_ml, nullptr);
}

// K/V cache maps are stable per (layer buffer, rows): encode once per process
static const CUtensorMap& kv_map(const void* ptr, int64_t rows) {
    static std::map<std::pair<const void*, int64_t>, CUtensorMap> cache;
    auto key = std::make_pair(ptr, rows);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, atc::map2d(ptr, rows, atc::DH, atc::DH, atc::CH)).first;
    return it->second;
}

void tc_attention_run(bass_ctx* ctx, const AttnPlan& p, const void* kc, const void* vc, const Seqs& seqs_dev,
                      float* part_o, float* part_ml, void* out) {
    using namespace atc;
    const int64_t kv_rows = (int64_t)p.n_slots * p.H * p.cap;
    const CUtensorMap& tk = kv_map(kc, kv_rows);
    const CUtensorMap& tv = kv_map(vc, kv_rows);
    const Work* wd = static_cast<const Work*>(p.work);
    __nv_bfloat16* o = p.fused ? static_cast<__nv_bfloat16*>(out) : nullptr;
    auto go = [&](const Work* wp, int nw) {
        if (nw == 0) return;
        switch (p.NQ) {
            case 16: launch<16>(ctx, p.tq, tk, tv, seqs_dev, wp, nw, p.H, p.cap, p.pad_len, p.tmem_cols, part_o, part_ml, p.mc, o); break;
            case 32: launch<32>(ctx, p.tq, tk, tv, seqs_dev, wp, nw, p.H, p.cap, p.pad_len, p.tmem_cols, part_o, part_ml, p.mc, o); break;
            case 64: launch<64>(ctx, p.tq, tk, tv, seqs_dev, wp, nw, p.H, p.cap, p.pad_len, p.tmem_cols, part_o, part_ml, p.mc, o); break;
            default: launch<128>(ctx, p.tq, tk, tv, seqs_dev, wp, nw, p.H, p.cap, p.pad_len, p.tmem_cols, part_o, part_ml, p.mc, o); break;
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

// Work list.  Split mode: one item per (seq, q tile, 128-key chunk).  Fused
// mode (all tiles see <= MAXC chunks and (1 + chunks) * NQ TMEM columns fit):
// one item per (seq, q tile) walking its chunks.  RAGGED/SPLIT are exact;
// PAD covers the padded [max q] x [max L] grid (padded keys computed, masked).
void tc_attention_plan(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots, const std::vector<int32_t>& qn,
                       const std::vector<int32_t>& off, int H, int cap, DevBuf& work_buf, AttnPlan& plan,
                       bool allow_fused) {
    using namespace atc;
    const int n_seq = (int)qn.size();
    int max_qn = 0, max_L = 0;
    for (int i = 0; i < n_seq; ++i) {
        max_qn = std::max(max_qn, qn[i]);
        max_L = std::max(max_L, off[i] + qn[i]);
    }
    const int NQ = max_qn <= 16 ? 16 : max_qn <= 32 ? 32 : max_qn <= 64 ? 64 : 128;
    auto chunks_seen = [&](int i, int t0) {   // chunks visible to the last row of a tile
        const int len = strategy == BASS_PAD ? max_L : off[i] + std::min(qn[i], t0 + NQ);
        return (len + CH - 1) / CH;
    };
    // split mode (one CTA per chunk + combine) measured faster on the benchmark
    // (more CTAs in flight); the fused walk is opt-in and bitwise identical
    static const bool no_fuse = !(getenv("BASS_ATTN_FUSED") && atoi(getenv("BASS_ATTN_FUSED")) == 1);
    int max_nch = 0;
    for (int i = 0; i < n_seq; ++i)
        for (int t0 = 0; t0 < (strategy == BASS_PAD ? max_qn : qn[i]); t0 += NQ)
            max_nch = std::max(max_nch, chunks_seen(i, t0));
    const bool fused = allow_fused && !no_fuse && max_nch <= MAXC && (1 + max_nch) * NQ <= 512;
    std::vector<int32_t> w;
    std::vector<int> first(n_seq + 1, 0);
    for (int i = 0; i < n_seq; ++i) {
        first[i] = (int)w.size() / 4;
        const int rows = strategy == BASS_PAD ? max_qn : qn[i];
        for (int t0 = 0; t0 < rows; t0 += NQ) {
            const int nch = chunks_seen(i, t0);
            if (fused) {
                w.insert(w.end(), {i, t0, 0, nch});
            } else {
                for (int c = 0; c < nch; ++c) w.insert(w.end(), {i, t0, c, 0});
            }
        }
    }
    first[n_seq] = (int)w.size() / 4;
    Work* wd = (Work*)work_buf.need(std::max<size_t>(w.size(), 4) * 4, ctx->stream);
    void* h = ctx->staging.take(w.size() * 4);
    if (!h) {
        ctx->sync();
        h = ctx->staging.take(w.size() * 4);
    }
    std::memcpy(h, w.data(), w.size() * 4);
    BASS_CUDA(cudaMemcpyAsync(wd, h, w.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (int64_t)w.size() * 4;
    plan.tq = map2d(q, M, (int64_t)H * DH, (int64_t)H * DH, NQ);
    plan.NQ = NQ;
    plan.pad_len = strategy == BASS_PAD ? max_L : 0;
    plan.strategy = strategy;
    plan.H = H;
    plan.cap = cap;
    plan.n_slots = n_slots;
    plan.mc = (cap + CH - 1) / CH;
    plan.fused = fused;
    plan.tmem_cols = pow2_cols(fused ? (1 + max_nch) * NQ : 2 * NQ);
    plan.first = std::move(first);
    plan.work = wd;
    plan.valid = true;
}

}  // namespace bass
