// libbass runtime: contexts, device weights, ragged KV cache, the ragged
// forward (ref:model.py:177-246) and the C-ABI entry points of include/bass.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstring>

#include "runtime.h"
#include "cluster_sampling.cuh"
#include "quant.cuh"

using namespace bass;

// ------------------------------------------------------------ utilities
namespace bass {

void* Staging::take(size_t n) {
    n = (n + 255) & ~size_t(255);
    if (used + n > cap) return nullptr;
    void* p = base + used;
    used += n;
    return p;
}

static std::atomic<uint64_t> g_devbuf_epoch{0};
uint64_t devbuf_epoch() { return g_devbuf_epoch.load(); }

void* DevBuf::need(size_t n, cudaStream_t s) {
    if (n <= cap) return p;
    g_devbuf_epoch.fetch_add(1);   // a captured graph holding the old address is stale
    if (p) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        BASS_CUDA(cudaStreamIsCapturing(s, &cs));
        if (cs == cudaStreamCaptureStatusNone) {
            BASS_CUDA(cudaStreamSynchronize(s));
            BASS_CUDA(cudaFree(p));
        } else {
            retired.push_back(p);   // captured graph nodes still use it: freed with the buffer
        }
        p = nullptr;
    }
    size_t c = std::max(n, cap * 3 / 2);
    BASS_CUDA(cudaMalloc(&p, c));
    cap = c;
    return p;
}

void DevBuf::release() {
    for (void* r : retired) cudaFree(r);
    retired.clear();
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
}

void Batch::add_seq(int s, int offset, const int32_t* toks, int n) {
    slot.push_back(s);
    q0.push_back(rows());
    qn.push_back(n);
    off.push_back(offset);
    for (int t = 0; t < n; ++t) {
        tok.push_back(toks[t]);
        row_slot.push_back(s);
        row_pos.push_back(offset + t);
    }
}

}  // namespace bass

cudaEvent_t bass_ctx::ev() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    BASS_CUDA(cudaEventCreate(&e));
    return e;
}

void bass_ctx::resolve() {
    for (const Pending& p : pending) {
        float ms = 0.f;
        BASS_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        prof_ms[p.cls] += ms;
        prof_bytes[p.cls] += p.bytes;
        prof_flops[p.cls] += p.flops;
        prof_n[p.cls] += 1;
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    pending.clear();
}

void bass_ctx::sync() {
    BASS_CUDA(cudaStreamSynchronize(stream));
    staging.used = 0;
    if (!pending.empty()) resolve();
}

template <typename F>
static int guarded(bass_ctx* ctx, F&& f) {
    try {
        f();
        return BASS_OK;
    } catch (const Error& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return BASS_ERR_STATE;
    }
}

#define LAUNCHED(ctx) ((ctx)->launches++)

static void check_launch(bass_ctx* ctx) {
    LAUNCHED(ctx);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// stage `n` int32 values to device through pinned memory (async)
static void upload_i32(bass_ctx* ctx, int32_t* dev, const int32_t* src, size_t n) {
    if (n == 0) return;
    void* h = ctx->staging.take(n * 4);
    if (!h) {
        ctx->sync();
        h = ctx->staging.take(n * 4);
        if (!h) throw Error(BASS_ERR_MEMORY, "staging arena too small");
    }
    std::memcpy(h, src, n * 4);
    BASS_CUDA(cudaMemcpyAsync(dev, h, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (int64_t)n * 4;
}

// ------------------------------------------------------- weight kernels
namespace {

// dst[n, k] = src[k, n]  (reference input-major [K, N] -> output-major [N, K])
template <typename T>
__global__ void transpose_convert(const float* __restrict__ src, int K, int N, T* __restrict__ dst,
                                  int64_t dst_ld, int64_t row_off, bool packed) {
    __shared__ float tile[32][33];
    const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, n = n0 + threadIdx.x;
        tile[i][threadIdx.x] = (k < K && n < N) ? src[(int64_t)k * N + n] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int n = n0 + i, k = k0 + threadIdx.x;
        if (n < N && k < K)
            dst[packed ? packed_index(row_off + n, k, dst_ld) : (row_off + n) * dst_ld + k] = cvt<T>(tile[threadIdx.x][i]);
    }
}

// inverse of transpose_convert: device output-major rows -> reference [K, N] fp32
template <typename T>
__global__ void transpose_gather(const T* __restrict__ src, int K, int N, float* __restrict__ dst,
                                 int64_t src_ld, int64_t row_off, bool packed) {
    __shared__ float tile[32][33];
    const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int n = n0 + i, k = k0 + threadIdx.x;
        tile[threadIdx.x][i] = (n < N && k < K)
                                   ? ld(src, packed ? packed_index(row_off + n, k, src_ld) : (row_off + n) * src_ld + k)
                                   : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, n = n0 + threadIdx.x;
        if (k < K && n < N) dst[(int64_t)k * N + n] = tile[i][threadIdx.x];
    }
}

template <typename T>
__global__ void to_f32(const T* __restrict__ src, int64_t n, float* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = ld(src, i);
}

__global__ void pack_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, int N, int K,
                            int64_t src_stride, int64_t dst_stride, int n_mat) {
    const int64_t per = (int64_t)N * K;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per * n_mat; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mat = i / per, r = i - mat * per, n = r / K, k = r - n * K;
        dst[mat * dst_stride + packed_index(n, k, K)] = src[mat * src_stride + r];
    }
}

template <typename T>
__global__ void convert_copy(const float* __restrict__ src, int64_t n, T* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = cvt<T>(src[i]);
}

template <typename T>
__global__ void random_normal(T* __restrict__ dst, int64_t n, uint64_t seed, float std) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = splitmix64(seed ^ splitmix64(uint64_t(i)));
        const uint64_t b = splitmix64(a);
        const float u1 = (float((a >> 40) + 1) * (1.0f / 16777217.0f));
        const float u2 = float(b >> 40) * (1.0f / 16777216.0f);
        dst[i] = cvt<T>(std * sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2));
    }
}

__global__ void fill_f32(float* p, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace

// ------------------------------------------------------------ forward
namespace bass {

template <typename TA>
static void launch_layernorm(bass_model& m, const float* x, const int32_t* gather, const float* g,
                             const float* b, int rows, TA* out) {
    ProfScope prof(m.ctx, BASS_PROF_NORM, (double)rows * m.g.d_model * (4.0 + sizeof(TA)));
    BASS_CUDA(launch_pdl(layernorm_kernel<TA>, dim3(rows), dim3(256), 0, m.ctx->stream, x, gather, g, b,
                         m.g.d_model, out, m.ctx->trace(rows, BASS_TR_NORM)));
    check_launch(m.ctx);
}

static void launch_layernorm_any(bass_model& m, const float* x, const int32_t* gather, const float* g,
                                 const float* b, int rows, void* out) {
    if (m.dtype != BASS_F32) launch_layernorm(m, x, gather, g, b, rows, (__nv_bfloat16*)out);
    else launch_layernorm(m, x, gather, g, b, rows, (float*)out);
}

template <int MODE, typename TA>
static void gemm_simt(bass_model& m, const void* X, const void* W, int M, int N, int K, const Epi& e, bool packed) {
    dim3 grid((N + SG_BN - 1) / SG_BN, (M + SG_BM - 1) / SG_BM);
    gemm_simt_kernel<MODE, TA, TA><<<grid, 256, 0, m.ctx->stream>>>((const TA*)X, (const TA*)W, M, N, K, e, packed);
    check_launch(m.ctx);
}

// algorithmic bytes of one GEMM launch: weights + activations in + results out
static double gemm_bytes(const bass_model& m, int mode, int M, int N, int K) {
    const double es = (double)m.esize, ws = (double)m.wsize;
    double out = mode == EPI_STORE ? 4.0 * M * N : mode == EPI_RESID ? 8.0 * M * N : es * M * N;
    return ws * N * K + (m.int8() ? 1.0 : es) * M * K + out;
}

// W8A8 projection (BASS_INT8 models): int8 X [M, K] with per-token scales sx,
// packed int8 W with per-channel scales sw, on the tcgen05 kind::i8 GEMM
// (ref:model.py:160-164 `_linear` with a QuantTensor, quant.py:98-123)
static void gemm_i8(bass_model& m, int mode, const int8_t* X, const double* sx, const void* W, const double* sw,
                    int M, int N, int K, const Epi& e) {
    if (M == 0) return;
    ProfScope prof(m.ctx, BASS_PROF_GEMM, gemm_bytes(m, mode, M, N, K), 2.0 * M * N * K);
    BASS_REQUIRE(tc_gemm_supported(m, N, K), "int8 GEMM needs K % 128 == 0 and N >= 128");
    tc_gemm(m, mode, X, W, M, N, K, e, true, nullptr, sx, sw);
}

// c[n] = sum_k g[k] W[n, k], e[n] = sum_k b[k] W[n, k] (W packed bf16): the
// per-column constants of a LayerNorm folded into the following GEMM.  One
// warp per column, fixed-order sums.
__global__ void ln_fold_kernel(const __nv_bfloat16* __restrict__ w, int N, int K, const float* __restrict__ g,
                               const float* __restrict__ b, float* __restrict__ c, float* __restrict__ e) {
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (n >= N) return;
    float sc = 0.f, se = 0.f;
    for (int k = lane; k < K; k += 32) {
        const float v = __bfloat162float(w[packed_index(n, k, K)]);
        sc = fmaf(g[k], v, sc);
        se = fmaf(b[k], v, se);
    }
    sc = warp_sum(sc);
    se = warp_sum(se);
    if (lane == 0) {
        c[n] = sc;
        e[n] = se;
    }
}

// rows `lrows` of the folded-LN head input (bf16 X = x * g_f and the per
// (tile, row) {sum, sum^2}) into compact [R] buffers
__global__ void head_gather_kernel(const __nv_bfloat16* __restrict__ xb, const float2* __restrict__ st,
                                   const int32_t* __restrict__ lrows, int M, int R, int d, int tiles,
                                   __nv_bfloat16* __restrict__ xo, float2* __restrict__ so) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x, src = lrows[r];
    const uint4* in = reinterpret_cast<const uint4*>(xb + (int64_t)src * d);
    uint4* out = reinterpret_cast<uint4*>(xo + (int64_t)r * d);
    for (int c = threadIdx.x; c < d / 8; c += blockDim.x) out[c] = in[c];
    for (int t = threadIdx.x; t < tiles; t += blockDim.x) so[(int64_t)t * R + r] = st[(int64_t)t * M + src];
}

// the bf16 forward folds every LayerNorm into the following GEMM (see forward())
static bool uses_ln_fold(const bass_model& m) {
    return m.dtype == BASS_BF16 && m.packed && m.gemm_mode != BASS_GEMM_SIMT && tc_gemm_supported(m, m.g.d_model, m.g.d_model) &&
           m.g.d_model % 8 == 0;
}

static void ln_fold_prepare(bass_model& m) {
    if (m.lnfold_valid) return;
    const int d = m.g.d_model, L = m.g.n_layer;
    const size_t per = (size_t)(2 * 3 * d + 2 * 4 * d);
    const int V = m.g.vocab_size;
    // per layer [3d c][3d e][4d c][4d e], then the final LayerNorm -> head [V c][V e]
    float* base = (float*)m.lnfold.need((per * L + 2 * (size_t)V) * 4, m.ctx->stream);
    for (int l = 0; l < L; ++l) {
        float* p = base + per * l;
        const bass_layer& ly = m.layers[l];
        ln_fold_kernel<<<(3 * d + 7) / 8, 256, 0, m.ctx->stream>>>((const __nv_bfloat16*)ly.wqkv, 3 * d, d, ly.ln1_g,
                                                                    ly.ln1_b, p, p + 3 * d);
        ln_fold_kernel<<<(4 * d + 7) / 8, 256, 0, m.ctx->stream>>>((const __nv_bfloat16*)ly.wfc, 4 * d, d, ly.ln2_g,
                                                                    ly.ln2_b, p + 6 * d, p + 10 * d);
    }
    ln_fold_kernel<<<(V + 7) / 8, 256, 0, m.ctx->stream>>>((const __nv_bfloat16*)m.head, V, d, m.lnf_g, m.lnf_b,
                                                           base + per * L, base + per * L + V);
    BASS_CUDA(cudaGetLastError());
    m.lnfold_valid = true;
}

void pack_weights(cudaStream_t st, const void* src, void* dst, int N, int K, int n_mat) {
    pack_kernel<<<1184, 256, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, N, K, (int64_t)N * K,
                                      packed_rows(N) * K, n_mat);
    BASS_CUDA(cudaGetLastError());
}

void gemm(bass_model& m, int mode, const void* X, const void* W, int M, int N, int K, const Epi& e, bool packed,
          const TcNorm* norm) {
    if (M == 0) return;
    ProfScope prof(m.ctx, BASS_PROF_GEMM, gemm_bytes(m, mode, M, N, K), 2.0 * M * N * K);
    if (m.int8()) throw Error(BASS_ERR_STATE, "int8 models project through gemm_i8");
    const bool tc = m.dtype == BASS_BF16 && m.gemm_mode != BASS_GEMM_SIMT && tc_gemm_supported(m, N, K);
    if (m.gemm_mode == BASS_GEMM_TC && !tc)
        throw Error(BASS_ERR_STATE, "tcgen05 GEMM requested but unsupported for this shape/dtype");
    BASS_REQUIRE(!norm || tc, "fused LayerNorm needs the tcgen05 GEMM");
    if (tc) {
        // split-K clusters (gemm_tc.cu).  Persistent alternatives were measured
        // slower inside the PDL chain (static stream-K: staggered SM release;
        // dynamic k-chunks: per-chunk reduction latency) — DESIGN.md section 4
        tc_gemm(m, mode, X, W, M, N, K, e, packed, norm);
        return;
    }
#define BASS_GEMM_CASE(MD)                                                            \
    case MD:                                                                          \
        if (m.dtype == BASS_BF16) gemm_simt<MD, __nv_bfloat16>(m, X, W, M, N, K, e, packed); \
        else gemm_simt<MD, float>(m, X, W, M, N, K, e, packed);                              \
        break;
    switch (mode) {
        BASS_GEMM_CASE(EPI_QKV)
        BASS_GEMM_CASE(EPI_RESID)
        BASS_GEMM_CASE(EPI_GELU)
        BASS_GEMM_CASE(EPI_STORE)
        default: throw Error(BASS_ERR_STATE, "bad epilogue");
    }
#undef BASS_GEMM_CASE
}

template <typename TA, int DH>
static void launch_attention_t(bass_ctx* ctx, int strategy, const void* q, const void* kc, const void* vc,
                               const Seqs& seqs_dev, const std::vector<int32_t>& qn,
                               const std::vector<int32_t>& off, const int32_t* row_pos_dev, int M,
                               int H, int cap, int n_slots, DevBuf& work_buf, DevBuf& po, DevBuf& pml,
                               void* out) {
    const int n_seq = (int)qn.size();
    if constexpr (std::is_same<TA, __nv_bfloat16>::value && (DH == 128 || DH == 64)) {
        if (tc_attention_supported(BASS_BF16, DH)) {   // persistent TMA + tcgen05 kernel (attn_stream.cu)
            double abytes = 0.0, aflops = 0.0;
            for (int i = 0; i < n_seq; ++i) {
                abytes += (2.0 * H * (off[i] + qn[i]) * DH + 2.0 * H * qn[i] * DH) * sizeof(TA);
                aflops += 4.0 * H * DH * qn[i] * (off[i] + 0.5 * (qn[i] + 1));
            }
            ProfScope prof(ctx, BASS_PROF_ATTN, abytes, aflops);
            AttnPlan plan;
            std::vector<int32_t> ident(n_seq);
            for (int i = 0; i < n_seq; ++i) ident[i] = i;   // standalone: sequence i uses K/V entry i
            stream_attention_plan(ctx, strategy, q, M, n_slots, ident, qn, off, H, DH, cap, work_buf, plan);
            float* so = (float*)po.need((size_t)M * H * plan.mc * DH * 4, ctx->stream);
            float* sml = (float*)pml.need((size_t)M * H * plan.mc * 2 * 4, ctx->stream);
            stream_attention_run(ctx, plan, kc, vc, seqs_dev, so, sml, out);
            if (plan.needs_combine) {
                BASS_CUDA(launch_pdl(attn_combine_kernel<TA, DH>, dim3(M, H), dim3(DH), 0, ctx->stream,
                                     (const float*)so, (const float*)sml, row_pos_dev, H, plan.mc,
                                     stream_split_len(), (TA*)out, 1));
                check_launch(ctx);
            }
            return;
        }
    }
    const int max_chunks = (cap + AT_CHUNK - 1) / AT_CHUNK;
    float* part_o = (float*)po.need((size_t)M * H * max_chunks * DH * 4, ctx->stream);
    float* part_ml = (float*)pml.need((size_t)M * H * max_chunks * 2 * 4, ctx->stream);
    const size_t smem = (size_t)(DH * (AT_SUB + 1) + AT_SUB * DH + AT_QT * DH) * 4;
    static unsigned attr = 0;
    once_per_device(attr, [&] {
        BASS_CUDA(cudaFuncSetAttribute(attn_partial_kernel<TA, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    });
    int max_qn = 0, max_L = 0;
    for (int i = 0; i < n_seq; ++i) {
        max_qn = std::max(max_qn, qn[i]);
        max_L = std::max(max_L, off[i] + qn[i]);
    }
    // work lists: RAGGED/SPLIT exact tiles; PAD every tile of the padded [max_qn] range
    std::vector<int32_t> work;
    std::vector<int> seq_first(n_seq + 1, 0);
    for (int i = 0; i < n_seq; ++i) {
        seq_first[i] = (int)work.size() / 2;
        const int rows = strategy == BASS_PAD ? max_qn : qn[i];
        for (int t0 = 0; t0 < rows; t0 += AT_QT) {
            work.push_back(i);
            work.push_back(t0);
        }
    }
    seq_first[n_seq] = (int)work.size() / 2;
    AttnWork* wdev = (AttnWork*)work_buf.need(work.size() * 4, ctx->stream);
    upload_i32(ctx, (int32_t*)wdev, work.data(), work.size());
    // algorithmic bytes: real K/V rows + Q in + O out
    double abytes = 0.0, aflops = 0.0;
    for (int i = 0; i < n_seq; ++i) {
        abytes += (2.0 * H * (off[i] + qn[i]) * DH + 2.0 * H * qn[i] * DH) * sizeof(TA);
        aflops += 4.0 * H * DH * qn[i] * (off[i] + 0.5 * (qn[i] + 1));
    }
    ProfScope prof(ctx, BASS_PROF_ATTN, abytes, aflops);
    const int threads = AT_THREADS;
    if (strategy == BASS_SPLIT) {
        for (int i = 0; i < n_seq; ++i) {
            const int nw = seq_first[i + 1] - seq_first[i];
            dim3 grid((off[i] + qn[i] + AT_CHUNK - 1) / AT_CHUNK, H, nw);
            attn_partial_kernel<TA, DH><<<grid, threads, smem, ctx->stream>>>(
                (const TA*)q, (const TA*)kc, (const TA*)vc, seqs_dev, wdev + seq_first[i], H, cap, 0, part_o,
                part_ml, max_chunks);
            check_launch(ctx);
        }
    } else {
        const int nw = seq_first[n_seq];
        dim3 grid((max_L + AT_CHUNK - 1) / AT_CHUNK, H, nw);
        attn_partial_kernel<TA, DH><<<grid, threads, smem, ctx->stream>>>(
            (const TA*)q, (const TA*)kc, (const TA*)vc, seqs_dev, wdev, H, cap,
            strategy == BASS_PAD ? max_L : 0, part_o, part_ml, max_chunks);
        check_launch(ctx);
    }
    BASS_CUDA(launch_pdl(attn_combine_kernel<TA, DH>, dim3(M, H), dim3(DH), 0, ctx->stream, (const float*)part_o,
                         (const float*)part_ml, row_pos_dev, H, max_chunks, (int)AT_CHUNK, (TA*)out, 0));
    check_launch(ctx);
}

static void launch_attention(bass_ctx* ctx, int dtype, int dh, int strategy, const void* q, const void* kc,
                             const void* vc, const Seqs& seqs_dev, const std::vector<int32_t>& qn,
                             const std::vector<int32_t>& off, const int32_t* row_pos_dev, int M, int H, int cap,
                             int n_slots, DevBuf& work_buf, DevBuf& po, DevBuf& pml, void* out) {
#define BASS_ATT(T, D)                                                                                  \
    launch_attention_t<T, D>(ctx, strategy, q, kc, vc, seqs_dev, qn, off, row_pos_dev, M, H, cap, n_slots, \
                             work_buf, po, pml, out)
    if (dtype == BASS_BF16) {
        if (dh == 16) BASS_ATT(__nv_bfloat16, 16);
        else if (dh == 32) BASS_ATT(__nv_bfloat16, 32);
        else if (dh == 64) BASS_ATT(__nv_bfloat16, 64);
        else if (dh == 128) BASS_ATT(__nv_bfloat16, 128);
        else throw Error(BASS_ERR_VALUE, "d_head must be 16, 32, 64 or 128");
    } else {
        if (dh == 16) BASS_ATT(float, 16);
        else if (dh == 32) BASS_ATT(float, 32);
        else if (dh == 64) BASS_ATT(float, 64);
        else if (dh == 128) BASS_ATT(float, 128);
        else throw Error(BASS_ERR_VALUE, "d_head must be 16, 32, 64 or 128");
    }
#undef BASS_ATT
}

// forward's metadata block: tok, row_slot, row_pos | slot, q0, qn, off | logit_rows
static void append_meta(const Batch& b, std::vector<int32_t>& hm) {
    hm.insert(hm.end(), b.tok.begin(), b.tok.end());
    hm.insert(hm.end(), b.row_slot.begin(), b.row_slot.end());
    hm.insert(hm.end(), b.row_pos.begin(), b.row_pos.end());
    hm.insert(hm.end(), b.slot.begin(), b.slot.end());
    hm.insert(hm.end(), b.q0.begin(), b.q0.end());
    hm.insert(hm.end(), b.qn.begin(), b.qn.end());
    hm.insert(hm.end(), b.off.begin(), b.off.end());
    hm.insert(hm.end(), b.logit_rows.begin(), b.logit_rows.end());
}

// the forward's attention runs the stream kernel (its work list can be pre-staged)
bool model_uses_stream_attention(const bass_model& m);
static bool uses_stream_attention(const bass_model& m) { return model_uses_stream_attention(m); }
bool model_uses_stream_attention(const bass_model& m) {
    return m.dtype != BASS_F32 && tc_attention_supported(BASS_BF16, m.g.d_head);
}

PreMetaOff forward_premeta(const bass_model& m, const Batch& b, int strategy, const std::vector<int32_t>& safe,
                           std::vector<int32_t>& h) {
    auto align8 = [&] { h.resize((h.size() + 7) & ~(size_t)7, 0); };   // 32-byte sections
    PreMetaOff o;
    align8();
    o.meta = h.size();
    append_meta(b, h);
    if (uses_stream_attention(m)) {
        align8();
        o.work = h.size();
        o.has_work = true;
        stream_attention_work(strategy, b.slot, b.qn, b.off, safe, h);
    }
    return o;
}

void forward_prepare(bass_model& m) {
    if (uses_ln_fold(m)) ln_fold_prepare(m);
}

void forward(bass_model& m, bass_kv& kv, const Batch& b, int strategy, float* logits_out,
             const int32_t* proposals, int pstride, const PreMeta* pre) {
    bass_ctx* ctx = m.ctx;
    // live-row bound of a device-planned forward, seen by every GEMM launch below
    struct LiveRows {
        bass_model& m;
        ~LiveRows() { m.dev_rows = nullptr; }
    } live_rows{m};
    const bool devp = pre && pre->dev;
    m.dev_rows = devp ? pre->m_act : nullptr;
    cudaStream_t st = ctx->stream;
    const bass_geometry& g = m.g;
    const int M = b.rows(), n_seq = (int)b.slot.size(), R = (int)b.logit_rows.size();
    const int d = g.d_model, H = g.n_head, dh = g.d_head, V = g.vocab_size;
    const size_t es = m.esize;
    int32_t* meta;
    if (pre && pre->meta) {
        meta = const_cast<int32_t*>(pre->meta);
    } else {
        const size_t nmeta = 3 * (size_t)M + 4 * (size_t)n_seq + R;
        meta = (int32_t*)m.meta.need(nmeta * 4, st);
        std::vector<int32_t> hm;
        hm.reserve(nmeta);
        append_meta(b, hm);
        upload_i32(ctx, meta, hm.data(), hm.size());
    }
    Rows rows{meta, meta + M, meta + 2 * M};
    Seqs seqs{meta + 3 * M, meta + 3 * M + n_seq, meta + 3 * M + 2 * n_seq, meta + 3 * M + 3 * n_seq};
    const int32_t* lrows = meta + 3 * M + 4 * n_seq;

    float* x = (float*)m.x.need((size_t)M * d * 4, st);
    void* h = m.h.need((size_t)M * d * es, st);
    void* q = m.q.need((size_t)M * d * es, st);
    void* cx = m.ctxb.need((size_t)M * d * es, st);
    // int8 models: fp32 [M, 4d] GELU output of the FC projection
    void* f = m.f.need((size_t)M * 4 * d * (m.int8() ? 4 : es), st);
    DevBuf& work_buf = m.attn_work;

    // tcgen05 attention: one plan (work list, Q map) for all layers of this forward
    AttnPlan plan;
    double attn_bytes = 0.0, attn_flops = 0.0;
    float *pa_o = nullptr, *pa_ml = nullptr;
    if (uses_stream_attention(m) && pre && pre->dev) {
        // device-planned (decode-loop graph): lengths live on the device; the
        // algorithmic bytes are accounted by the engine from the step trace
        stream_attention_plan_dev(ctx, strategy, q, M, kv.n_slots, b.qn, H, dh, kv.cap, pre->work, pre->work_stride,
                                  pre->max_len, plan);
        pa_o = (float*)m.part_o.need((size_t)M * H * plan.mc * dh * 4, st);
        pa_ml = (float*)m.part_ml.need((size_t)M * H * plan.mc * 2 * 4, st);
    } else if (uses_stream_attention(m)) {
        stream_attention_plan(ctx, strategy, q, M, kv.n_slots, b.slot, b.qn, b.off, H, dh, kv.cap, work_buf, plan,
                              pre ? pre->work : nullptr);
        pa_o = (float*)m.part_o.need((size_t)M * H * plan.mc * dh * 4, st);
        pa_ml = (float*)m.part_ml.need((size_t)M * H * plan.mc * 2 * 4, st);
        for (int i = 0; i < n_seq; ++i) {
            attn_bytes += (2.0 * H * (b.off[i] + b.qn[i]) * dh + 2.0 * H * b.qn[i] * dh) * es;
            attn_flops += 4.0 * H * dh * b.qn[i] * (b.off[i] + 0.5 * (b.qn[i] + 1));
        }
    }

    // layer li's attention (its Q from the QKV projection; K/V rows appended there)
    auto run_attention = [&](int li, void* kc, void* vc) {
        if (plan.valid) {
            ProfScope prof(ctx, BASS_PROF_ATTN, attn_bytes, attn_flops);
            stream_attention_run(ctx, plan, kc, vc, seqs, pa_o, pa_ml, cx);
            if (plan.needs_combine) {
                if (dh == 64)
                    BASS_CUDA(launch_pdl(attn_combine_kernel<__nv_bfloat16, 64>, dim3(M, H), dim3(64), 0, st,
                                         (const float*)pa_o, (const float*)pa_ml, rows.pos, H, plan.mc,
                                         stream_split_len(), (__nv_bfloat16*)cx, 1));
                else
                    BASS_CUDA(launch_pdl(attn_combine_kernel<__nv_bfloat16, 128>, dim3(M, H), dim3(128), 0, st,
                                         (const float*)pa_o, (const float*)pa_ml, rows.pos, H, plan.mc,
                                         stream_split_len(), (__nv_bfloat16*)cx, 1));
                check_launch(ctx);
            }
        } else {
            launch_attention(ctx, m.dtype == BASS_F32 ? BASS_F32 : BASS_BF16, dh, strategy, q, kc, vc, seqs, b.qn,
                             b.off, rows.pos, M, H, kv.cap,
                             kv.n_slots, work_buf, m.part_o, m.part_ml, cx);
        }
        (void)li;
    };
    auto kc_of = [&](int li) { return (void*)((char*)kv.k + li * kv.layer_elems() * es); };
    auto vc_of = [&](int li) { return (void*)((char*)kv.v + li * kv.layer_elems() * es); };
    auto qkv_epi = [&](int li) {
        Epi e{};
        e.out = q;
        e.kc = kc_of(li);
        e.vc = vc_of(li);
        e.row_slot = rows.slot;
        e.row_pos = rows.pos;
        e.d = d; e.dh = dh; e.H = H; e.cap = kv.cap;
        return e;
    };
    Epi r{};
    r.x = x;
    Epi ge{};
    ge.out = f;
    Epi so{};
    so.out = logits_out;
    void* hs = R > 0 ? m.hs.need((size_t)R * d * es, st) : nullptr;

    if (m.int8()) {
        // W8A8 forward (ref:model.py:211-246 with `quantized`): every linear
        // layer takes a per-token int8 input (its LayerNorm / GELU / the
        // attention context quantized by one row kernel) and dequantizes in the
        // GEMM epilogue; q / k / v are fake-quantized per (token, head) on
        // their way to the attention and the cache.
        const int RM = std::max(M, R);
        int8_t* xq = (int8_t*)m.xq.need((size_t)RM * 4 * d, st);
        // per-token scales [RM] | FC amax [RM]
        double* xs = (double*)m.xs.need((size_t)RM * (8 + 4), st);
        float* amax_fc = (float*)(xs + RM);
        float* f32 = (float*)f;
        BASS_CUDA(launch_pdl(embed_kernel<__nv_bfloat16>, dim3(M), dim3(256), 0, st,
                             (const __nv_bfloat16*)m.tok_emb, (const __nv_bfloat16*)m.pos_emb, rows, proposals,
                             pstride, d, x, (float*)nullptr, (float*)nullptr, (__nv_bfloat16*)nullptr,
                             (const float*)nullptr));
        check_launch(ctx);
        auto ln_q = [&](const float* g_, const float* b_, const int32_t* gather, int nrows) {
            ProfScope prof(ctx, BASS_PROF_NORM, (double)nrows * d * 5.0);
            BASS_CUDA(launch_pdl(ln_quant_kernel, dim3(nrows), dim3(LN_THREADS), 0, st, (const float*)x, gather, g_,
                                 b_, d, xq, xs, (float*)nullptr, 0, amax_fc, ctx->trace(nrows, BASS_TR_NORM)));
            check_launch(ctx);
        };
        Epi ef{};
        ef.out = f32;
        ef.amax = amax_fc;
        const int qchunks = (4 * d + QR_CHUNK - 1) / QR_CHUNK, cchunks = (d + QR_CHUNK - 1) / QR_CHUNK;
        for (int li = 0; li < g.n_layer; ++li) {
            const bass_layer& L = m.layers[li];
            ln_q(L.ln1_g, L.ln1_b, nullptr, M);
            // q / k / v fake-quantized per (token, head) in the QKV epilogue
            gemm_i8(m, EPI_QKV, xq, xs, L.wqkv, L.sqkv, M, 3 * d, d, qkv_epi(li));
            run_attention(li, kc_of(li), vc_of(li));
            {
                ProfScope prof(ctx, BASS_PROF_NORM, (double)M * d * 3.0);
                BASS_CUDA(launch_pdl(quant_ctx_kernel, dim3(M, cchunks), dim3(256), 0, st, (const __nv_bfloat16*)cx,
                                     d, xq, xs, ctx->trace(M * cchunks, BASS_TR_NORM)));
                check_launch(ctx);
            }
            gemm_i8(m, EPI_RESID, xq, xs, L.wo, L.so, M, d, d, r);
            ln_q(L.ln2_g, L.ln2_b, nullptr, M);
            gemm_i8(m, EPI_GELU, xq, xs, L.wfc, L.sfc, M, 4 * d, d, ef);
            {
                ProfScope prof(ctx, BASS_PROF_NORM, (double)M * 4 * d * 5.0);
                BASS_CUDA(launch_pdl(quant_amax_rows_kernel, dim3(M, qchunks), dim3(256), 0, st, (const float*)f32,
                                     4 * d, (const float*)amax_fc, xq, xs, ctx->trace(M * qchunks, BASS_TR_NORM)));
                check_launch(ctx);
            }
            gemm_i8(m, EPI_RESID, xq, xs, L.wproj, L.sproj, M, d, 4 * d, r);
        }
        if (R > 0) {
            ln_q(m.lnf_g, m.lnf_b, lrows, R);
            m.dev_rows = devp ? pre->r_act : nullptr;
            gemm_i8(m, EPI_STORE, xq, xs, m.head, m.shead, R, V, d, so);
        }
        return;
    }

    // LayerNorms folded into the QKV / FC GEMMs (bf16 tcgen05 path):
    //   LN(x) W^T = rstd * (((x - K) * g) W^T - (mean - K) * c) + e,  c = W g, e = W b,
    // for any per-row shift K.  The embedding and the residual GEMMs write
    // X = bf16((x - K) * g_next) and per-(128-column tile, row) sums of
    // (x - K) and (x - K)^2 with K ~ the row mean, so neither the bf16 operand
    // nor the variance loses the row's deviations when |mean| >> std; the
    // next GEMM applies rstd and (mean - K) in its epilogue — no LayerNorm
    // kernels between projections.  K: the embedding writes each row's exact
    // mean to `kmean`; every LayerNorm consumer (QKV, FC) turns it into the
    // exact mean of the stream it normalised (K + mean(x - K)), which is the
    // shift the following residual GEMM centres on (the mean of the stream it
    // adds into).
    const bool lnfuse = uses_ln_fold(m);
    const int stat_tiles = (d + 127) / 128;
    const bool headfold = tc_gemm_supported(m, V, d);
    float *lstats = nullptr, *kmean = nullptr;
    if (lnfuse) {
        if (!m.lnfold_valid) {
            // lazily computed per weight upload; never inside a stream capture
            // (forward_prepare runs it first), or the constants would be computed
            // only when the captured graph replays
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            BASS_CUDA(cudaStreamIsCapturing(st, &cs));
            if (cs != cudaStreamCaptureStatusNone)
                throw Error(BASS_ERR_STATE, "folded-LayerNorm constants missing while capturing (forward_prepare)");
        }
        ln_fold_prepare(m);
        const size_t slot = (size_t)stat_tiles * (M + R) * 2;   // + gathered head rows
        lstats = (float*)m.lnstats.need((slot + (size_t)M) * 4, st);
        kmean = lstats + slot;
    }
    if (m.dtype == BASS_BF16)
        BASS_CUDA(launch_pdl(embed_kernel<__nv_bfloat16>, dim3(M), dim3(256), 0, st,
                             (const __nv_bfloat16*)m.tok_emb, (const __nv_bfloat16*)m.pos_emb, rows, proposals,
                             pstride, d, x, lstats, kmean, lnfuse ? (__nv_bfloat16*)h : (__nv_bfloat16*)nullptr,
                             (const float*)m.layers[0].ln1_g));
    else
        BASS_CUDA(launch_pdl(embed_kernel<float>, dim3(M), dim3(128), 0, st, (const float*)m.tok_emb,
                             (const float*)m.pos_emb, rows, proposals, pstride, d, x, (float*)nullptr,
                             (float*)nullptr, (__nv_bfloat16*)nullptr, (const float*)nullptr));
    check_launch(ctx);
    if (lnfuse) {
        const size_t per = (size_t)(2 * 3 * d + 2 * 4 * d);
        const float* fold = (const float*)m.lnfold.p;
        // residual producer: x += acc, statistics of x - K (K = kmean), X of the next GEMM
        auto resid_epi = [&](const float* g_next) {
            Epi e = r;
            e.stats = lstats;
            e.shift = kmean;
            e.xb = (__nv_bfloat16*)h;
            e.xg = g_next;
            return e;
        };
        for (int li = 0; li < g.n_layer; ++li) {
            const bass_layer& L = m.layers[li];
            const float* fl = fold + per * li;
            const TcNorm n1{lstats, fl, fl + 3 * d, kmean, li == 0 ? 1 : stat_tiles};   // embedding: one whole-row tile
            gemm(m, EPI_QKV, h, L.wqkv, M, 3 * d, d, qkv_epi(li), m.packed, &n1);
            run_attention(li, kc_of(li), vc_of(li));
            // x += ctx Wo^T; X of FC = bf16((x - K) * ln2_g)
            gemm(m, EPI_RESID, cx, L.wo, M, d, d, resid_epi(L.ln2_g), m.packed);
            const TcNorm n2{lstats, fl + 6 * d, fl + 10 * d, kmean, stat_tiles};
            gemm(m, EPI_GELU, h, L.wfc, M, 4 * d, d, ge, m.packed, &n2);
            // x += f Wproj^T; X of the next QKV (or of the head: final LayerNorm
            // folded) = bf16((x - K) * g)
            Epi rp = r;
            if (li + 1 < g.n_layer) rp = resid_epi(m.layers[li + 1].ln1_g);
            else if (R > 0 && headfold) rp = resid_epi(m.lnf_g);
            gemm(m, EPI_RESID, f, L.wproj, M, d, 4 * d, rp, m.packed);
        }
        if (R > 0 && headfold) {
            // every logit row goes through the same folded path (a row's bits
            // never depend on whether the block also carried prompt rows)
            bool ident = R == M;
            for (int i = 0; ident && i < R; ++i) ident = b.logit_rows[i] == i;
            const float* hf = (const float*)m.lnfold.p + per * g.n_layer;
            const void* X = h;
            const float* hst = lstats;
            if (!ident) {
                float* cst = lstats + (size_t)stat_tiles * M * 2;
                BASS_CUDA(launch_pdl(head_gather_kernel, dim3(R), dim3(128), 0, st, (const __nv_bfloat16*)h,
                                     (const float2*)lstats, lrows, M, R, d, stat_tiles, (__nv_bfloat16*)hs,
                                     (float2*)cst));
                check_launch(ctx);
                X = hs;
                hst = cst;
            }
            const TcNorm nh{hst, hf, hf + V, nullptr, stat_tiles};
            m.dev_rows = devp ? pre->r_act : nullptr;
            gemm(m, EPI_STORE, X, m.head, R, V, d, so, m.packed, &nh);
        } else if (R > 0) {
            launch_layernorm_any(m, x, lrows, m.lnf_g, m.lnf_b, R, hs);
            gemm(m, EPI_STORE, hs, m.head, R, V, d, so, m.packed);
        }
        return;
    }

    for (int li = 0; li < g.n_layer; ++li) {
        const bass_layer& L = m.layers[li];
        launch_layernorm_any(m, x, nullptr, L.ln1_g, L.ln1_b, M, h);
        gemm(m, EPI_QKV, h, L.wqkv, M, 3 * d, d, qkv_epi(li), m.packed);
        run_attention(li, kc_of(li), vc_of(li));
        gemm(m, EPI_RESID, cx, L.wo, M, d, d, r, m.packed);
        launch_layernorm_any(m, x, nullptr, L.ln2_g, L.ln2_b, M, h);
        gemm(m, EPI_GELU, h, L.wfc, M, 4 * d, d, ge, m.packed);
        gemm(m, EPI_RESID, f, L.wproj, M, d, 4 * d, r, m.packed);
    }
    if (R > 0) {
        launch_layernorm_any(m, x, lrows, m.lnf_g, m.lnf_b, R, hs);
        gemm(m, EPI_STORE, hs, m.head, R, V, d, so, m.packed);
    }
}

}  // namespace bass

// ------------------------------------------------------------ C ABI
extern "C" {

int bass_version(void) { return 1; }

int bass_device_arch(int device) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return -1;
    return p.major * 10 + p.minor;
}

int bass_ctx_create(int device, bass_ctx** out) {
    bass_ctx* c = new bass_ctx();
    int rc = guarded(c, [&] {
        BASS_CUDA(cudaSetDevice(device));
        c->device = device;
        BASS_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        BASS_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        c->staging.cap = 64u << 20;
        BASS_CUDA(cudaMallocHost((void**)&c->staging.base, c->staging.cap));
    });
    if (rc != BASS_OK) {
        *out = nullptr;
        static std::string last;
        last = c->err;
        delete c;
        return rc;
    }
    *out = c;
    return BASS_OK;
}

int bass_ctx_destroy(bass_ctx* c) {
    if (!c) return BASS_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (c->staging.base) cudaFreeHost(c->staging.base);
    for (DevBuf* b : {&c->scr_meta, &c->scr_work, &c->scr_po, &c->scr_pml}) b->release();
    delete c;
    return BASS_OK;
}

int bass_ctx_set_stream(bass_ctx* c, void* s) {
    return guarded(c, [&] {
        BASS_CUDA(cudaStreamSynchronize(c->stream));
        if (c->own_stream) cudaStreamDestroy(c->stream);
        c->stream = (cudaStream_t)s;
        c->own_stream = false;
    });
}

int bass_ctx_sync(bass_ctx* c) {
    return guarded(c, [&] { c->sync(); });
}

const char* bass_last_error(const bass_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t bass_ctx_launches(const bass_ctx* c) { return c ? c->launches : 0; }

int bass_ctx_transfer_bytes(const bass_ctx* c, int64_t* h2d, int64_t* d2h) {
    *h2d = c->h2d_bytes;
    *d2h = c->d2h_bytes;
    return BASS_OK;
}

int bass_ctx_profile(bass_ctx* c, int enable) {
    return guarded(c, [&] {
        c->sync();
        c->profile = enable != 0;
        for (int i = 0; i < BASS_PROF_N; ++i) {
            c->prof_ms[i] = c->prof_bytes[i] = c->prof_flops[i] = 0.0;
            c->prof_n[i] = 0;
        }
    });
}

int bass_ctx_profile_read(bass_ctx* c, int cls, int64_t* launches, double* ms, double* bytes, double* flops) {
    return guarded(c, [&] {
        BASS_REQUIRE(cls >= 0 && cls < BASS_PROF_N, "unknown profile class");
        c->sync();
        *launches = c->prof_n[cls];
        *ms = c->prof_ms[cls];
        *bytes = c->prof_bytes[cls];
        *flops = c->prof_flops[cls];
    });
}

int bass_ctx_algo_read(bass_ctx* c, int cls, int64_t* launches, double* bytes, double* flops) {
    return guarded(c, [&] {
        BASS_REQUIRE(cls >= 0 && cls < BASS_PROF_N, "unknown profile class");
        *launches = c->algo_n[cls];
        *bytes = c->algo_bytes[cls];
        *flops = c->algo_flops[cls];
    });
}

// ---------------------------------------------------------------- model
int bass_model_create(bass_ctx* c, const bass_geometry* g, int dtype, bass_model** out) {
    *out = nullptr;
    return guarded(c, [&] {
        BASS_REQUIRE(g->n_layer >= 1 && g->n_head >= 1 && g->d_model >= 1 && g->d_head >= 1 &&
                         g->vocab_size >= 1 && g->max_seq_len >= 1,
                     "geometry: all sizes must be >= 1");
        BASS_REQUIRE(g->d_model == g->n_head * g->d_head, "geometry: d_model != n_head * d_head");
        BASS_REQUIRE(g->d_model % 4 == 0 && g->d_model <= 4 * LN_THREADS * LN_NV,
                     "d_model must be a multiple of 4 and <= 8192");
        BASS_REQUIRE(dtype == BASS_BF16 || dtype == BASS_F32 || dtype == BASS_INT8,
                     "dtype must be BASS_BF16, BASS_F32 or BASS_INT8");
        BASS_REQUIRE(dtype != BASS_INT8 || (g->d_model % 128 == 0 && g->vocab_size >= 128),
                     "INT8 models need d_model % 128 == 0 and vocab_size >= 128 (tcgen05 kind::i8 tiles)");
        BASS_REQUIRE(g->d_head == 16 || g->d_head == 32 || g->d_head == 64 || g->d_head == 128,
                     "d_head must be 16, 32, 64 or 128");
        BASS_CUDA(cudaSetDevice(c->device));
        bass_model* m = new bass_model();
        m->ctx = c;
        m->g = *g;
        m->dtype = dtype;
        m->esize = dtype == BASS_F32 ? 4 : 2;
        m->wsize = dtype == BASS_INT8 ? 1 : m->esize;
        const int64_t d = g->d_model, V = g->vocab_size, S = g->max_seq_len, L = g->n_layer;
        // bf16 / int8 GEMM weights live in the packed tile layout (rows padded to 128)
        m->packed = (dtype == BASS_BF16 && d % 64 == 0) || dtype == BASS_INT8;
        auto rows = [&](int64_t N) { return m->packed ? packed_rows(N) : N; };
        const int64_t per_layer = (rows(3 * d) + rows(d) + rows(4 * d)) * d + rows(d) * 4 * d;
        const int64_t emb = V * d + S * d, mats = L * per_layer + rows(V) * d;
        m->weight_bytes = emb * (int64_t)m->esize + mats * (int64_t)m->wsize;
        BASS_CUDA(cudaMalloc(&m->wblob, (size_t)m->weight_bytes));
        const int64_t nf = L * 4 * d + 2 * d;
        BASS_CUDA(cudaMalloc((void**)&m->fblob, (size_t)nf * 4));
        if (dtype == BASS_INT8) BASS_CUDA(cudaMalloc((void**)&m->sblob, (size_t)(L * 9 * d + V) * 8));
        char* p = (char*)m->wblob;
        auto take = [&](int64_t n) { void* r = p; p += n * m->esize; return r; };
        auto take_w = [&](int64_t n) { void* r = p; p += n * m->wsize; return r; };
        m->tok_emb = take(V * d);
        m->pos_emb = take(S * d);
        float* fp = m->fblob;
        double* sp = m->sblob;
        auto take_s = [&](int64_t n) { double* r = sp; if (sp) sp += n; return r; };
        m->layers.resize(L);
        for (int i = 0; i < L; ++i) {
            bass_layer& ly = m->layers[i];
            ly.wqkv = take_w(rows(3 * d) * d);
            ly.wo = take_w(rows(d) * d);
            ly.wfc = take_w(rows(4 * d) * d);
            ly.wproj = take_w(rows(d) * 4 * d);
            ly.ln1_g = fp; fp += d;
            ly.ln1_b = fp; fp += d;
            ly.ln2_g = fp; fp += d;
            ly.ln2_b = fp; fp += d;
            ly.sqkv = take_s(3 * d);
            ly.so = take_s(d);
            ly.sfc = take_s(4 * d);
            ly.sproj = take_s(d);
        }
        m->head = take_w(rows(V) * d);
        m->shead = take_s(V);
        m->lnf_g = fp; fp += d;
        m->lnf_b = fp; fp += d;
        // LN defaults (gain 1, bias 0) — ref:model.py:121-130
        for (int i = 0; i < L; ++i) {
            fill_f32<<<32, 256, 0, c->stream>>>(m->layers[i].ln1_g, d, 1.f);
            fill_f32<<<32, 256, 0, c->stream>>>(m->layers[i].ln1_b, d, 0.f);
            fill_f32<<<32, 256, 0, c->stream>>>(m->layers[i].ln2_g, d, 1.f);
            fill_f32<<<32, 256, 0, c->stream>>>(m->layers[i].ln2_b, d, 0.f);
        }
        fill_f32<<<32, 256, 0, c->stream>>>(m->lnf_g, d, 1.f);
        fill_f32<<<32, 256, 0, c->stream>>>(m->lnf_b, d, 0.f);
        BASS_CUDA(cudaGetLastError());
        BASS_CUDA(cudaStreamSynchronize(c->stream));
        *out = m;
    });
}

int bass_model_destroy(bass_model* m) {
    if (!m) return BASS_OK;
    cudaSetDevice(m->ctx->device);
    cudaStreamSynchronize(m->ctx->stream);
    tc_release(*m);
    cudaFree(m->wblob);
    cudaFree(m->fblob);
    if (m->sblob) cudaFree(m->sblob);
    for (DevBuf* b : {&m->x, &m->h, &m->q, &m->ctxb, &m->f, &m->hs, &m->meta, &m->part_o, &m->part_ml,
                      &m->logits_tmp, &m->lnstats, &m->lnfold, &m->attn_work, &m->xq, &m->xs})
        b->release();
    delete m;
    return BASS_OK;
}

int bass_model_set_weight(bass_model* m, int tensor, int layer, const float* host, int64_t n) {
    return guarded(m->ctx, [&] {
        m->lnfold_valid = false;
        const bass_geometry& g = m->g;
        const int64_t d = g.d_model, V = g.vocab_size, S = g.max_seq_len;
        BASS_REQUIRE(tensor >= BASS_W_TOK_EMB && tensor <= BASS_W_HEAD, "unknown tensor id");
        const bool per_layer = tensor >= BASS_W_LN1_G && tensor <= BASS_W_LN2_B;
        BASS_REQUIRE(!per_layer || (layer >= 0 && layer < g.n_layer), "layer index out of range");
        cudaStream_t st = m->ctx->stream;
        auto upload_tmp = [&](int64_t count) {
            BASS_REQUIRE(n == count, "geometry: element count does not match the tensor");
            float* tmp;
            BASS_CUDA(cudaMallocAsync((void**)&tmp, count * 4, st));
            BASS_CUDA(cudaMemcpyAsync(tmp, host, count * 4, cudaMemcpyHostToDevice, st));
            return tmp;
        };
        auto put_matrix = [&](int64_t K, int64_t N, void* dst, int64_t row_off, double* scale = nullptr) {
            // reference [K, N] -> device output-major rows [row_off + n][K]
            float* tmp = upload_tmp(K * N);
            dim3 grid((N + 31) / 32, (K + 31) / 32), blk(32, 8);
            if (m->int8()) {
                // fp32 [N, K], then per-output-channel int8 quantization into the
                // packed layout (ref:model.py:135-143 prepare_quantized)
                float* t2;
                BASS_CUDA(cudaMallocAsync((void**)&t2, K * N * 4, st));
                transpose_convert<<<grid, blk, 0, st>>>(tmp, (int)K, (int)N, t2, K, 0, false);
                quant_weight_rows_kernel<<<(unsigned)N, 256, 0, st>>>(t2, (int)K, (int8_t*)dst, row_off, scale);
                BASS_CUDA(cudaGetLastError());
                BASS_CUDA(cudaFreeAsync(t2, st));
                BASS_CUDA(cudaFreeAsync(tmp, st));
                return;
            }
            if (m->dtype == BASS_BF16)
                transpose_convert<<<grid, blk, 0, st>>>(tmp, (int)K, (int)N, (__nv_bfloat16*)dst, K, row_off,
                                                        m->packed);
            else
                transpose_convert<<<grid, blk, 0, st>>>(tmp, (int)K, (int)N, (float*)dst, K, row_off, false);
            BASS_CUDA(cudaGetLastError());
            BASS_CUDA(cudaFreeAsync(tmp, st));
        };
        auto put_rows = [&](int64_t count, void* dst) {
            float* tmp = upload_tmp(count);
            if (m->dtype != BASS_F32) convert_copy<<<256, 256, 0, st>>>(tmp, count, (__nv_bfloat16*)dst);
            else convert_copy<<<256, 256, 0, st>>>(tmp, count, (float*)dst);
            BASS_CUDA(cudaGetLastError());
            BASS_CUDA(cudaFreeAsync(tmp, st));
        };
        auto put_f32 = [&](float* dst) {
            BASS_REQUIRE(n == d, "geometry: LN parameter must have d_model elements");
            BASS_CUDA(cudaMemcpyAsync(dst, host, d * 4, cudaMemcpyHostToDevice, st));
        };
        const bool layer_mat = tensor >= BASS_W_WQ && tensor <= BASS_W_PROJ && tensor != BASS_W_LN2_G &&
                               tensor != BASS_W_LN2_B;
        if (layer_mat) BASS_REQUIRE(layer >= 0 && layer < g.n_layer, "layer index out of range");
        switch (tensor) {
            case BASS_W_TOK_EMB: put_rows(V * d, m->tok_emb); break;
            case BASS_W_POS_EMB: put_rows(S * d, m->pos_emb); break;
            case BASS_W_LN1_G: put_f32(m->layers[layer].ln1_g); break;
            case BASS_W_LN1_B: put_f32(m->layers[layer].ln1_b); break;
            case BASS_W_LN2_G: put_f32(m->layers[layer].ln2_g); break;
            case BASS_W_LN2_B: put_f32(m->layers[layer].ln2_b); break;
            case BASS_W_WQ: put_matrix(d, d, m->layers[layer].wqkv, 0, m->layers[layer].sqkv); break;
            case BASS_W_WK: put_matrix(d, d, m->layers[layer].wqkv, d, m->layers[layer].sqkv); break;
            case BASS_W_WV: put_matrix(d, d, m->layers[layer].wqkv, 2 * d, m->layers[layer].sqkv); break;
            case BASS_W_WO: put_matrix(d, d, m->layers[layer].wo, 0, m->layers[layer].so); break;
            case BASS_W_FC: put_matrix(d, 4 * d, m->layers[layer].wfc, 0, m->layers[layer].sfc); break;
            case BASS_W_PROJ: put_matrix(4 * d, d, m->layers[layer].wproj, 0, m->layers[layer].sproj); break;
            case BASS_W_LNF_G: put_f32(m->lnf_g); break;
            case BASS_W_LNF_B: put_f32(m->lnf_b); break;
            case BASS_W_HEAD: put_matrix(d, V, m->head, 0, m->shead); break;
        }
        BASS_CUDA(cudaStreamSynchronize(st));
    });
}

// read one tensor back in the reference layout (inverse of bass_model_set_weight)
int bass_model_get_weight(const bass_model* mc, int tensor, int layer, float* host, int64_t n) {
    bass_model* m = const_cast<bass_model*>(mc);
    return guarded(m->ctx, [&] {
        const bass_geometry& g = m->g;
        const int64_t d = g.d_model, V = g.vocab_size, S = g.max_seq_len;
        BASS_REQUIRE(tensor >= BASS_W_TOK_EMB && tensor <= BASS_W_HEAD, "unknown tensor id");
        const bool per_layer = tensor >= BASS_W_LN1_G && tensor <= BASS_W_PROJ;
        BASS_REQUIRE(!per_layer || (layer >= 0 && layer < g.n_layer), "layer index out of range");
        cudaStream_t st = m->ctx->stream;
        float* tmp = nullptr;
        auto get_matrix = [&](int64_t K, int64_t N, const void* src, int64_t row_off, const double* scale = nullptr) {
            BASS_REQUIRE(n == K * N, "geometry: element count does not match the tensor");
            BASS_CUDA(cudaMallocAsync((void**)&tmp, K * N * 4, st));
            dim3 grid((N + 31) / 32, (K + 31) / 32), blk(32, 8);
            if (m->int8())   // dequantized values payload * scale (ref:quant.py:86-95)
                dequant_gather_kernel<<<1184, 256, 0, st>>>((const int8_t*)src, scale, (int)K, (int)N, row_off, tmp,
                                                            nullptr);
            else if (m->dtype == BASS_BF16)
                transpose_gather<<<grid, blk, 0, st>>>((const __nv_bfloat16*)src, (int)K, (int)N, tmp, K, row_off,
                                                       m->packed);
            else
                transpose_gather<<<grid, blk, 0, st>>>((const float*)src, (int)K, (int)N, tmp, K, row_off, false);
        };
        auto get_rows = [&](int64_t count, const void* src) {
            BASS_REQUIRE(n == count, "geometry: element count does not match the tensor");
            BASS_CUDA(cudaMallocAsync((void**)&tmp, count * 4, st));
            if (m->dtype != BASS_F32) to_f32<<<256, 256, 0, st>>>((const __nv_bfloat16*)src, count, tmp);
            else to_f32<<<256, 256, 0, st>>>((const float*)src, count, tmp);
        };
        auto get_f32 = [&](const float* src) {
            BASS_REQUIRE(n == d, "geometry: LN parameter must have d_model elements");
            BASS_CUDA(cudaMemcpyAsync(host, src, d * 4, cudaMemcpyDeviceToHost, st));
        };
        const bass_layer* L = per_layer ? &m->layers[layer] : nullptr;
        switch (tensor) {
            case BASS_W_TOK_EMB: get_rows(V * d, m->tok_emb); break;
            case BASS_W_POS_EMB: get_rows(S * d, m->pos_emb); break;
            case BASS_W_LN1_G: get_f32(L->ln1_g); break;
            case BASS_W_LN1_B: get_f32(L->ln1_b); break;
            case BASS_W_LN2_G: get_f32(L->ln2_g); break;
            case BASS_W_LN2_B: get_f32(L->ln2_b); break;
            case BASS_W_WQ: get_matrix(d, d, L->wqkv, 0, L->sqkv); break;
            case BASS_W_WK: get_matrix(d, d, L->wqkv, d, L->sqkv); break;
            case BASS_W_WV: get_matrix(d, d, L->wqkv, 2 * d, L->sqkv); break;
            case BASS_W_WO: get_matrix(d, d, L->wo, 0, L->so); break;
            case BASS_W_FC: get_matrix(d, 4 * d, L->wfc, 0, L->sfc); break;
            case BASS_W_PROJ: get_matrix(4 * d, d, L->wproj, 0, L->sproj); break;
            case BASS_W_LNF_G: get_f32(m->lnf_g); break;
            case BASS_W_LNF_B: get_f32(m->lnf_b); break;
            case BASS_W_HEAD: get_matrix(d, V, m->head, 0, m->shead); break;
        }
        BASS_CUDA(cudaGetLastError());
        if (tmp) {
            BASS_CUDA(cudaMemcpyAsync(host, tmp, n * 4, cudaMemcpyDeviceToHost, st));
            BASS_CUDA(cudaFreeAsync(tmp, st));
        }
        BASS_CUDA(cudaStreamSynchronize(st));
    });
}

// one (layer, matrix) of an int8 model: where its packed rows and scales live
struct QMat {
    const int8_t* w;
    const double* s;
    int64_t K, N, row_off;
};
static QMat qmat(const bass_model* m, int tensor, int layer) {
    const int64_t d = m->g.d_model;
    if (tensor == BASS_W_HEAD) return {(const int8_t*)m->head, m->shead, d, m->g.vocab_size, 0};
    const bass_layer& L = m->layers[layer];
    switch (tensor) {
        case BASS_W_WQ: return {(const int8_t*)L.wqkv, L.sqkv, d, d, 0};
        case BASS_W_WK: return {(const int8_t*)L.wqkv, L.sqkv, d, d, d};
        case BASS_W_WV: return {(const int8_t*)L.wqkv, L.sqkv, d, d, 2 * d};
        case BASS_W_WO: return {(const int8_t*)L.wo, L.so, d, d, 0};
        case BASS_W_FC: return {(const int8_t*)L.wfc, L.sfc, d, 4 * d, 0};
        case BASS_W_PROJ: return {(const int8_t*)L.wproj, L.sproj, 4 * d, d, 0};
        default: throw Error(BASS_ERR_VALUE, "tensor is not a quantized matrix");
    }
}

int bass_model_get_qweight(const bass_model* mc, int tensor, int layer, int8_t* payload, double* scales, int64_t n) {
    bass_model* m = const_cast<bass_model*>(mc);
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(m->int8(), "not an INT8 model");
        BASS_REQUIRE(tensor == BASS_W_HEAD || (layer >= 0 && layer < m->g.n_layer), "layer index out of range");
        const QMat q = qmat(m, tensor, layer);
        BASS_REQUIRE(n == q.K * q.N, "geometry: element count does not match the tensor");
        cudaStream_t st = m->ctx->stream;
        int8_t* tmp;
        BASS_CUDA(cudaMallocAsync((void**)&tmp, n, st));
        dequant_gather_kernel<<<1184, 256, 0, st>>>(q.w, q.s, (int)q.K, (int)q.N, q.row_off, nullptr, tmp);
        BASS_CUDA(cudaGetLastError());
        BASS_CUDA(cudaMemcpyAsync(payload, tmp, n, cudaMemcpyDeviceToHost, st));
        BASS_CUDA(cudaMemcpyAsync(scales, q.s + q.row_off, q.N * 8, cudaMemcpyDeviceToHost, st));
        BASS_CUDA(cudaFreeAsync(tmp, st));
        BASS_CUDA(cudaStreamSynchronize(st));
    });
}

int bass_model_init_random(bass_model* m, uint64_t seed, float std) {
    return guarded(m->ctx, [&] {
        m->lnfold_valid = false;
        if (m->int8()) {
            // bf16 embeddings; every matrix drawn in fp32 [N, K] and quantized per channel
            cudaStream_t st = m->ctx->stream;
            const int64_t d = m->g.d_model, V = m->g.vocab_size, S = m->g.max_seq_len;
            random_normal<<<m->ctx->sm_count * 8, 256, 0, st>>>((__nv_bfloat16*)m->wblob, (V + S) * d, seed, std);
            float* t;
            BASS_CUDA(cudaMallocAsync((void**)&t, (size_t)std::max(V, 4 * d) * d * 4, st));
            uint64_t sub = 0;
            auto one = [&](const QMat& q) {
                random_normal<<<m->ctx->sm_count * 8, 256, 0, st>>>(t, q.K * q.N, seed * 0x9E3779B97F4A7C15ull + ++sub, std);
                quant_weight_rows_kernel<<<(unsigned)q.N, 256, 0, st>>>(t, (int)q.K, const_cast<int8_t*>(q.w),
                                                                         q.row_off, const_cast<double*>(q.s));
            };
            for (int l = 0; l < m->g.n_layer; ++l)
                for (int tid : {BASS_W_WQ, BASS_W_WK, BASS_W_WV, BASS_W_WO, BASS_W_FC, BASS_W_PROJ})
                    one(qmat(m, tid, l));
            one(qmat(m, BASS_W_HEAD, 0));
            BASS_CUDA(cudaGetLastError());
            BASS_CUDA(cudaFreeAsync(t, st));
            BASS_CUDA(cudaStreamSynchronize(st));
            return;
        }
        const int64_t n = m->weight_bytes / (int64_t)m->esize;
        if (m->dtype == BASS_BF16)
            random_normal<<<m->ctx->sm_count * 8, 256, 0, m->ctx->stream>>>((__nv_bfloat16*)m->wblob, n, seed, std);
        else
            random_normal<<<m->ctx->sm_count * 8, 256, 0, m->ctx->stream>>>((float*)m->wblob, n, seed, std);
        BASS_CUDA(cudaGetLastError());
        BASS_CUDA(cudaStreamSynchronize(m->ctx->stream));
    });
}

int bass_model_set_gemm(bass_model* m, int mode) {
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(mode >= BASS_GEMM_AUTO && mode <= BASS_GEMM_TC, "unknown gemm mode");
        m->gemm_mode = mode;
    });
}

int bass_model_set_split(bass_model* m, int N, int K, int splits) {
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(splits >= 0 && splits <= 8, "split count must be in [0, 8] (0: the default rule)");
        tc_set_split(*m, N, K, splits);
    });
}

int64_t bass_model_weight_bytes(const bass_model* m) { return m ? m->weight_bytes : 0; }

// ------------------------------------------------------------------- KV
int bass_kv_create(bass_model* m, int n_slots, int capacity, bass_kv** out) {
    *out = nullptr;
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(n_slots >= 1 && capacity >= 1, "geometry: cache sizes must be positive");
        BASS_REQUIRE(capacity <= m->g.max_seq_len, "capacity exceeds max_seq_len");
        bass_kv* kv = new bass_kv();
        kv->m = m;
        kv->ctx = m->ctx;
        kv->n_slots = n_slots;
        kv->cap = capacity;
        kv->len.assign(n_slots, 0);
        const size_t bytes = kv->layer_elems() * m->g.n_layer * m->esize;
        BASS_CUDA(cudaMalloc(&kv->k, bytes));
        BASS_CUDA(cudaMalloc(&kv->v, bytes));
        // finite contents everywhere: masked keys get P = 0, and 0 * (finite) = 0
        BASS_CUDA(cudaMemset(kv->k, 0, bytes));
        BASS_CUDA(cudaMemset(kv->v, 0, bytes));
        *out = kv;
    });
}

int bass_kv_destroy(bass_kv* kv) {
    if (!kv) return BASS_OK;
    cudaStreamSynchronize(kv->ctx->stream);
    cudaFree(kv->k);
    cudaFree(kv->v);
    delete kv;
    return BASS_OK;
}

int bass_kv_lengths(const bass_kv* kv, int32_t* out) {
    std::memcpy(out, kv->len.data(), kv->len.size() * 4);
    return BASS_OK;
}

int bass_kv_truncate(bass_kv* kv, int n, const int32_t* slots, const int32_t* lens) {
    return guarded(kv->m->ctx, [&] {
        for (int i = 0; i < n; ++i) {
            BASS_REQUIRE(slots[i] >= 0 && slots[i] < kv->n_slots, "slot out of range");
            BASS_REQUIRE(lens[i] >= 0, "negative length");
            BASS_REQUIRE(lens[i] <= kv->len[slots[i]], "truncate to " + std::to_string(lens[i]) +
                                                           " exceeds current length " +
                                                           std::to_string(kv->len[slots[i]]));
        }
        for (int i = 0; i < n; ++i) kv->len[slots[i]] = lens[i];
    });
}

int bass_forward_ragged(bass_model* m, bass_kv* kv, int n_seq, const int32_t* slots, const int32_t* cu_q,
                        const int32_t* tokens, int strategy, int rows_mode, float* logits_host) {
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(n_seq >= 1, "active_seqs and new_tokens must align and be non-empty");
        BASS_REQUIRE(kv->m == m, "cache belongs to another model");
        const bass_geometry& g = m->g;
        Batch b;
        std::vector<char> seen(kv->n_slots, 0);
        for (int i = 0; i < n_seq; ++i) {
            const int s = slots[i], n = cu_q[i + 1] - cu_q[i];
            BASS_REQUIRE(s >= 0 && s < kv->n_slots, "slot out of range");
            BASS_REQUIRE(!seen[s], "duplicate slot in one forward");
            seen[s] = 1;
            BASS_REQUIRE(n >= 1, "sequence " + std::to_string(s) + ": empty token block");
            const int off = kv->len[s];
            BASS_REQUIRE(off + n <= g.max_seq_len, "sequence " + std::to_string(s) + ": context " +
                                                       std::to_string(off + n) + " exceeds max_seq_len " +
                                                       std::to_string(g.max_seq_len));
            BASS_REQUIRE(off + n <= kv->cap, "sequence " + std::to_string(s) + ": context exceeds cache capacity");
            for (int t = cu_q[i]; t < cu_q[i + 1]; ++t)
                BASS_REQUIRE(tokens[t] >= 0 && tokens[t] < g.vocab_size,
                             "sequence " + std::to_string(s) + ": token id outside vocab");
            b.add_seq(s, off, tokens + cu_q[i], n);
            if (rows_mode == 1) b.logit_rows.push_back(b.rows() - 1);
        }
        if (rows_mode == 0)
            for (int r = 0; r < b.rows(); ++r) b.logit_rows.push_back(r);
        const size_t R = b.logit_rows.size();
        float* lg = (float*)m->logits_tmp.need(R * g.vocab_size * 4, m->ctx->stream);
        forward(*m, *kv, b, strategy, lg, nullptr, 0);
        BASS_CUDA(cudaMemcpyAsync(logits_host, lg, R * g.vocab_size * 4, cudaMemcpyDeviceToHost, m->ctx->stream));
        m->ctx->sync();
        for (int i = 0; i < n_seq; ++i) kv->len[slots[i]] += cu_q[i + 1] - cu_q[i];
    });
}

// ------------------------------------------------------ standalone kernels
int bass_gemm_bench(bass_model* m, int mode, int M, int N, int K, const void* x, const void* w, float* y, int reps,
                    int n_w, double* ms_per_launch) {
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(reps >= 1, "reps must be >= 1");
        const bool packed = mode == 3;   // tcgen05 on packed copies of the weights
        if (packed) mode = BASS_GEMM_TC;
        const int saved = m->gemm_mode;
        m->gemm_mode = mode;
        Epi e{};
        e.out = y;
        void* wp = nullptr;
        if (packed) {
            BASS_CUDA(cudaMalloc(&wp, (size_t)packed_rows(N) * K * 2 * n_w));
            pack_weights(m->ctx->stream, w, wp, N, K, n_w);
            w = wp;
        }
        cudaEvent_t a, b;
        BASS_CUDA(cudaEventCreate(&a));
        BASS_CUDA(cudaEventCreate(&b));
        // launch i streams weight copy i % n_w (n_w copies > L2 defeat caching)
        const size_t wbytes = (size_t)(packed ? packed_rows(N) : N) * K * m->esize;
        for (int i = 0; i < n_w; ++i) gemm(*m, EPI_STORE, x, (const char*)w + i * wbytes, M, N, K, e, packed);   // warm
        BASS_CUDA(cudaEventRecord(a, m->ctx->stream));
        for (int i = 0; i < reps; ++i)
            gemm(*m, EPI_STORE, x, (const char*)w + (i % n_w) * wbytes, M, N, K, e, packed);
        BASS_CUDA(cudaEventRecord(b, m->ctx->stream));
        m->gemm_mode = saved;
        m->ctx->sync();
        float ms = 0.f;
        BASS_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_per_launch = ms / reps;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (wp) cudaFree(wp);
    });
}

int bass_int_gemm_dequant(bass_ctx* c, int M, int N, int K, const int8_t* a, const double* sa, const int8_t* w,
                          const double* sw, float* out) {
    return guarded(c, [&] {
        BASS_REQUIRE(M >= 1 && N >= 1 && K >= 1, "geometry: GEMM sizes must be positive");
        BASS_REQUIRE(K % 128 == 0 && N >= 128, "int8 GEMM needs K % 128 == 0 and N >= 128");
        cudaStream_t st = c->stream;
        bass_model tmp;   // a weightless int8 'model': only the GEMM state (tensor maps, split rule)
        tmp.ctx = c;
        tmp.dtype = BASS_INT8;
        tmp.esize = 2;
        tmp.wsize = 1;
        tmp.packed = true;
        struct Bufs {
            bass_model* m;
            std::vector<void*> p;
            ~Bufs() {
                for (void* q : p) cudaFree(q);
                tc_release(*m);
            }
        } bufs{&tmp, {}};
        auto dalloc = [&](size_t n) {
            void* q = nullptr;
            BASS_CUDA(cudaMalloc(&q, n));
            bufs.p.push_back(q);
            return q;
        };
        int8_t* ad = (int8_t*)dalloc((size_t)M * K);
        double* sad = (double*)dalloc((size_t)M * 8);
        int8_t* wr = (int8_t*)dalloc((size_t)K * N);
        int8_t* wp = (int8_t*)dalloc((size_t)packed_rows(N) * K);
        double* swd = (double*)dalloc((size_t)N * 8);
        float* od = (float*)dalloc((size_t)M * N * 4);
        BASS_CUDA(cudaMemcpyAsync(ad, a, (size_t)M * K, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(sad, sa, (size_t)M * 8, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(wr, w, (size_t)K * N, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(swd, sw, (size_t)N * 8, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemsetAsync(wp, 0, (size_t)packed_rows(N) * K, st));
        pack_i8_ref_kernel<<<1184, 256, 0, st>>>(wr, K, N, wp);
        BASS_CUDA(cudaGetLastError());
        Epi e{};
        e.out = od;
        gemm_i8(tmp, EPI_STORE, ad, sad, wp, swd, M, N, K, e);
        BASS_CUDA(cudaMemcpyAsync(out, od, (size_t)M * N * 4, cudaMemcpyDeviceToHost, st));
        BASS_CUDA(cudaStreamSynchronize(st));
    });
}

int bass_gemm(bass_model* m, int mode, int M, int N, int K, const void* x, const void* w, float* y) {
    return guarded(m->ctx, [&] {
        BASS_REQUIRE(M >= 1 && N >= 1 && K >= 1, "geometry: GEMM sizes must be positive");
        BASS_REQUIRE(mode == BASS_GEMM_SIMT || mode == BASS_GEMM_TC || mode == 3,
                     "gemm mode must be SIMT, TC or 3 (TC on a packed copy)");
        // mode 3: the weights repacked into the model layout first — the
        // forward's own path (incl. the serial split-K kernel for M > 256)
        const bool packed = mode == 3;
        void* wp = nullptr;
        if (packed) {
            BASS_REQUIRE(m->dtype == BASS_BF16 && K % 64 == 0, "packed GEMM: bf16, K % 64 == 0");
            BASS_CUDA(cudaMalloc(&wp, (size_t)packed_rows(N) * K * 2));
            BASS_CUDA(cudaMemsetAsync(wp, 0, (size_t)packed_rows(N) * K * 2, m->ctx->stream));
            pack_weights(m->ctx->stream, w, wp, N, K, 1);
            w = wp;
            mode = BASS_GEMM_TC;
        }
        const int saved = m->gemm_mode;
        m->gemm_mode = mode;
        Epi e{};
        e.out = y;
        try {
            gemm(*m, EPI_STORE, x, w, M, N, K, e, packed);
        } catch (...) {
            m->gemm_mode = saved;
            if (wp) cudaFree(wp);
            throw;
        }
        m->gemm_mode = saved;
        m->ctx->sync();
        if (wp) cudaFree(wp);
    });
}

int bass_attention(bass_ctx* c, int strategy, int dtype, int n_seq, int n_head, int d_head, const int32_t* cu_q,
                   const int32_t* offsets, const void* q, const void* k, const void* v, int kv_stride, void* out) {
    return guarded(c, [&] {
        BASS_REQUIRE(n_seq >= 1, "empty workload");
        std::vector<int32_t> slot(n_seq), q0(n_seq), qn(n_seq), off(n_seq), row_pos;
        for (int i = 0; i < n_seq; ++i) {
            slot[i] = i;
            q0[i] = cu_q[i];
            qn[i] = cu_q[i + 1] - cu_q[i];
            off[i] = offsets[i];
            BASS_REQUIRE(qn[i] >= 1, "every sequence needs at least one query");
            BASS_REQUIRE(off[i] >= 0 && off[i] + qn[i] <= kv_stride, "offset exceeds history");
            for (int t = 0; t < qn[i]; ++t) row_pos.push_back(off[i] + t);
        }
        const int M = cu_q[n_seq];
        DevBuf &meta = c->scr_meta, &work = c->scr_work, &po = c->scr_po, &pml = c->scr_pml;
        int32_t* dm = (int32_t*)meta.need((4 * (size_t)n_seq + M) * 4, c->stream);
        std::vector<int32_t> hm;
        for (auto* v_ : {&slot, &q0, &qn, &off}) hm.insert(hm.end(), v_->begin(), v_->end());
        hm.insert(hm.end(), row_pos.begin(), row_pos.end());
        upload_i32(c, dm, hm.data(), hm.size());
        Seqs seqs{dm, dm + n_seq, dm + 2 * n_seq, dm + 3 * n_seq};
        launch_attention(c, dtype, d_head, strategy, q, k, v, seqs, qn, off, dm + 4 * n_seq, M, n_head, kv_stride,
                         n_seq, work, po, pml, out);
        c->sync();
    });
}

int bass_trace_enable(bass_ctx* c, int64_t records) {
    return guarded(c, [&] {
        c->sync();
        if (c->trace_buf) cudaFree(c->trace_buf);
        c->trace_buf = nullptr;
        c->trace_cap = c->trace_n = 0;
        if (records > 0) {
            BASS_CUDA(cudaMalloc((void**)&c->trace_buf, (size_t)records * 32));
            BASS_CUDA(cudaMemset(c->trace_buf, 0, (size_t)records * 32));
            c->trace_cap = records;
        }
    });
}

int bass_trace_read(bass_ctx* c, uint64_t* host, int64_t max_records, int64_t* n_out) {
    return guarded(c, [&] {
        c->sync();
        const int64_t n = std::min<int64_t>(max_records, c->trace_n);
        if (n > 0) BASS_CUDA(cudaMemcpy(host, c->trace_buf, (size_t)n * 32, cudaMemcpyDeviceToHost));
        *n_out = n;
        c->trace_n = 0;
    });
}

#ifdef BASS_GEMM_PROBE
}
namespace bass { namespace tc { void gemm_probe_set(void* p, int n, int k); } }
extern "C" {
// debug build: on = 1 arms the stamps for GEMMs of shape (n, k); on = 0
// copies the last such launch's [16][16] globaltimer stamps to `out`
int bass_gemm_probe(int on, int n, int k, unsigned long long* out) {
    static unsigned long long* dp = nullptr;
    if (on) {
        if (!dp) cudaMalloc(&dp, 16 * 16 * 8);
        cudaMemset(dp, 0, 16 * 16 * 8);
        bass::tc::gemm_probe_set(dp, n, k);
    } else if (dp) {
        cudaDeviceSynchronize();
        bass::tc::gemm_probe_set(nullptr, 0, 0);
        cudaMemcpy(out, dp, 16 * 16 * 8, cudaMemcpyDeviceToHost);
    }
    return 0;
}
#endif
#ifdef BASS_ATTN_PROBE
}
namespace bass { namespace ast { void attn_probe_set(void* p); } }
extern "C" {
// debug build: on = 1 arms the stamps (every attention launch overwrites
// them), on = 0 copies the last launch's [16][32] stamps to `out` and disarms
int bass_attn_probe(int on, unsigned long long* out) {
    static unsigned long long* dp = nullptr;
    if (on) {
        if (!dp) cudaMalloc(&dp, 16 * 32 * 8);
        cudaMemset(dp, 0, 16 * 32 * 8);
        bass::ast::attn_probe_set(dp);
    } else if (dp) {
        cudaDeviceSynchronize();
        bass::ast::attn_probe_set(nullptr);
        cudaMemcpy(out, dp, 16 * 32 * 8, cudaMemcpyDeviceToHost);
    }
    return 0;
}
#endif
int bass_attention_bench(bass_ctx* c, int strategy, int n_seq, int n_head, int d_head, const int32_t* cu_q,
                         const int32_t* offsets, const void* q, const void* k, const void* v, int kv_stride, int n_kv,
                         void* out, int reps, double* ms_per_call) {
    return guarded(c, [&] {
        BASS_REQUIRE(n_seq >= 1 && reps >= 1 && n_kv >= 1, "attention bench: bad sizes");
        BASS_REQUIRE(tc_attention_supported(BASS_BF16, d_head), "attention bench: d_head must be 64 or 128");
        const int DHb = d_head;
        std::vector<int32_t> slot(n_seq), q0(n_seq), qn(n_seq), off(n_seq), row_pos;
        for (int i = 0; i < n_seq; ++i) {
            slot[i] = i;
            q0[i] = cu_q[i];
            qn[i] = cu_q[i + 1] - cu_q[i];
            off[i] = offsets[i];
            BASS_REQUIRE(qn[i] >= 1 && off[i] >= 0 && off[i] + qn[i] <= kv_stride, "attention bench: bad lengths");
            for (int t = 0; t < qn[i]; ++t) row_pos.push_back(off[i] + t);
        }
        const int M = cu_q[n_seq], H = n_head;
        DevBuf &meta = c->scr_meta, &work = c->scr_work, &po = c->scr_po, &pml = c->scr_pml;
        int32_t* dm = (int32_t*)meta.need((4 * (size_t)n_seq + M) * 4, c->stream);
        std::vector<int32_t> hm;
        for (auto* v_ : {&slot, &q0, &qn, &off}) hm.insert(hm.end(), v_->begin(), v_->end());
        hm.insert(hm.end(), row_pos.begin(), row_pos.end());
        upload_i32(c, dm, hm.data(), hm.size());
        Seqs seqs{dm, dm + n_seq, dm + 2 * n_seq, dm + 3 * n_seq};
        AttnPlan plan;
        stream_attention_plan(c, strategy, q, M, n_seq, slot, qn, off, H, DHb, kv_stride, work, plan);
        float* so = (float*)po.need((size_t)M * H * plan.mc * DHb * 4, c->stream);
        float* sml = (float*)pml.need((size_t)M * H * plan.mc * 2 * 4, c->stream);
        const size_t kv_bytes = (size_t)n_seq * H * kv_stride * DHb * 2;
        auto call = [&](int i) {
            const char* kc = (const char*)k + (size_t)(i % n_kv) * kv_bytes;
            const char* vc = (const char*)v + (size_t)(i % n_kv) * kv_bytes;
            stream_attention_run(c, plan, kc, vc, seqs, so, sml, out);
            if (plan.needs_combine) {
                if (DHb == 64)
                    BASS_CUDA(launch_pdl(attn_combine_kernel<__nv_bfloat16, 64>, dim3(M, H), dim3(64), 0, c->stream,
                                         (const float*)so, (const float*)sml, (const int32_t*)(dm + 4 * n_seq), H,
                                         plan.mc, stream_split_len(), (__nv_bfloat16*)out, 1));
                else
                    BASS_CUDA(launch_pdl(attn_combine_kernel<__nv_bfloat16, 128>, dim3(M, H), dim3(128), 0, c->stream,
                                         (const float*)so, (const float*)sml, (const int32_t*)(dm + 4 * n_seq), H,
                                         plan.mc, stream_split_len(), (__nv_bfloat16*)out, 1));
                check_launch(c);
            }
        };
        for (int i = 0; i < n_kv; ++i) call(i);   // warm (tensor maps, first-launch costs)
        cudaEvent_t a, b;
        BASS_CUDA(cudaEventCreate(&a));
        BASS_CUDA(cudaEventCreate(&b));
        BASS_CUDA(cudaEventRecord(a, c->stream));
        for (int i = 0; i < reps; ++i) call(i);
        BASS_CUDA(cudaEventRecord(b, c->stream));
        c->sync();
        float ms = 0.f;
        BASS_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_per_call = ms / reps;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
#ifdef BASS_ATTN_PROBE
        {   // one more call with the pipeline stamps on (debug build)
            unsigned long long* dp;
            BASS_CUDA(cudaMalloc(&dp, 16 * 32 * 8));
            BASS_CUDA(cudaMemset(dp, 0, 16 * 32 * 8));
            ast::attn_probe_set(dp);
            call(0);
            c->sync();
            ast::attn_probe_set(nullptr);
            std::vector<unsigned long long> hp(16 * 32);
            BASS_CUDA(cudaMemcpy(hp.data(), dp, hp.size() * 8, cudaMemcpyDeviceToHost));
            cudaFree(dp);
            for (int b2 = 0; b2 < 16; ++b2) {
                fprintf(stderr, "probe cta %2d:", b2);
                for (int i = 1; i < 27; ++i)
                    fprintf(stderr, " %6.0f", hp[b2 * 32 + i] ? (double)(hp[b2 * 32 + i] - hp[b2 * 32]) / 1.965 : -1.0);
                fprintf(stderr, "\n");
            }
        }
#endif
    });
}

int bass_rng_uniforms(bass_ctx* c, int n, uint64_t seed, const int64_t* sid, const int32_t* role, const int64_t* ctr,
                      double* out) {
    return guarded(c, [&] {
        if (n <= 0) return;
        int64_t *ds, *dc;
        int32_t* dr;
        double* dout;
        BASS_CUDA(cudaMallocAsync((void**)&ds, n * 8, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&dc, n * 8, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&dr, n * 4, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&dout, n * 16, c->stream));
        BASS_CUDA(cudaMemcpyAsync(ds, sid, n * 8, cudaMemcpyHostToDevice, c->stream));
        BASS_CUDA(cudaMemcpyAsync(dc, ctr, n * 8, cudaMemcpyHostToDevice, c->stream));
        BASS_CUDA(cudaMemcpyAsync(dr, role, n * 4, cudaMemcpyHostToDevice, c->stream));
        rng_kernel<<<(n + 127) / 128, 128, 0, c->stream>>>(n, seed, ds, dr, dc, dout);
        check_launch(c);
        BASS_CUDA(cudaMemcpyAsync(out, dout, n * 16, cudaMemcpyDeviceToHost, c->stream));
        for (void* p : {(void*)ds, (void*)dc, (void*)dr, (void*)dout}) BASS_CUDA(cudaFreeAsync(p, c->stream));
        c->sync();
    });
}

int bass_shape_sample(bass_ctx* c, int n, int V, const float* logits, double T, double top_p, const double* u,
                      int32_t* tok_out, double* probs_out) {
    return guarded(c, [&] {
        BASS_REQUIRE(top_p > 0.0 && top_p <= 1.0, "top_p must be in (0, 1]");
        BASS_REQUIRE(T >= 0.0, "temperature must be >= 0");
        if (n <= 0) return;
        for (int i = 0; i < n; ++i) {
            bool finite = false;
            for (int k = 0; k < V && !finite; ++k) finite = std::isfinite(logits[(int64_t)i * V + k]);
            BASS_REQUIRE(finite, "all logits are -inf; distribution undefined");
        }
        float* dl;
        double *du, *scr, *dp = nullptr;
        int32_t* dt;
        BASS_CUDA(cudaMallocAsync((void**)&dl, (size_t)n * V * 4, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&du, (size_t)n * 8, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&scr, (size_t)n * V * 8, c->stream));
        BASS_CUDA(cudaMallocAsync((void**)&dt, (size_t)n * 4, c->stream));
        if (probs_out) BASS_CUDA(cudaMallocAsync((void**)&dp, (size_t)n * V * 8, c->stream));
        BASS_CUDA(cudaMemcpyAsync(dl, logits, (size_t)n * V * 4, cudaMemcpyHostToDevice, c->stream));
        BASS_CUDA(cudaMemcpyAsync(du, u, (size_t)n * 8, cudaMemcpyHostToDevice, c->stream));
        cl_shape_sample_kernel<<<n * CL_CTAS, CL_THREADS, 0, c->stream>>>(dl, V, T, top_p, du, scr, dt, dp);
        check_launch(c);
        BASS_CUDA(cudaMemcpyAsync(tok_out, dt, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream));
        if (probs_out)
            BASS_CUDA(cudaMemcpyAsync(probs_out, dp, (size_t)n * V * 8, cudaMemcpyDeviceToHost, c->stream));
        for (void* p : {(void*)dl, (void*)du, (void*)scr, (void*)dt}) BASS_CUDA(cudaFreeAsync(p, c->stream));
        if (dp) BASS_CUDA(cudaFreeAsync(dp, c->stream));
        c->sync();
    });
}

int bass_accept(bass_ctx* c, int n, int V, const float* ql, const float* pl, double T, double top_p,
                const int32_t* tok, uint64_t seed, const int64_t* sid, const int64_t* ctr, int32_t* acc_out,
                int32_t* corr_out) {
    return guarded(c, [&] {
        if (n <= 0) return;
        float *dq, *dp;
        double* scr;
        int32_t *dt, *da, *dc;
        int64_t *ds, *dr;
        cudaStream_t st = c->stream;
        BASS_CUDA(cudaMallocAsync((void**)&dq, (size_t)n * V * 4, st));
        BASS_CUDA(cudaMallocAsync((void**)&dp, (size_t)n * V * 4, st));
        BASS_CUDA(cudaMallocAsync((void**)&scr, (size_t)n * V * 16, st));
        BASS_CUDA(cudaMallocAsync((void**)&dt, (size_t)n * 4, st));
        BASS_CUDA(cudaMallocAsync((void**)&da, (size_t)n * 4, st));
        BASS_CUDA(cudaMallocAsync((void**)&dc, (size_t)n * 4, st));
        BASS_CUDA(cudaMallocAsync((void**)&ds, (size_t)n * 8, st));
        BASS_CUDA(cudaMallocAsync((void**)&dr, (size_t)n * 8, st));
        BASS_CUDA(cudaMemcpyAsync(dq, ql, (size_t)n * V * 4, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(dp, pl, (size_t)n * V * 4, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(dt, tok, (size_t)n * 4, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(ds, sid, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        BASS_CUDA(cudaMemcpyAsync(dr, ctr, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        cl_accept_pairs_kernel<<<n * CL_CTAS, CL_THREADS, 0, st>>>(dq, dp, V, T, top_p, dt, seed, ds, dr, scr, da, dc);
        check_launch(c);
        BASS_CUDA(cudaMemcpyAsync(acc_out, da, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        BASS_CUDA(cudaMemcpyAsync(corr_out, dc, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        for (void* p : {(void*)dq, (void*)dp, (void*)scr, (void*)dt, (void*)da, (void*)dc, (void*)ds, (void*)dr})
            BASS_CUDA(cudaFreeAsync(p, st));
        c->sync();
        for (int i = 0; i < n; ++i)
            BASS_REQUIRE(corr_out[i] != -2, "draft token " + std::to_string(tok[i]) + " has zero draft probability");
    });
}

}  // extern "C"
