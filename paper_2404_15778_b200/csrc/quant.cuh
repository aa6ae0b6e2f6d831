// INT8 W8A8 numerics of the reference's quantized inference path
// (ref:quant.py:55-129, model.py:135-143, 160-164, 219-222):
//   - weights: one scale per output channel, scale = max|w| / 127 (1 for an
//     all-zero channel), payload = clip(round_half_away(w / scale), +-127);
//   - activations entering every linear layer: one scale per token row;
//   - q / k / v: fake-quantized per (token, head) in the QKV GEMM epilogue
//     (gemm_tc.cu) — the attention sees the dequantized values (stored bf16,
//     like the bf16 path's cache);
//   - the GEMM accumulates int8 x int8 exactly (tcgen05 kind::i8, s32 in
//     TMEM) and dequantizes in its epilogue: out = acc * s_token * s_channel.
// Scales are fp64 like the reference's; the row kernels below compute the
// values they quantize in fp32.
#pragma once

#include "model_kernels.cuh"

namespace bass {

constexpr int QMAX = 127;   // ref:quant.py:19

// Packed int8 weight layout: 128 x 128 tiles (16 KB, the same bytes per tile
// as the bf16 128 x 64 tiles), tile (nt, kb) at nt * K/128 + kb, each the
// shared-memory image of a K-major 128-byte-swizzled kind::i8 UMMA operand.
BASS_DEV int64_t packed_index_i8(int64_t n, int64_t k, int64_t K) {
    const int64_t tile = (n >> 7) * (K >> 7) + (k >> 7);
    const int r = (int)(n & 127), c = (int)((k & 127) >> 4);
    return tile * 16384 + r * 128 + ((c ^ (r & 7)) << 4) + (k & 15);
}

// sign(x) * floor(|x| + 0.5), clipped to [-127, 127] (ref:quant.py:44-52)
BASS_DEV int8_t quant_round(double x) {
    double r = floor(fabs(x) + 0.5);
    r = r > (double)QMAX ? (double)QMAX : r;
    return (int8_t)(x < 0.0 ? -r : r);
}
BASS_DEV double group_scale(float amax) { return amax > 0.f ? (double)amax / (double)QMAX : 1.0; }

BASS_DEV double block_max_d(double v, double* scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        double r = lane < nw ? scratch[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
        if (lane == 0) scratch[0] = r;
    }
    __syncthreads();
    const double r = scratch[0];
    __syncthreads();
    return r;
}

// Weight channel quantization (ref:quant.py:55-63): row n of the output-major
// fp32 matrix src [N, K] -> packed int8 rows row_off + n of dst (row length
// K), scale -> scale[row_off + n].  One CTA per output channel; fp64 scale and
// division, so the payload equals the reference's bit for bit.
static __global__ void quant_weight_rows_kernel(const float* __restrict__ src, int K, int8_t* __restrict__ dst,
                                         int64_t row_off, double* __restrict__ scale) {
    __shared__ double red[32];
    const int n = blockIdx.x;
    const float* row = src + (int64_t)n * K;
    double amax = 0.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) amax = fmax(amax, fabs((double)row[k]));
    amax = block_max_d(amax, red);
    const double s = amax > 0.0 ? amax / (double)QMAX : 1.0;
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        dst[packed_index_i8(row_off + n, k, K)] = quant_round((double)row[k] / s);
    if (threadIdx.x == 0) scale[row_off + n] = s;
}

// dequantized packed int8 rows -> reference [K, N] fp32 (get_weight) or the
// raw payload in the reference layout (get_qweight)
static __global__ void dequant_gather_kernel(const int8_t* __restrict__ w, const double* __restrict__ scale, int K, int N,
                                      int64_t row_off, float* __restrict__ out_f, int8_t* __restrict__ out_q) {
    const int64_t total = (int64_t)K * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / N, n = i - k * N;
        const int8_t q = w[packed_index_i8(row_off + n, k, K)];
        if (out_f) out_f[i] = (float)((double)q * scale[row_off + n]);
        if (out_q) out_q[i] = q;
    }
}

// reference-layout int8 payload [K, N] (input-major, ref:quant.py:55-63) ->
// packed output-major tiles (rows beyond N stay as the caller zeroed them)
static __global__ void pack_i8_ref_kernel(const int8_t* __restrict__ src, int K, int N, int8_t* __restrict__ dst) {
    const int64_t total = (int64_t)K * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / N, n = i - k * N;
        dst[packed_index_i8(n, k, K)] = src[i];
    }
}

// Per-token activation quantization fused with the LayerNorm that produces
// it (ref:model.py:214-222 _layer_norm -> _linear -> quantize per token):
// LN(x[src]) in fp32 (two passes over the register-resident row), then
// scale = max|h| / 127 and the int8 payload.  `gather` (optional) selects the
// source rows (final LayerNorm of the logit rows).  It also clears the row's
// amax accumulators of the QKV (n_groups per row) and FC epilogues: every
// projection that fills them follows a LayerNorm.
static __global__ void __launch_bounds__(LN_THREADS) ln_quant_kernel(const float* __restrict__ x,
                                                              const int32_t* __restrict__ gather,
                                                              const float* __restrict__ g,
                                                              const float* __restrict__ b, int d,
                                                              int8_t* __restrict__ out, double* __restrict__ scale,
                                                              float* __restrict__ amax_g, int n_groups,
                                                              float* __restrict__ amax_r, TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    __shared__ float red[33];
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    for (int t = threadIdx.x; t < n_groups; t += blockDim.x) amax_g[(int64_t)r * n_groups + t] = 0.f;
    if (threadIdx.x == 0 && amax_r) amax_r[r] = 0.f;
    const int src = gather ? gather[r] : r;
    const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)src * d);
    const int n4 = d >> 2;
    float4 v[LN_NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) {
        const int c = threadIdx.x + i * LN_THREADS;
        v[i] = c < n4 ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mean = block_sum(s, red) / float(d);
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) {
        const int c = threadIdx.x + i * LN_THREADS;
        if (c < n4) {
            const float a = v[i].x - mean, bb = v[i].y - mean, cc = v[i].z - mean, dd = v[i].w - mean;
            q += (a * a + bb * bb) + (cc * cc + dd * dd);
        }
    }
    const float var = block_sum(q, red) / float(d);
    const float rstd = 1.0f / sqrtf(var + kLnEps);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) {
        const int c = threadIdx.x + i * LN_THREADS;
        if (c < n4) {
            const float4 gg = g4[c], bv = b4[c];
            v[i].x = (v[i].x - mean) * rstd * gg.x + bv.x;
            v[i].y = (v[i].y - mean) * rstd * gg.y + bv.y;
            v[i].z = (v[i].z - mean) * rstd * gg.z + bv.z;
            v[i].w = (v[i].w - mean) * rstd * gg.w + bv.w;
            amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)), fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
        }
    }
    amax = block_max(amax, red);
    const double sc = group_scale(amax);
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) {
        const int c = threadIdx.x + i * LN_THREADS;
        if (c < n4) {
            char4 o;
            o.x = quant_round((double)v[i].x / sc);
            o.y = quant_round((double)v[i].y / sc);
            o.z = quant_round((double)v[i].z / sc);
            o.w = quant_round((double)v[i].w / sc);
            reinterpret_cast<char4*>(out + (int64_t)r * d)[c] = o;
        }
    }
    if (threadIdx.x == 0) scale[r] = sc;
    trace_end(tr, t_start);
}

// Per-token quantization of the attention context (bf16 [M, d]) before Wo.
// Grid (rows, chunks of QR_CHUNK columns): every CTA reduces the whole row's
// max |value| (one L2-resident read of d bf16) and quantizes its own chunk.
constexpr int QR_CHUNK = 1024;
static __global__ void __launch_bounds__(256) quant_ctx_kernel(const __nv_bfloat16* __restrict__ in, int d,
                                                        int8_t* __restrict__ out, double* __restrict__ scale,
                                                        TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    __shared__ float red[33];
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    const uint4* row = reinterpret_cast<const uint4*>(in + (int64_t)r * d);   // d % 8 == 0
    float amax = 0.f;
    for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
        const uint4 u = row[c];
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int k = 0; k < 8; ++k) amax = fmaxf(amax, fabsf(__bfloat162float(h[k])));
    }
    amax = block_max(amax, red);
    const double sc = group_scale(amax);
    const int c0 = blockIdx.y * QR_CHUNK, c1 = min(d, c0 + QR_CHUNK);
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x)
        out[(int64_t)r * d + c] = quant_round((double)__bfloat162float(in[(int64_t)r * d + c]) / sc);
    if (threadIdx.x == 0 && blockIdx.y == 0) scale[r] = sc;
    trace_end(tr, t_start);
}

// Per-token quantization of the GELU output (fp32 [M, n], GELU and the row's
// max |value| already applied / accumulated by the FC GEMM epilogue) before
// Wproj.  Grid (rows, chunks of QR_CHUNK columns).
static __global__ void __launch_bounds__(256) quant_amax_rows_kernel(const float* __restrict__ in, int n,
                                                              const float* __restrict__ amax_r,
                                                              int8_t* __restrict__ out, double* __restrict__ scale,
                                                              TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    const double sc = group_scale(amax_r[r]);
    const int c0 = blockIdx.y * QR_CHUNK, c1 = min(n, c0 + QR_CHUNK);
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x)
        out[(int64_t)r * n + c] = quant_round((double)in[(int64_t)r * n + c] / sc);
    if (threadIdx.x == 0 && blockIdx.y == 0) scale[r] = sc;
    trace_end(tr, t_start);
}

}  // namespace bass
