// Ragged decoder forward: embedding, LayerNorm, SIMT GEMM (parity/fp32
// path), ragged attention (PAD / SPLIT / RAGGED work list) and the split-KV
// combine.  Every reduction runs in a fixed order that depends only on the
// row's own data and absolute key positions, never on which other rows share
// the launch: a row's result is bitwise independent of batch composition and
// block length (the reference's purity contract, ref:model.py:267-271).
#pragma once
#include <type_traits>

#include "common.cuh"

namespace bass {

constexpr float kLnEps = 1e-5f;   // ref:model.py:31

// ---------------------------------------------------------------- metadata
struct Rows {                    // one entry per new token row (length M)
    const int32_t* tok;          // >= 0: token id; < 0: proposals[slot][-tok-1]
    const int32_t* slot;
    const int32_t* pos;          // absolute position = cache offset + t
};
struct Seqs {                    // one entry per sequence in the block
    const int32_t* slot;
    const int32_t* q0;           // first row of this sequence
    const int32_t* qn;           // rows in this sequence
    const int32_t* off;          // committed cache length before the block
};

// ------------------------------------------------------------- embedding
// x[r] = tok_emb[id] + pos_emb[pos]   (ref:model.py:203-209)
// `stats` (optional, bf16 folded-LayerNorm path): the row's exact mean K ->
// shift[r] (the row-mean array `kmean` of forward()), {sum (x - K), sum (x - K)^2} -> stats[r] (one 'tile' covering the
// whole row, fixed-order sums) and X = bf16((x - K) * xg) -> xb for the
// layer-0 QKV GEMM (see forward(): centring keeps a large row mean from
// swallowing the deviations).
template <typename TW>
__global__ void embed_kernel(const TW* __restrict__ tok_emb, const TW* __restrict__ pos_emb,
                             Rows rows, const int32_t* __restrict__ proposals, int pstride,
                             int d, float* __restrict__ x, float* __restrict__ stats,
                             float* __restrict__ shift, __nv_bfloat16* __restrict__ xb,
                             const float* __restrict__ xg) {
    __shared__ float red[2][33];
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    int id = rows.tok[r];
    if (id < 0) id = proposals[rows.slot[r] * pstride + (-id - 1)];
    const int p = rows.pos[r];
    float s1 = 0.f, s2 = 0.f;
    if constexpr (std::is_same<TW, __nv_bfloat16>::value) {
        constexpr int NV = 4;   // d <= 8 * NV * blockDim: the row stays in registers
        if ((d & 7) == 0 && (d >> 3) <= NV * (int)blockDim.x) {
            const int n8 = d >> 3;
            uint4 te[NV], pe[NV];   // every load of the row issued before the first use
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int c8 = threadIdx.x + u * blockDim.x;
                if (c8 < n8) {
                    te[u] = __ldg(reinterpret_cast<const uint4*>(tok_emb + (int64_t)id * d) + c8);
                    pe[u] = __ldg(reinterpret_cast<const uint4*>(pos_emb + (int64_t)p * d) + c8);
                }
            }
            float v[NV][8];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int c8 = threadIdx.x + u * blockDim.x;
                if (c8 >= n8) continue;
                const __nv_bfloat16* tb = reinterpret_cast<const __nv_bfloat16*>(&te[u]);
                const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pe[u]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    v[u][k] = __bfloat162float(tb[k]) + __bfloat162float(pb[k]);
                    s1 += v[u][k];
                }
                float4* xo = reinterpret_cast<float4*>(x + (int64_t)r * d) + 2 * c8;
                xo[0] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
                xo[1] = make_float4(v[u][4], v[u][5], v[u][6], v[u][7]);
            }
            if (!stats) return;
            const float K = block_sum(s1, red[0]) / (float)d;
            s1 = 0.f;
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int c8 = threadIdx.x + u * blockDim.x;
                if (c8 >= n8) continue;
                const float4 g0 = __ldg(reinterpret_cast<const float4*>(xg) + 2 * c8);
                const float4 g1 = __ldg(reinterpret_cast<const float4*>(xg) + 2 * c8 + 1);
                const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                uint4 ob;
                __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&ob);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float c = v[u][k] - K;
                    s1 += c;
                    s2 += c * c;
                    o[k] = __float2bfloat16_rn(c * gg[k]);
                }
                reinterpret_cast<uint4*>(xb + (int64_t)r * d)[c8] = ob;
            }
            const float a = block_sum(s1, red[0]), b = block_sum(s2, red[1]);
            if (threadIdx.x == 0) {
                reinterpret_cast<float2*>(stats)[r] = make_float2(a, b);
                shift[r] = K;
            }
            return;
        }
    }
    // generic rows (fp32 tables, or rows too long for the register path)
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float v = ld(tok_emb, (int64_t)id * d + c) + ld(pos_emb, (int64_t)p * d + c);
        x[(int64_t)r * d + c] = v;
        s1 += v;
    }
    if (!stats) return;
    const float K = block_sum(s1, red[0]) / (float)d;
    s1 = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {   // this thread's own writes: no barrier needed
        const float cv = x[(int64_t)r * d + c] - K;
        xb[(int64_t)r * d + c] = __float2bfloat16_rn(cv * xg[c]);
        s1 += cv;
        s2 += cv * cv;
    }
    const float a = block_sum(s1, red[0]), b = block_sum(s2, red[1]);
    if (threadIdx.x == 0) {
        reinterpret_cast<float2*>(stats)[r] = make_float2(a, b);
        shift[r] = K;
    }
}

// ------------------------------------------------------------- layernorm
// (x - mean) / sqrt(var + eps) * g + b, population variance, two passes
// (ref:model.py:150-153).  Optional row gather (final LN of selected rows).
// Single pass over HBM: the row is held in registers (NV float4 per thread,
// all loads issued before the first reduction), so the kernel is bound by one
// read of x and one write of the normalised row rather than by load latency.
constexpr int LN_THREADS = 256, LN_NV = 8;   // d <= 8192 with 16-byte rows

template <typename TA>
__global__ void __launch_bounds__(LN_THREADS) layernorm_kernel(const float* __restrict__ x,
                                                               const int32_t* __restrict__ gather,
                                                               const float* __restrict__ g,
                                                               const float* __restrict__ b, int d,
                                                               TA* __restrict__ out, TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    __shared__ float red[33];
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
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
#pragma unroll
    for (int i = 0; i < LN_NV; ++i) {
        const int c = threadIdx.x + i * LN_THREADS;
        if (c < n4) {
            const float4 gg = g4[c], bv = b4[c];
            const int64_t o = (int64_t)r * d + 4 * c;
            st(out, o + 0, (v[i].x - mean) * rstd * gg.x + bv.x);
            st(out, o + 1, (v[i].y - mean) * rstd * gg.y + bv.y);
            st(out, o + 2, (v[i].z - mean) * rstd * gg.z + bv.z);
            st(out, o + 3, (v[i].w - mean) * rstd * gg.w + bv.w);
        }
    }
    trace_end(tr, t_start);
}

// ------------------------------------------------------------- epilogues
enum EpiMode { EPI_QKV = 0, EPI_RESID = 1, EPI_GELU = 2, EPI_STORE = 3 };

struct Epi {
    float* x;            // EPI_RESID: x[m, n] += acc (fp32 residual stream)
    float* stats;        // EPI_RESID (tcgen05 path, optional): per (128-column tile, row) {sum c, sum c^2},
                         //   c = x_new - K with the row shift K = shift[row] (the mean of x before the add)
    const float* shift;
    __nv_bfloat16* xb;   //   ... with it: bf16(c * xg) = X of the next GEMM (its LayerNorm folded)
    const float* xg;     //   the next LayerNorm's gain
    void* out;           // EPI_QKV: q [M, d] (act); EPI_GELU: [M, N] (act); EPI_STORE: [M, N] fp32
    void* kc;            // EPI_QKV: this layer's K cache [slot][H][cap][dh] (act dtype)
    void* vc;
    const int32_t* row_slot;
    const int32_t* row_pos;
    int d, dh, H, cap;
    float* amax;         // W8A8 QKV / GELU epilogues: running max |value| per (row, head) / per row (uint-ordered atomics)
};

BASS_DEV float gelu_erf(float v) {   // ref:model.py:156-157 (exact erf form)
    return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
}

template <int MODE, typename TA>
BASS_DEV void epilogue(const Epi& e, int m, int n, int N, float acc) {
    if constexpr (MODE == EPI_QKV) {
        const int part = n / e.d, nn = n - part * e.d;
        if (part == 0) {
            st(reinterpret_cast<TA*>(e.out), (int64_t)m * e.d + nn, acc);
        } else {
            const int h = nn / e.dh, c = nn - h * e.dh;
            TA* base = reinterpret_cast<TA*>(part == 1 ? e.kc : e.vc);
            const int64_t idx = (((int64_t)e.row_slot[m] * e.H + h) * e.cap + e.row_pos[m]) * e.dh + c;
            st(base, idx, acc);     // KV append (ref:kv_cache.py:63-84)
        }
    } else if constexpr (MODE == EPI_RESID) {
        e.x[(int64_t)m * N + n] += acc;
    } else if constexpr (MODE == EPI_GELU) {
        st(reinterpret_cast<TA*>(e.out), (int64_t)m * N + n, gelu_erf(acc));
    } else {
        reinterpret_cast<float*>(e.out)[(int64_t)m * N + n] = acc;
    }
}

// ----------------------------------------------------------- SIMT GEMM
// Y[m, n] = sum_k X[m, k] * W[n, k]  (W stored output-major [N, K]).
// Each output is one thread's sequential FMA chain over k = 0..K-1, so it
// does not depend on M or on the other rows.  Used for the fp32 parity mode
// (true FFMA, no TF32) and as the reference kernel for the tcgen05 GEMM.
constexpr int SG_BN = 64, SG_BM = 16, SG_BK = 32;

template <int MODE, typename TA, typename TW>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const TA* __restrict__ X,
                                                         const TW* __restrict__ W, int M, int N,
                                                         int K, Epi e, bool packed) {
    __shared__ float Ws[SG_BK][SG_BN + 1];
    __shared__ float Xs[SG_BM][SG_BK + 1];
    const int t = threadIdx.x;
    const int n0 = blockIdx.x * SG_BN, m0 = blockIdx.y * SG_BM;
    const int f = t & 63, tg = t >> 6;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k0 = 0; k0 < K; k0 += SG_BK) {
#pragma unroll
        for (int j = 0; j < (SG_BN * SG_BK) / 256; ++j) {
            const int i = t + 256 * j, nn = i / SG_BK, kk = i % SG_BK;
            const int gn = n0 + nn, gk = k0 + kk;
            Ws[kk][nn] = (gn < N && gk < K) ? ld(W, packed ? packed_index(gn, gk, K) : (int64_t)gn * K + gk) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < (SG_BM * SG_BK) / 256; ++j) {
            const int i = t + 256 * j, mm = i / SG_BK, kk = i % SG_BK;
            const int gm = m0 + mm, gk = k0 + kk;
            Xs[mm][kk] = (gm < M && gk < K) ? ld(X, (int64_t)gm * K + gk) : 0.f;
        }
        __syncthreads();
        const int kmax = min(SG_BK, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            const float w = Ws[kk][f];
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r] = fmaf(Xs[tg * 4 + r][kk], w, acc[r]);
        }
        __syncthreads();
    }
    const int n = n0 + f;
    if (n >= N) return;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int m = m0 + tg * 4 + r;
        if (m < M) epilogue<MODE, TA>(e, m, n, N, acc[r]);
    }
}

// ------------------------------------------------------ ragged attention
// softmax((q . k) / sqrt(dh), causal s <= off + t) . v per (sequence, head)
// (ref:attention.py:85-137).  Work unit = (q tile of 16 rows, head, KV chunk
// of 256 absolute key positions); inside a chunk, 64-key sub-tiles are folded
// with an online softmax; chunk partials are merged by attn_combine_kernel
// in chunk order.  Chunk / sub-tile boundaries are absolute key positions,
// so a row's arithmetic is identical for PAD, SPLIT and RAGGED launches and
// for any q_len (prefill, verify, single-token decode).
constexpr int AT_QT = 16, AT_CHUNK = 256, AT_SUB = 64, AT_THREADS = 128;

struct AttnWork {                 // one q tile of one sequence
    int32_t seq, t0;
};

template <typename TA, int DH>
__global__ void __launch_bounds__(AT_THREADS) attn_partial_kernel(
    const TA* __restrict__ q, const TA* __restrict__ kc, const TA* __restrict__ vc, Seqs seqs,
    const AttnWork* __restrict__ work, int H, int cap, int pad_kv_len,
    float* __restrict__ part_o, float* __restrict__ part_ml, int max_chunks) {
    constexpr int EPL = (DH + 31) / 32;               // head dims per lane (guarded)
    extern __shared__ float smem[];
    float* Kt = smem;                                  // [DH][AT_SUB + 1]
    float* Vs = Kt + DH * (AT_SUB + 1);                // [AT_SUB][DH]
    float* Qs = Vs + AT_SUB * DH;                      // [AT_QT][DH]

    pdl_trigger();
    pdl_wait();
    const AttnWork wk = work[blockIdx.z];
    const int h = blockIdx.y, c = blockIdx.x;
    const int slot = seqs.slot[wk.seq], qn = seqs.qn[wk.seq], off = seqs.off[wk.seq];
    const int q0row = seqs.q0[wk.seq];
    const int L = off + qn;                           // keys visible to the last row
    const int kv_len = pad_kv_len > 0 ? pad_kv_len : L;   // PAD: padded key range
    const int c_begin = c * AT_CHUNK;
    if (c_begin >= kv_len) return;
    const int t_last = min(qn, wk.t0 + AT_QT) - 1;
    if (wk.t0 >= qn || off + t_last < c_begin) return;   // no row of the tile sees this chunk

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float scale = sqrtf(float(DH));

    for (int i = threadIdx.x; i < AT_QT * DH; i += AT_THREADS) {
        const int rr = i / DH, cc = i % DH, t = wk.t0 + rr;
        Qs[i] = t < qn ? ld(q, ((int64_t)(q0row + t) * H + h) * DH + cc) : 0.f;
    }
    // each warp owns 4 rows of the tile
    float m_run[4], l_run[4], o[4][EPL];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        m_run[r] = -INFINITY;
        l_run[r] = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) o[r][e] = 0.f;
    }
    const int64_t kvbase = ((int64_t)slot * H + h) * cap;
    const int c_end = min(c_begin + AT_CHUNK, kv_len);
    for (int s0 = c_begin; s0 < c_end; s0 += AT_SUB) {
        __syncthreads();
        for (int i = threadIdx.x; i < AT_SUB * DH; i += AT_THREADS) {
            const int j = i / DH, cc = i % DH, s = s0 + j;
            // keys past the sequence's own history are PAD's zero padding
            // (ref:attention.py:116-121): never read, so stale cache rows
            // (possibly NaN bit patterns) cannot leak through 0 * V.
            float kv = 0.f, vv = 0.f;
            if (s < c_end && s < L) {
                kv = ld(kc, (kvbase + s) * DH + cc);
                vv = ld(vc, (kvbase + s) * DH + cc);
            }
            Kt[cc * (AT_SUB + 1) + j] = kv;
            Vs[j * DH + cc] = vv;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int rr = warp * 4 + r, t = wk.t0 + rr;
            if (t >= qn) continue;
            const int lim = off + t;                      // last visible key
            if (lim < s0) continue;
            float sc[2];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = lane + 32 * jj;
                float a = 0.f;
#pragma unroll 8
                for (int cc = 0; cc < DH; ++cc) a = fmaf(Qs[rr * DH + cc], Kt[cc * (AT_SUB + 1) + j], a);
                const int s = s0 + j;
                sc[jj] = (s <= lim && s < c_end && s < L) ? a / scale : -INFINITY;
            }
            const float mx = warp_max(fmaxf(sc[0], sc[1]));
            const float m_new = fmaxf(m_run[r], mx);
            if (m_new == -INFINITY) continue;
            const float alpha = __expf(m_run[r] - m_new);
            float p[2];
            p[0] = sc[0] == -INFINITY ? 0.f : expf(sc[0] - m_new);
            p[1] = sc[1] == -INFINITY ? 0.f : expf(sc[1] - m_new);
            l_run[r] = l_run[r] * alpha + warp_sum(p[0] + p[1]);
#pragma unroll
            for (int e = 0; e < EPL; ++e) o[r][e] *= alpha;
            for (int j = 0; j < AT_SUB; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p[j >> 5], j & 31);
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (lane + 32 * e < DH) o[r][e] = fmaf(pj, Vs[j * DH + lane + 32 * e], o[r][e]);
            }
            m_run[r] = m_new;
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int t = wk.t0 + warp * 4 + r;
        if (t >= qn || off + t < c_begin) continue;
        const int64_t slotidx = ((int64_t)(q0row + t) * H + h) * max_chunks + c;
#pragma unroll
        for (int e = 0; e < EPL; ++e)
            if (lane + 32 * e < DH) part_o[slotidx * DH + lane + 32 * e] = o[r][e];
        if (lane == 0) {
            part_ml[slotidx * 2] = m_run[r];
            part_ml[slotidx * 2 + 1] = l_run[r];
        }
    }
}

// merge chunk partials of one (row, head) in chunk order; writes ctx [M, H*dh]
template <typename TA, int DH>
__global__ void attn_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                    const int32_t* __restrict__ row_pos, int H, int max_chunks,
                                    int chunk, TA* __restrict__ out, int skip_single = 0) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x, h = blockIdx.y;
    const int nc = row_pos[r] / chunk + 1;
    if (skip_single && nc == 1) return;   // already written normalised by the attention kernel
    const int64_t base = ((int64_t)r * H + h) * max_chunks;
    float mx = -INFINITY;
    for (int c = 0; c < nc; ++c) mx = fmaxf(mx, part_ml[(base + c) * 2]);
    for (int e = threadIdx.x; e < DH; e += blockDim.x) {
        float num = 0.f, den = 0.f;
        for (int c = 0; c < nc; ++c) {
            const float m = part_ml[(base + c) * 2];
            if (m == -INFINITY) continue;
            const float w = expf(m - mx);
            num = fmaf(w, part_o[(base + c) * DH + e], num);
            den = fmaf(w, part_ml[(base + c) * 2 + 1], den);
        }
        st(out, ((int64_t)r * H + h) * DH + e, num / den);
    }
}

}  // namespace bass
