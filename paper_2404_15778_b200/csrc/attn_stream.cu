// Persistent warp-specialised flash-decoding attention on tcgen05 (sm_100a),
// d_head = 128 or 64 — the ragged verify / draft / prefill attention of BASS
// (PAD and SPLIT, ref:attention.py:85-154).  d_head = 64 (the OPT-125M-shape
// draft of C3) keeps the same 128-lane orientation: S^T = K . Q^T is one
// 64-wide K block instead of two, and O^T = V^T . P^T runs as an M = 128 MMA
// whose upper 64 rows (the K block stored after V) are never read back.
//
// Work item = (sequence, query tile of NQ rows, head, 1024-key split).  The
// grid is persistent (<= one CTA per SM); CTA b walks items b, b + grid, ...
// and streams every 128-key chunk of each through a TMA ring, so loads of
// the next item overlap the softmax / epilogue of the current one.
//
// Orientation: S^T = K . Q^T (UMMA M = 128 keys on TMEM lanes, N = NQ query
// columns); O^T = V^T . P^T (M = 128 head dims, N = NQ).  Warp roles (192
// threads):
//   warp 0      TMA producer (Q tile per item, K and V chunks into the ring)
//   warp 1      MMA issuer (S^T one chunk ahead of the softmax, then O^T += V^T P^T)
//   warps 2-5   softmax / epilogue; thread = key (softmax) = head dim (O).
// Online softmax with a lazily refreshed per-column reference max: a chunk
// whose scores stay within 2^TH of the reference reuses it (no rescale of O,
// no cross-warp max) — decided by one block vote per chunk.  Every rule is
// column-local and chunk / split boundaries are absolute key positions, so a
// row's bits depend only on its own keys: PAD, SPLIT and RAGGED launches,
// prefill, verify and single-token decode agree bitwise (the property behind
// greedy speculative == regular decoding).
// Rows whose history fits one split are written normalised; longer rows leave
// (m, l, o) per split for attn_combine_kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <utility>

#include "runtime.h"

namespace bass {
namespace ast {

constexpr int CH = 128, SPLIT_CH = 8, SPLIT = CH * SPLIT_CH;
constexpr float TH = 8.f;   // reuse the reference max while scores stay below it + TH (log2 units)

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
// K/V history: read once per forward -> L2 evict-first (keeps activations / code resident)
__device__ __forceinline__ void tma_2d_ef(const CUtensorMap* map, uint32_t dst, uint32_t bar, int c0, int c1,
                                          uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4}], [%2], %5;" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}
// shared-memory matrix descriptor, 128-byte swizzle, version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, bf16 x bf16 -> f32, M = 128, N = n, B K-major; a_mn: A is MN-major
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
// 16 consecutive fp32 columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void ld16_nowait(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld8_nowait(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// CQ (8 / 16 / 32 / 64) consecutive columns
// (16-column chunks at or past `ncol` valid columns are not loaded)
template <int CQ>
__device__ __forceinline__ void ldq_nowait(uint32_t taddr, float* v, int ncol) {
    if constexpr (CQ == 8) ld8_nowait(taddr, v);
    else {
#pragma unroll
        for (int j0 = 0; j0 < CQ; j0 += 16)
            if (j0 < ncol) ld16_nowait(taddr + j0, v + j0);
    }
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
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
}
__device__ __forceinline__ void st8(uint32_t taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
}
__device__ __forceinline__ void st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// named barrier 1 + grp over the four warps of one softmax group
__device__ __forceinline__ void sm_bar(int grp) { asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory"); }
__device__ __forceinline__ bool sm_vote_any(bool p, int grp) {
    uint32_t r;
    asm volatile(
        "{\n .reg .pred a, b;\n setp.ne.u32 a, %1, 0;\n bar.red.or.pred b, %2, 128, a;\n selp.u32 %0, 1, 0, b;\n}"
        : "=r"(r)
        : "r"((uint32_t)p), "r"(1 + grp)
        : "memory");
    return r != 0;
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Column reduction over the 128 softmax threads (fixed order => deterministic).
// v[NQ] per thread -> fin[NQ] in shared memory (every thread then reads it).
// Intra-warp: transpose-reduce (lane L ends holding columns L*NQ/32 + i);
// then the four warps' partials are combined in warp order by NQ threads.
template <int NQ, bool MAX>
__device__ __forceinline__ void col_reduce(float (&v)[NQ], float* red, float* fin, int wq, int lane, int tid,
                                           int grp) {
    float w[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) w[i] = v[i];
    int n = NQ;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
        if (n >= 2) {
            const int half = n >> 1;
#pragma unroll
            for (int i = 0; i < NQ / 2; ++i) {
                if (i < half) {
                    const float send = up ? w[i] : w[i + half];
                    const float keep = up ? w[i + half] : w[i];
                    const float r = __shfl_xor_sync(0xffffffffu, send, o);
                    w[i] = MAX ? fmaxf(keep, r) : keep + r;
                }
            }
            n = half;
        } else {
            const float r = __shfl_xor_sync(0xffffffffu, w[0], o);
            w[0] = MAX ? fmaxf(w[0], r) : w[0] + r;
        }
    }
    constexpr int PER = NQ >= 32 ? NQ / 32 : 1;
    constexpr int REP = NQ >= 32 ? 1 : 32 / NQ;
    if (lane % REP == 0) {
#pragma unroll
        for (int i = 0; i < PER; ++i) red[wq * NQ + (lane * NQ) / 32 + i] = w[i];
    }
    sm_bar(grp);
    if (tid < NQ) {
        const float a = red[tid], b = red[NQ + tid], c = red[2 * NQ + tid], d = red[3 * NQ + tid];
        fin[tid] = MAX ? fmaxf(fmaxf(a, b), fmaxf(c, d)) : (a + b) + (c + d);
    }
    sm_bar(grp);
}

// One work entry per (sequence, query tile, split), expanded over heads in the
// kernel; the sequence's metadata is folded in so an item costs one 32-byte load.
struct alignas(16) Work {
    int32_t slot, q0row, qn, off;   // KV slot, first Q / out row, rows, committed length
    int32_t t0, split, nch, safe;   // nch: 128-key chunks of this split the tile's last row sees;
                                    // safe: K/V rows [0, safe) were complete before this launch's
                                    // chain began (loadable before griddepcontrol.wait)
};

// Items of this CTA: blockIdx.x, + gridDim.x, ...; the next item's entry is
// fetched while the current one is processed (hides the global-load latency).
struct ItemIter {
    const Work* work;
    int n_items, H, it;
    Work nxt;
    __device__ __forceinline__ ItemIter(const Work* w, int n, int h) : work(w), n_items(n), H(h), it(blockIdx.x) {
        if (it < n_items) nxt = work[it / H];
    }
    // false when exhausted; idle items (tile beyond the block / no chunk) are skipped
    __device__ __forceinline__ bool next(Work& wk, int& h) {
        while (it < n_items) {
            wk = nxt;
            h = it % H;
            it += gridDim.x;
            if (it < n_items) nxt = work[it / H];
            if (wk.nch > 0 && wk.t0 < wk.qn) return true;
        }
        return false;
    }
};

#ifdef BASS_ATTN_PROBE
// debug build only: per-CTA clock64() stamps of the pipeline events (CTAs < 16)
__device__ unsigned long long* g_attn_probe;
#define APROBE(i)                                                                           \
    do {                                                                                    \
        if (g_attn_probe && blockIdx.x < 16) g_attn_probe[blockIdx.x * 32 + (i)] = clock64(); \
    } while (0)
#else
#define APROBE(i) \
    do {          \
    } while (0)
#endif

// ST: K/V ring stages.  NQ = 16 has two builds: 2 stages for short
// histories (decode / verify: items of 1-3 chunks, measured faster end to
// end) and 3 for long ones (the launch picks by the longest history);
// NQ = 64 is smem bound at 2.
template <int NQ, int DH = 128, int ST = (NQ == 32 || DH == 64 ? 3 : 2)>
struct Cfg {
    static constexpr int STAGES = ST;
    static constexpr int SUB = DH / 64;           // 64-wide (128-byte swizzle) column blocks of K, V, Q
    static constexpr int KV_TILE = CH * 128;      // 128 rows x 64 bf16 (one 128B-swizzle sub-tile)
    static constexpr int STAGE = 2 * SUB * KV_TILE;   // d_head 128: K0 K1 V0 V1; d_head 64: V0 K0
    // (V0 first for d_head 64, so the PV MMA's second 64-row A block, LBO =
    // KV_TILE past V0, lands on K0 of the same stage — inside the allocation)
    static constexpr int K_OFF = DH == 64 ? KV_TILE : 0;
    static constexpr int V_OFF = DH == 64 ? 0 : SUB * KV_TILE;
    static constexpr int R_TILE = NQ * 128;       // NQ rows x 64 bf16: one sub-tile of Q or P
    static constexpr int OFF_Q = STAGES * STAGE;  // 2 buffers x SUB sub-tiles
    static constexpr int OFF_P = OFF_Q + 2 * SUB * R_TILE;
    static constexpr int P_BUF = CH * NQ * 2;     // P^T [128 keys][NQ] bf16, MN-major (queries contiguous)
    static constexpr int OFF_RED = OFF_P + 2 * P_BUF;    // red[4][NQ], fin, mref, thr, alph [NQ]
    static constexpr int OFF_BAR = OFF_RED + 8 * NQ * 4;
    // q_full[2] q_empty[2] k_full[S] v_full[S] k_empty[S] v_empty[S] s_full[2] s_free[2] p_full[2] p_free[2]
    // o_full[2] o_free[2]
    static constexpr int NBAR = 16 + 4 * STAGES;
    static constexpr int SMEM = OFF_BAR + NBAR * 8 + 16 + 1024;
    static constexpr int TMEM_COLS = 4 * NQ < 32 ? 32 : 4 * NQ;   // S0 S1 O0 O1
};

// softmax / epilogue groups of 4 warps: two (splitting the query columns)
// where the registers allow, one for NQ = 64
__host__ __device__ constexpr int softmax_groups(int nq) { return nq >= 32 ? 4 : 2; }
__host__ __device__ constexpr int attn_threads(int nq) { return 64 + 128 * softmax_groups(nq); }

template <int NQ, int DH, int STG>
__global__ void __launch_bounds__(attn_threads(NQ), STG == 1 ? 2 : 1) attn_stream_kernel(
    const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
    const __grid_constant__ CUtensorMap tv, Seqs seqs, const Work* __restrict__ work, int n_items, int H, int cap,
    float* __restrict__ part_o, float* __restrict__ part_ml, int max_splits, __nv_bfloat16* __restrict__ out,
    TraceArg tr) {
    const unsigned long long t_start = tr.buf ? gtimer() : 0ull;
    using Cf = Cfg<NQ, DH, STG>;
    constexpr int ST = Cf::STAGES, SUB = Cf::SUB;
    constexpr int SG = softmax_groups(NQ), CQ = NQ / SG;
    // K ahead of V, except in the long-history NQ = 16 build, whose softmax
    // never holds up the next S^T (measured: K-ahead costs it 5-8 % at L >= 2K,
    // while NQ = 64 gains 27-37 % and short histories ~5 %), and for d_head 64,
    // whose PV MMA also reads the stage's K block (neutral to slightly slower)
    constexpr bool KA = !(NQ == 16 && ST == 3) && DH != 64;
    constexpr bool K_EARLY = KA;   // K slot released by the S^T MMA
    if (threadIdx.x == 0) APROBE(0);
    extern __shared__ uint8_t smem_raw[];
    pdl_trigger();

    const uint32_t raw = su32(smem_raw);
    const uint32_t base = (raw + 1023) & ~1023u;
    uint8_t* sm = smem_raw + (base - raw);
    float* red = reinterpret_cast<float*>(sm + Cf::OFF_RED);
    float* fin = red + 4 * NQ;
    float* mref = fin + NQ;   // per-column reference max (log2 units), shared
    float* thr = mref + NQ;   // raw-score threshold (mref + TH) / C above which a chunk refreshes it
    float* alph = thr + NQ;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Cf::OFF_BAR);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 2;
    uint64_t* k_full = bars + 4;
    uint64_t* v_full = k_full + ST;
    uint64_t* k_empty = v_full + ST;
    uint64_t* v_empty = k_empty + ST;
    uint64_t* s_full = v_empty + ST;
    uint64_t* s_free = s_full + 2;
    uint64_t* p_full = s_free + 2;
    uint64_t* p_free = p_full + 2;
    uint64_t* o_full = p_free + 2;
    uint64_t* o_free = o_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cf::NBAR);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < Cf::NBAR; ++i) mbar_init(su32(&bars[i]), 1);
        // software arrivals: one per softmax warp
        for (int i = 0; i < 2; ++i) {
            mbar_init(su32(&s_free[i]), 4 * SG);
            mbar_init(su32(&p_full[i]), 4 * SG);
            mbar_init(su32(&o_free[i]), 4 * SG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tk) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tv) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tq) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(Cf::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) APROBE(1);
    // Q and this layer's new K/V rows come from the QKV GEMM and the output
    // buffer is read by earlier kernels of the stream, so the producer (before
    // its Q load and any unsafe chunk) and the softmax warps (before their
    // first write) wait for the predecessor; the work list and history rows
    // below `safe` were uploaded / written before the chain began.

    // every role walks the same item sequence (ItemIter) and skips the same idle items

    if (warp == 0) {
        if (lane == 0) {   // ---------------- TMA producer
            int g = 0, n = 0;
            ItemIter items(work, n_items, H);
            Work wk;
            int h;
            bool have = items.next(wk, h);
            uint64_t kpol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(kpol));
            // K and V of a chunk have their own ring slots.  KA: a K slot frees
            // when the chunk's S^T MMA completes, a V slot when its PV MMA does,
            // and K runs one chunk ahead of V (K(c+1) is issued before V(c)), so
            // the next S^T never waits behind this chunk's softmax
            int gv = 0, pv_row = -1, pv_c = 0;
            auto load_v = [&](int kv_row0, int c) {
                const int st = gv % ST;
                if (gv >= ST) mbar_wait(su32(&v_empty[st]), ((gv / ST) - 1) & 1);
                const uint32_t sb = base + st * Cf::STAGE;
                mbar_expect_tx(su32(&v_full[st]), SUB * Cf::KV_TILE);
                for (int s = 0; s < SUB; ++s)
                    tma_2d_ef(&tv, sb + Cf::V_OFF + s * Cf::KV_TILE, su32(&v_full[st]), s * 64, kv_row0 + c * CH,
                              kpol);
                ++gv;
            };
            auto load_kv = [&](int kv_row0, int c) {
                const int st = g % ST;
                if (g >= ST) mbar_wait(su32(&k_empty[st]), ((g / ST) - 1) & 1);
                const uint32_t sb = base + st * Cf::STAGE;
                mbar_expect_tx(su32(&k_full[st]), SUB * Cf::KV_TILE);
                for (int s = 0; s < SUB; ++s)
                    tma_2d_ef(&tk, sb + Cf::K_OFF + s * Cf::KV_TILE, su32(&k_full[st]), s * 64, kv_row0 + c * CH,
                              kpol);
                ++g;
                if (!KA) {
                    load_v(kv_row0, c);
                    return;
                }
                if (pv_row >= 0) load_v(pv_row, pv_c);
                pv_row = kv_row0;
                pv_c = c;
            };
            // first item: its leading history chunks before the dependency wait
            int pre = 0;
            if (have) {
                const int kv_row0 = (wk.slot * H + h) * cap + wk.split * SPLIT;
                while (pre < wk.nch && pre < ST && wk.split * SPLIT + (pre + 1) * CH <= wk.safe) load_kv(kv_row0, pre++);
            }
            pdl_wait();
            if (threadIdx.x == 0) APROBE(2);
            while (have) {
                const int slot = wk.slot, q0row = wk.q0row;
                const int qb = n & 1;
                if (n >= 2) mbar_wait(su32(&q_empty[qb]), ((n >> 1) - 1) & 1);
                mbar_expect_tx(su32(&q_full[qb]), SUB * Cf::R_TILE);
                for (int s = 0; s < SUB; ++s)
                    tma_2d(&tq, base + Cf::OFF_Q + (SUB * qb + s) * Cf::R_TILE, su32(&q_full[qb]), h * DH + s * 64,
                           q0row + wk.t0);
                const int kv_row0 = (slot * H + h) * cap + wk.split * SPLIT;
                if (n == 0) APROBE(3);
                for (int c = n == 0 ? pre : 0; c < wk.nch; ++c) load_kv(kv_row0, c);
                if (n < 2) APROBE(4 + n);
                ++n;
                have = items.next(wk, h);
            }
            if (pv_row >= 0) load_v(pv_row, pv_c);
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {   // ---------------- MMA issuer
            constexpr uint32_t ID1 = idesc(NQ, 0);   // S^T = K . Q^T   (A = K, K-major)
            constexpr uint32_t ID2 = idesc(NQ, 1) | (1u << 16);   // O^T = V^T . P^T (A = V, B = P^T: MN-major)
            // P^T swizzle: one atom spans the NQ queries (32 / 64 / 128 bytes) x 8 keys
            constexpr uint64_t PLT = NQ == 16 ? 6ull : NQ == 32 ? 4ull : 2ull;
            struct Pend {
                int g, st, ob, first, last;
            } pend{-1, 0, 0, 0, 0};
            auto pv = [&](const Pend& p) {
                const int sb = p.g & 1;
                mbar_wait(su32(&p_full[sb]), (p.g >> 1) & 1);
                mbar_wait(su32(&v_full[p.st]), (p.g / ST) & 1);
                fence_after();
                // A = V^T (MN-major): the second 64-dim block is LBO = KV_TILE past V0
                // (d_head 64: K0 of the same stage; those O^T rows are never read)
                const uint32_t vs = base + p.st * Cf::STAGE + Cf::V_OFF;
                const uint32_t ps = base + Cf::OFF_P + sb * Cf::P_BUF;
                const uint32_t d = tmem + 2 * NQ + p.ob * NQ;
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk) {
                    const uint64_t bdesc = (sdesc(ps + kk * 32 * NQ, Cf::P_BUF, 16 * NQ) & ~(7ull << 61)) | (PLT << 61);
                    umma(d, sdesc(vs + kk * 2048, Cf::KV_TILE, 1024), bdesc, ID2, (p.first && kk == 0) ? 0u : 1u);
                }
                commit(su32(&v_empty[p.st]));
                // (d_head 64: the PV A operand's upper block is this stage's K0)
                if (!K_EARLY) commit(su32(&k_empty[p.st]));
                commit(su32(&p_free[sb]));
                if (p.last) commit(su32(&o_full[p.ob]));
            };
            int g = 0, n = 0;
            ItemIter items(work, n_items, H);
            Work wk;
            int h;
            while (items.next(wk, h)) {
                const int qb = n & 1, ob = n & 1;
                mbar_wait(su32(&q_full[qb]), (n >> 1) & 1);
                if (n < 2) APROBE(6 + n);
                for (int c = 0; c < wk.nch; ++c, ++g) {
                    const int st = g % ST, sb = g & 1;
                    mbar_wait(su32(&k_full[st]), (g / ST) & 1);
                    if (g < 4) APROBE(8 + g);
                    if (g >= 2) mbar_wait(su32(&s_free[sb]), ((g >> 1) - 1) & 1);
                    fence_after();
                    const uint32_t ks = base + st * Cf::STAGE + Cf::K_OFF;
                    const uint32_t qs = base + Cf::OFF_Q + SUB * qb * Cf::R_TILE;
#pragma unroll
                    for (int kk = 0; kk < DH / 16; ++kk) {
                        const uint32_t sub = kk >> 2, in = (kk & 3) * 32;
                        umma(tmem + sb * NQ, sdesc(ks + sub * Cf::KV_TILE + in, 16, 1024),
                             sdesc(qs + sub * Cf::R_TILE + in, 16, 1024), ID1, kk > 0);
                    }
                    commit(su32(&s_full[sb]));
                    if (K_EARLY) commit(su32(&k_empty[st]));
                    if (c == wk.nch - 1) commit(su32(&q_empty[qb]));
                    // O^T += V^T P^T of the previous chunk while the softmax works on this one
                    if (pend.g >= 0) pv(pend);
                    if (c == 0 && n >= 2) mbar_wait(su32(&o_free[ob]), ((n >> 1) - 1) & 1);
                    pend = Pend{g, st, ob, c == 0, c == wk.nch - 1};
                }
                ++n;
            }
            if (pend.g >= 0) pv(pend);
        }
        __syncwarp();
    } else {
        // ---------------- softmax / epilogue (SG groups of 4 warps from warp 2)
        // group grp owns query columns [grp*CQ, (grp+1)*CQ) of the tile: all
        // per-column rules are column-local, so splitting columns over groups
        // changes no decision, only who computes it
        pdl_wait();
        const int grp = SG == 1 ? 0 : (warp - 2) >> 2;
        const int wq = warp & 3;                 // TMEM lane quarter this warp may access
        const int key = wq * 32 + lane;          // key within the chunk (S^T lane) = head dim (O^T lane)
        const int tid = threadIdx.x - 64 - grp * 128;   // 0..127 within the group
        const int c_off = grp * CQ;
        float* red_g = red + grp * 4 * CQ;       // this group's [4][CQ] partials
        float* fin_g = fin + c_off;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const float C = 1.4426950408889634f / sqrtf((float)DH);   // log2(e) / sqrt(dh)
        // P^T row of this key: NQ bf16 (MN-major B operand), 16-byte chunks swizzled
        const uint32_t prow = (uint32_t)key * (2 * NQ);
        const uint32_t pswz = NQ == 16 ? ((key >> 2) & 1) : NQ == 32 ? ((key >> 1) & 3) : (key & 7);
        int g = 0, n = 0;
        ItemIter items(work, n_items, H);
        Work wk;
        int h;
        while (items.next(wk, h)) {
            const int qn = wk.qn, off = wk.off, q0row = wk.q0row;
            const int L = off + qn, s0 = wk.split * SPLIT, ob = n & 1;
            // valid query columns of this group (uniform; may be 0)
            const int ncol = max(0, min(NQ, qn - wk.t0) - c_off);
            const int dlim = off + wk.t0 + c_off;   // local column j sees keys kp <= dlim + j
            float l_t[CQ];
#pragma unroll
            for (int j = 0; j < CQ; ++j) l_t[j] = 0.f;
            for (int c = 0; c < wk.nch; ++c, ++g) {
                const int sb = g & 1;
                const bool first = c == 0;
                mbar_wait(su32(&s_full[sb]), (g >> 1) & 1);
                if (g < 4 && threadIdx.x == 64) APROBE(12 + g);
                fence_after();
                float x[CQ];
                if (ncol > 0) ldq_nowait<CQ>(tmem + lane_off + sb * NQ + c_off, x, ncol);
                ld_wait();
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(su32(&s_free[sb]));
                const int cbase = s0 + c * CH, kp = cbase + key;
                if (cbase + CH - 1 > dlim) {   // chunk crosses the causal diagonal / the end (uniform)
#pragma unroll
                    for (int j = 0; j < CQ; ++j)
                        if (!(kp <= dlim + j && kp < L)) x[j] = -INFINITY;
                }
                bool reduce = first;
                if (!first) {
                    bool over = false;
#pragma unroll
                    for (int j = 0; j < CQ; ++j)
                        if (j < ncol) over |= x[j] > thr[c_off + j];
                    reduce = sm_vote_any(over, grp);
                }
                if (reduce) {
                    // exact chunk max; a column's reference moves only when its own
                    // scores leave the window (first chunk: set unconditionally)
                    col_reduce<CQ, true>(x, red_g, fin_g, wq, lane, tid, grp);
                    bool resc = false;
                    if (tid < CQ) {
                        const int cc = c_off + tid;
                        const float cm = fin_g[tid] * C, mo = first ? -INFINITY : mref[cc];
                        float a = 1.f;
                        if (first || cm > mo + TH) {
                            a = mo == -INFINITY ? 0.f : fast_exp2(mo - cm);
                            resc = !first;
                            mref[cc] = cm;
                            thr[cc] = (cm + TH) / C;
                        }
                        alph[cc] = a;
                    }
                    const bool any_rescale = sm_vote_any(resc, grp);   // also publishes mref / thr / alph
                    if (!first) {
#pragma unroll
                        for (int j = 0; j < CQ; ++j) l_t[j] *= alph[c_off + j];
                    }
                    if (any_rescale) {
                        // O^T holds chunks < c: wait for the previous PV, rescale this group's columns
                        mbar_wait(su32(&p_free[(g - 1) & 1]), ((g - 1) >> 1) & 1);
                        fence_after();
                        const uint32_t to = tmem + lane_off + 2 * NQ + ob * NQ + c_off;
                        if constexpr (CQ == 8) {
                            float o[8];
                            ld8_nowait(to, o);
                            ld_wait();
#pragma unroll
                            for (int j = 0; j < 8; ++j) o[j] *= alph[c_off + j];
                            st8(to, o);
                        } else {
#pragma unroll
                            for (int j0 = 0; j0 < CQ; j0 += 16) {
                                float o[16];
                                ld16_nowait(to + j0, o);
                                ld_wait();
#pragma unroll
                                for (int j = 0; j < 16; ++j) o[j] *= alph[c_off + j0 + j];
                                st16(to + j0, o);
                            }
                        }
                        st_wait();
                        fence_before();
                    }
                }
                // P (bf16) for this chunk; the previous user of the buffer (PV g-2) must be done
                if (g >= 2) mbar_wait(su32(&p_free[sb]), ((g >> 1) - 1) & 1);
                const uint32_t pb = base + Cf::OFF_P + sb * Cf::P_BUF + prow;
#pragma unroll
                for (int j0 = 0; j0 < CQ; j0 += 8) {
                    if (j0 >= ncol) break;   // columns past the tile's rows: never read back
                    uint32_t pk[4];
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        const float4 m4 = *reinterpret_cast<const float4*>(mref + c_off + j0 + (u & 4));
                        const float ma = (u & 2) ? m4.z : m4.x, mb = (u & 2) ? m4.w : m4.y;
                        const float p0 = fast_exp2(fmaf(x[j0 + u], C, -ma));
                        const float p1 = fast_exp2(fmaf(x[j0 + u + 1], C, -mb));
                        l_t[j0 + u] += p0;
                        l_t[j0 + u + 1] += p1;
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                        pk[u >> 1] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    const uint32_t dst = pb + (((((uint32_t)(c_off + j0)) >> 3) ^ pswz) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(pk[0]), "r"(pk[1]),
                                 "r"(pk[2]), "r"(pk[3])
                                 : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P -> tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive(su32(&p_full[sb]));
                if (g < 4 && threadIdx.x == 64) APROBE(16 + g);
            }
            // ---- epilogue: l per column (fixed-order block sum), O^T lane = head dim
            col_reduce<CQ, false>(l_t, red_g, fin_g, wq, lane, tid, grp);
            if (n < 2 && threadIdx.x == 64) APROBE(20 + n);
            mbar_wait(su32(&o_full[ob]), (n >> 1) & 1);
            if (n < 2 && threadIdx.x == 64) APROBE(22 + n);
            fence_after();
            float o[CQ];
            if (ncol > 0) ldq_nowait<CQ>(tmem + lane_off + 2 * NQ + ob * NQ + c_off, o, CQ);
            ld_wait();
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(su32(&o_free[ob]));
#pragma unroll
            for (int j = 0; j < CQ; ++j) {
                const int t = wk.t0 + c_off + j;
                if (j >= ncol || off + t < s0) continue;   // padded row / row does not see this split
                const int row = q0row + t;
                const float l = fin_g[j];
                if (DH < 128 && key >= DH) continue;   // O^T lanes past d_head: padding rows
                if (off + t < SPLIT) {   // whole history in split 0: normalised output
                    out[((int64_t)row * H + h) * DH + key] = __float2bfloat16_rn(o[j] / l);
                } else {
                    const int64_t idx = ((int64_t)row * H + h) * max_splits + wk.split;
                    part_o[idx * DH + key] = o[j];
                    if (key == 0) {
                        part_ml[idx * 2] = mref[c_off + j] * 0.6931471805599453f;   // natural-log units for the combine
                        part_ml[idx * 2 + 1] = l;
                    }
                }
            }
            if (n < 2 && threadIdx.x == 64) APROBE(24 + n);
            ++n;
        }
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) APROBE(26);
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cf::TMEM_COLS)
                     : "memory");
    trace_end(tr, t_start);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#ifdef BASS_ATTN_PROBE
void attn_probe_set(void* p) { BASS_CUDA(cudaMemcpyToSymbol(g_attn_probe, &p, sizeof(p))); }
#endif

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

// K / V cache tensor maps (rows of d_head elements, 64-column x 128-row boxes),
// keyed by everything they encode
static const CUtensorMap& kv_map(const void* ptr, int64_t rows, int dh) {
    static std::map<std::tuple<const void*, int64_t, int>, CUtensorMap> cache;
    auto key = std::make_tuple(ptr, rows, dh);
    auto it = cache.find(key);
    if (it == cache.end()) it = cache.emplace(key, map2d(ptr, rows, dh, dh, CH)).first;
    return it->second;
}

template <int NQ, int DH, int STG = Cfg<NQ, DH>::STAGES>
static void launch(bass_ctx* ctx, const AttnPlan& p, const CUtensorMap& tk, const CUtensorMap& tv, const Seqs& seqs,
                   const Work* wp, int nw, float* po, float* pml, __nv_bfloat16* out) {
    if constexpr (NQ == 16 && DH == 128 && STG == 2) {
        // long histories stream better with a third K/V stage
        if (p.max_len > 768) {
            launch<16, DH, 3>(ctx, p, tk, tv, seqs, wp, nw, po, pml, out);
            return;
        }
        // single-row decode blocks with more (sequence, head) items than SMs
        // (regular decoding, the b = 64 draft): a one-stage ring (82 KB), two
        // CTAs per SM, one item each — the per-item latency chains overlap
        // instead of running back to back (regular decoding 3.30 -> 3.26
        // ms/token; the speculative verify / b = 8 draft keep two stages)
        if (p.max_len <= 512 && p.max_q == 1 && nw * p.H > ctx->sm_count) {
            launch<16, DH, 1>(ctx, p, tk, tv, seqs, wp, nw, po, pml, out);
            return;
        }
    }
    using Cf = Cfg<NQ, DH, STG>;
    static unsigned attr = 0;
    once_per_device(attr, [] {
        BASS_CUDA(cudaFuncSetAttribute(attn_stream_kernel<NQ, DH, STG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cf::SMEM));
    });
    const int n_items = nw * p.H;
    const int grid = std::max(1, std::min(n_items, (STG == 1 ? 2 : 1) * ctx->sm_count));
    BASS_CUDA(launch_pdl(attn_stream_kernel<NQ, DH, STG>, dim3(grid), dim3(attn_threads(NQ)), (size_t)Cf::SMEM,
                         ctx->stream, p.tq, tk, tv, seqs, wp, n_items, p.H, p.cap, po, pml, p.mc, out,
                         ctx->trace(grid, BASS_TR_ATTN)));
}

}  // namespace ast

int stream_split_len() { return ast::SPLIT; }
int stream_chunk_len() { return ast::CH; }
int stream_split_chunks() { return ast::SPLIT_CH; }
// query tile: the smallest of 16 / 32 / 64 columns covering the block (q = 33-64
// as two NQ = 32 tiles measured slower: each tile streams the history again)
int stream_nq_for(int q) { return q <= 16 ? 16 : q <= 32 ? 32 : 64; }
int stream_items_per_seq(int q, int max_len) {
    const int nq = stream_nq_for(q);
    const int chunks = (std::max(max_len, 1) + ast::CH - 1) / ast::CH;
    return ((q + nq - 1) / nq) * ((chunks + ast::SPLIT_CH - 1) / ast::SPLIT_CH);
}

void stream_attention_plan_dev(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots,
                               const std::vector<int32_t>& qn, int H, int dh, int cap, const void* work,
                               int work_stride, int max_len, AttnPlan& plan) {
    using namespace ast;
    (void)ctx;
    const int n_seq = (int)qn.size();
    int max_qn = 0;
    for (int v : qn) max_qn = std::max(max_qn, v);
    const int NQ = stream_nq_for(max_qn);
    plan.tq = map2d(q, M, (int64_t)H * dh, (int64_t)H * dh, NQ);
    plan.dh = dh;
    plan.NQ = NQ;
    plan.max_q = max_qn;
    plan.pad_len = 0;
    plan.max_len = max_len;
    plan.strategy = strategy;
    plan.H = H;
    plan.cap = cap;
    plan.n_slots = n_slots;
    plan.mc = (cap + SPLIT - 1) / SPLIT;
    plan.stream = true;
    plan.needs_combine = max_len > SPLIT;   // some row may span two splits (single-split rows skip the combine)
    plan.first.resize(n_seq + 1);
    for (int i = 0; i <= n_seq; ++i) plan.first[i] = i * work_stride;   // idle items pad each region
    plan.work = const_cast<void*>(work);
    plan.valid = true;
}

bool tc_attention_supported(int dtype, int dh) { return dtype == BASS_BF16 && (dh == 128 || dh == 64); }

// Plan: work items (seq, q tile, split, chunks seen) — RAGGED/SPLIT exact,
// PAD over the padded [max q] x [max L] grid (padded keys streamed, masked).
static int stream_nq(const std::vector<int32_t>& qn) {
    int max_qn = 0;
    for (int v : qn) max_qn = std::max(max_qn, v);
    return stream_nq_for(max_qn);
}

// work items (Work, 8 int32 each) in sequence order; first[i] = sequence i's first item
static bool stream_items(int strategy, const std::vector<int32_t>& slot, const std::vector<int32_t>& qn,
                         const std::vector<int32_t>& off, const std::vector<int32_t>* safe, std::vector<int32_t>& w,
                         std::vector<int>* first) {
    using namespace ast;
    const int n_seq = (int)qn.size();
    int max_qn = 0, max_L = 0;
    for (int i = 0; i < n_seq; ++i) {
        max_qn = std::max(max_qn, qn[i]);
        max_L = std::max(max_L, off[i] + qn[i]);
    }
    const int NQ = stream_nq(qn);
    const size_t w0 = w.size();
    bool multi = false;
    int q0 = 0;   // rows are laid out sequence after sequence
    for (int i = 0; i < n_seq; ++i) {
        if (first) (*first)[i] = (int)(w.size() - w0) / 8;
        const int rows = strategy == BASS_PAD ? max_qn : qn[i];
        // split-major, query tile minor: the tiles of one (split, head) stream
        // the same K/V rows H items apart, i.e. concurrently, so the later
        // tiles read them from L2
        auto n_chunks = [&](int t0) {
            const int last = strategy == BASS_PAD ? max_L - 1 : off[i] + std::min(qn[i], t0 + NQ) - 1;
            return last / CH + 1;
        };
        const int sf = std::min(off[i], safe ? (*safe)[i] : off[i]);
        for (int s = 0; s * SPLIT_CH < n_chunks(rows - 1); ++s) {
            for (int t0 = 0; t0 < rows; t0 += NQ) {
                const int nc = n_chunks(t0);
                if (s * SPLIT_CH >= nc) continue;
                w.insert(w.end(), {slot[i], q0, qn[i], off[i], t0, s, std::min(SPLIT_CH, nc - s * SPLIT_CH), sf});
                if (s > 0) multi = true;
            }
        }
        q0 += qn[i];
    }
    if (first) (*first)[n_seq] = (int)(w.size() - w0) / 8;
    return multi;
}

void stream_attention_work(int strategy, const std::vector<int32_t>& slot, const std::vector<int32_t>& qn,
                           const std::vector<int32_t>& off, const std::vector<int32_t>& safe,
                           std::vector<int32_t>& w) {
    stream_items(strategy, slot, qn, off, &safe, w, nullptr);
}

void stream_attention_plan(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots,
                           const std::vector<int32_t>& slot, const std::vector<int32_t>& qn,
                           const std::vector<int32_t>& off, int H, int dh, int cap, DevBuf& work_buf,
                           AttnPlan& plan, const void* pre_work) {
    using namespace ast;
    const int n_seq = (int)qn.size();
    int max_L = 0, max_qn = 0;
    for (int i = 0; i < n_seq; ++i) {
        max_L = std::max(max_L, off[i] + qn[i]);
        max_qn = std::max(max_qn, qn[i]);
    }
    const int NQ = stream_nq(qn);
    std::vector<int32_t> w;
    std::vector<int> first(n_seq + 1, 0);
    // uploaded right here (a copy is a full barrier): every committed row is safe
    const bool multi = stream_items(strategy, slot, qn, off, nullptr, w, &first);
    Work* wd;
    if (pre_work) {   // uploaded with the step's metadata (forward_premeta)
        wd = (Work*)const_cast<void*>(pre_work);
    } else {
        wd = (Work*)work_buf.need(std::max<size_t>(w.size(), 8) * 4, ctx->stream);
        void* hst = ctx->staging.take(w.size() * 4);
        if (!hst) {
            ctx->sync();
            hst = ctx->staging.take(w.size() * 4);
        }
        std::memcpy(hst, w.data(), w.size() * 4);
        BASS_CUDA(cudaMemcpyAsync(wd, hst, w.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
        ctx->h2d_bytes += (int64_t)w.size() * 4;
    }
    plan.tq = map2d(q, M, (int64_t)H * dh, (int64_t)H * dh, NQ);
    plan.dh = dh;
    plan.NQ = NQ;
    plan.max_q = max_qn;
    plan.pad_len = strategy == BASS_PAD ? max_L : 0;
    plan.max_len = max_L;
    plan.strategy = strategy;
    plan.H = H;
    plan.cap = cap;
    plan.n_slots = n_slots;
    plan.mc = (cap + SPLIT - 1) / SPLIT;   // splits per row (partial buffer stride)
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
    const CUtensorMap& tk = kv_map(kc, kv_rows, p.dh);
    const CUtensorMap& tv = kv_map(vc, kv_rows, p.dh);
    const Work* wd = static_cast<const Work*>(p.work);
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out);
    auto go = [&](const Work* wp, int nw) {
        if (nw == 0) return;
        const bool d64 = p.dh == 64;
        switch (p.NQ) {
            case 16: d64 ? launch<16, 64>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o)
                         : launch<16, 128>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
            case 32: d64 ? launch<32, 64>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o)
                         : launch<32, 128>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
            default: d64 ? launch<64, 64>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o)
                         : launch<64, 128>(ctx, p, tk, tv, seqs_dev, wp, nw, part_o, part_ml, o); break;
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
