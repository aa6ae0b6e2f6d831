// K9 on thread-block clusters: one logits row is shaped / sampled /
// accept-tested by a cluster of CL_CTAS CTAs, each owning a contiguous
// 1/CL_CTAS of the vocabulary; every cross-CTA reduction (argmax, sums, the
// radix-select histograms, prefix scans) goes through distributed shared
// memory and is combined in cluster-rank order, so every CTA of the cluster
// reaches the same decisions and the results are deterministic.
//
// The arithmetic is the single-CTA restatement of ref:sampling.py:69-146
// (shaping: softmax(z / T) with max subtraction in fp64, top-p nucleus kept as
// "keys above a boundary + ties up to an id" found by a 4-pass radix select
// over the orderable logit key, renormalised; inverse CDF
// searchsorted(cumsum(p), u * csum[-1], 'right'); accept iff u p(x) < q(x),
// else resample normalize(max(q - p, 0)) with the second draw), distributed:
// only the order in which fp64 partial sums are added differs.
//
// A row used to be one CTA (512 threads) walking V = 50272 logits through
// fp64 exp and four radix passes — ~300 us per row on one SM while the other
// 147 idle (C3 sampled decoding, regular_pick 341 us per launch); a cluster
// cuts the per-row latency by ~CL_CTAS and spreads a step's rows over SMs.
#pragma once
#include "sampling_kernels.cuh"

namespace bass {

constexpr int CL_CTAS = 8, CL_THREADS = 256;

BASS_DEV uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
BASS_DEV void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
BASS_DEV uint32_t cl_map(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
BASS_DEV double cl_ldd(const double* p, uint32_t rank) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(cl_map(p, rank)) : "memory");
    return v;
}
BASS_DEV float cl_ldf(const float* p, uint32_t rank) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cl_map(p, rank)) : "memory");
    return v;
}
BASS_DEV int cl_ldi(const int* p, uint32_t rank) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(cl_map(p, rank)) : "memory");
    return v;
}

struct ClSmem {
    int cnt[256];                          // this CTA's bucket counts (current pass)
    double wmass[CL_THREADS / 32][256];    // per-warp bucket masses (merged in warp order)
    int hcnt[4][256];                      // per pass: this CTA's histogram (read by the cluster)
    double hmass[4][256];
    int gcnt[256];                         // cluster-merged histogram (rank order)
    double gmass[256];
    double dred[33];
    float fred[33];
    int ired[33];
    double xd[24];                         // cluster exchange slots, each used once per kernel
    int xi[24];
    float xf[8];
    Shaped sh;
    int sel, found;
    double before;
};

// sequence of cluster reductions of one kernel: every CTA runs the same
// sequence, each reduction owns fresh exchange slots (no reuse -> one barrier)
struct Cl {
    ClSmem& sm;
    int c0, c1;   // this CTA's vocabulary range
    int nd = 0, ni = 0, nf = 0;
    BASS_DEV Cl(ClSmem& s, int V) : sm(s) {
        const int r = (int)cl_rank();
        c0 = (int)((int64_t)r * V / CL_CTAS);
        c1 = (int)((int64_t)(r + 1) * V / CL_CTAS);
    }
    // block value (valid in every thread) -> cluster sum in rank order (every thread)
    BASS_DEV double sum(double block_v) {
        const int k = nd++;
        if (threadIdx.x == 0) sm.xd[k] = block_v;
        cl_sync();
        double s = 0.0;
        for (int r = 0; r < CL_CTAS; ++r) s += cl_ldd(&sm.xd[k], r);
        return s;
    }
    // exclusive prefix over ranks + total
    BASS_DEV double exscan(double block_v, double* total) {
        const int k = nd++;
        if (threadIdx.x == 0) sm.xd[k] = block_v;
        cl_sync();
        const int me = (int)cl_rank();
        double pre = 0.0, s = 0.0;
        for (int r = 0; r < CL_CTAS; ++r) {
            const double v = cl_ldd(&sm.xd[k], r);
            if (r < me) pre += v;
            s += v;
        }
        *total = s;
        return pre;
    }
    BASS_DEV int exscan_i(int block_v, int* total) {
        const int k = ni++;
        if (threadIdx.x == 0) sm.xi[k] = block_v;
        cl_sync();
        const int me = (int)cl_rank();
        int pre = 0, s = 0;
        for (int r = 0; r < CL_CTAS; ++r) {
            const int v = cl_ldi(&sm.xi[k], r);
            if (r < me) pre += v;
            s += v;
        }
        *total = s;
        return pre;
    }
    BASS_DEV int min_i(int block_v) {
        const int k = ni++;
        if (threadIdx.x == 0) sm.xi[k] = block_v;
        cl_sync();
        int m = 0x7fffffff;
        for (int r = 0; r < CL_CTAS; ++r) m = min(m, cl_ldi(&sm.xi[k], r));
        return m;
    }
    BASS_DEV double max_d(double block_v) {
        const int k = nd++;
        if (threadIdx.x == 0) sm.xd[k] = block_v;
        cl_sync();
        double m = -1.0;
        for (int r = 0; r < CL_CTAS; ++r) m = fmax(m, cl_ldd(&sm.xd[k], r));
        return m;
    }
    BASS_DEV ArgMax argmax(ArgMax block_a) {
        const int kf = nf++, ki = ni++;
        if (threadIdx.x == 0) {
            sm.xf[kf] = block_a.v;
            sm.xi[ki] = block_a.i;
        }
        cl_sync();
        ArgMax g{-INFINITY, 0x7fffffff};
        for (int r = 0; r < CL_CTAS; ++r) g = better(g, ArgMax{cl_ldf(&sm.xf[kf], r), cl_ldi(&sm.xi[ki], r)});
        return g;
    }
};

// row argmax (first index on ties) and log-sum-exp over the cluster
BASS_DEV ArgMax cl_row_argmax(const float* __restrict__ row, Cl& cl) {
    ArgMax a{-INFINITY, 0x7fffffff};
    for (int i = cl.c0 + threadIdx.x; i < cl.c1; i += blockDim.x) a = better(a, ArgMax{row[i], i});
    return cl.argmax(block_argmax(a, cl.sm.fred, cl.sm.ired));
}

// Shape one row (ref:sampling.py:69-104); e: the row's fp64 scratch (each CTA
// writes its own range).  Leaves the summary in cl.sm.sh (every thread).
BASS_DEV void cl_shape_row(const float* __restrict__ row, int V, double T, double top_p, double* __restrict__ e,
                           Cl& cl) {
    ClSmem& sm = cl.sm;
    const int tid = threadIdx.x, nt = blockDim.x;
    const ArgMax a = cl_row_argmax(row, cl);
    if (T == 0.0) {
        __syncthreads();
        if (tid == 0) {
            sm.sh = Shaped{};
            sm.sh.greedy = 1;
            sm.sh.argmax = a.i;
        }
        __syncthreads();
        return;
    }
    const double zmax = double(a.v) / T;
    double s = 0.0;
    for (int i = cl.c0 + tid; i < cl.c1; i += nt) {
        const double ei = exp(double(row[i]) / T - zmax);   // exp(-inf) = 0
        e[i] = ei;
        s += ei;
    }
    const double S = cl.sum(block_sum(s, sm.dred));
    // radix select over the key, descending: the bucket where the running
    // mass (descending key order) first reaches top_p
    uint32_t prefix = 0;
    double before = 0.0;
    int keep_all = 0;
    const int lane = tid & 31, wid = tid >> 5;
    for (int pass = 0; pass < 4 && !keep_all; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int b = tid; b < 256; b += nt) sm.cnt[b] = 0;
        for (int b = tid; b < (CL_THREADS / 32) * 256; b += nt) (&sm.wmass[0][0])[b] = 0.0;
        __syncthreads();
        // warp-aggregated: lanes hitting the same bucket are summed (lane
        // order) and the group's leader adds to its warp's private histogram
        for (int i0 = cl.c0; i0 < cl.c1; i0 += nt) {   // uniform trip count: warps stay converged
            const int i = i0 + tid;
            int b = -1;
            double m = 0.0;
            if (i < cl.c1) {
                const uint32_t k = fkey(row[i]);
                if (pass == 0 || (k >> (shift + 8)) == prefix) {
                    b = (k >> shift) & 255;
                    m = e[i] / S;
                }
            }
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            if (b >= 0) {
                double g = 0.0;
                for (unsigned mm = peers; mm; mm &= mm - 1) g += __shfl_sync(peers, m, __ffs(mm) - 1);
                if (lane == __ffs(peers) - 1) {
                    atomicAdd(&sm.cnt[b], __popc(peers));
                    sm.wmass[wid][b] += g;
                }
            }
        }
        __syncthreads();
        for (int b = tid; b < 256; b += nt) {
            double mb = 0.0;
#pragma unroll
            for (int w = 0; w < CL_THREADS / 32; ++w) mb += sm.wmass[w][b];
            sm.hmass[pass][b] = mb;
            sm.hcnt[pass][b] = sm.cnt[b];
        }
        cl_sync();   // every CTA's histogram of this pass is published
        for (int b = tid; b < 256; b += nt) {
            int c = 0;
            double mb = 0.0;
            for (int r = 0; r < CL_CTAS; ++r) {
                c += cl_ldi(&sm.hcnt[pass][b], r);
                mb += cl_ldd(&sm.hmass[pass][b], r);
            }
            sm.gcnt[b] = c;
            sm.gmass[b] = mb;
        }
        __syncthreads();
        if (tid == 0) {
            double run = before;
            int sel = -1, last_nonempty = -1;
            for (int b = 255; b >= 0; --b) {
                if (sm.gcnt[b] == 0) continue;
                last_nonempty = b;
                if (run + sm.gmass[b] >= top_p) {
                    sel = b;
                    break;
                }
                run += sm.gmass[b];
            }
            if (sel < 0) {
                // never reaches top_p: at pass 0 keep everything (searchsorted
                // clamps to n-1); deeper, take the last bucket
                if (pass == 0) {
                    sm.found = 0;
                } else {
                    sel = last_nonempty;
                    double r2 = before;
                    for (int b = 255; b > sel; --b) r2 += sm.gmass[b];
                    run = r2;
                    sm.found = 1;
                }
            } else {
                sm.found = 1;
            }
            sm.sel = sel;
            sm.before = run;
        }
        __syncthreads();
        if (!sm.found) {
            keep_all = 1;
            break;
        }
        prefix = (prefix << 8) | uint32_t(sm.sel);
        before = sm.before;
        __syncthreads();
    }
    int id_lim = 0x7fffffff;
    if (!keep_all) {
        // ties at the boundary key share one probability f; members kept in id order
        const int g = sm.gcnt[sm.sel];
        const uint32_t ukey = prefix;
        __syncthreads();
        if (tid == 0) sm.found = -1;
        __syncthreads();
        for (int i = cl.c0 + tid; i < cl.c1; i += nt)
            if (fkey(row[i]) == ukey) atomicMax(&sm.found, i);
        __syncthreads();
        const double f = cl.max_d(sm.found >= 0 ? e[sm.found] / S : -1.0);
        int need = 0;
        {
            double run = before;
            while (need < g) {
                run += f;
                ++need;
                if (run >= top_p) break;
            }
        }
        if (need < g) {
            // id of the need-th member in ascending id order
            const int n = cl.c1 - cl.c0, chunk = (n + nt - 1) / nt;
            const int lo = cl.c0 + min(n, tid * chunk), hi = cl.c0 + min(n, (tid + 1) * chunk);
            int c = 0;
            for (int i = lo; i < hi; ++i) c += fkey(row[i]) == ukey;
            int tot;
            const int pre_blk = block_exclusive_scan(c, sm.ired, &tot);
            int all;
            const int pre = cl.exscan_i(tot, &all) + pre_blk;
            __syncthreads();
            if (tid == 0) sm.found = 0x7fffffff;
            __syncthreads();
            if (pre < need && pre + c >= need) {
                int cc = pre;
                for (int i = lo; i < hi; ++i)
                    if (fkey(row[i]) == ukey && ++cc == need) {
                        sm.found = i;
                        break;
                    }
            }
            __syncthreads();
            id_lim = cl.min_i(sm.found);
        }
    }
    Shaped sh{};
    sh.greedy = 0;
    sh.argmax = a.i;
    sh.S = S;
    sh.keep_all = keep_all;
    sh.ukey = keep_all ? 0u : prefix;
    sh.id_lim = id_lim;
    double kf = 0.0;
    for (int i = cl.c0 + tid; i < cl.c1; i += nt)
        if (sh_kept(sh, row[i], i)) kf += e[i] / S;
    sh.Kf = cl.sum(block_sum(kf, sm.dred));
    __syncthreads();
    if (tid == 0) sm.sh = sh;
    __syncthreads();
}

// First index whose running sum (id order) of w(i) exceeds u * total, clamped
// to V-1 (ref:sampling.py:112-115), over the cluster.
template <typename W>
BASS_DEV int cl_inverse_cdf(int V, double u, W w, Cl& cl) {
    ClSmem& sm = cl.sm;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int n = cl.c1 - cl.c0, chunk = (n + nt - 1) / nt;
    const int lo = cl.c0 + min(n, tid * chunk), hi = cl.c0 + min(n, (tid + 1) * chunk);
    double loc = 0.0;
    for (int i = lo; i < hi; ++i) loc += w(i);
    double blk_total;
    const double pre_blk = block_exclusive_scan(loc, sm.dred, &blk_total);
    double total;
    const double pre = cl.exscan(blk_total, &total) + pre_blk;
    const double target = u * total;
    // the chosen element has positive weight (csum[i-1] <= target < csum[i]);
    // every thread proposes its first crossing, the cluster keeps the smallest
    int cand = 0x7fffffff;
    double c = pre;
    for (int i = lo; i < hi; ++i) {
        const double wi = w(i);
        c += wi;
        if (c > target && wi > 0.0) {
            cand = i;
            break;
        }
    }
    ArgMax am{-float(cand), cand};
    am = block_argmax(am, sm.fred, sm.ired);
    const int idx = cl.min_i(am.i);
    return idx == 0x7fffffff ? V - 1 : min(idx, V - 1);
}

// accept / resample given both rows' shaping: -1 accepted, else the corrected
// token; -2 zero draft probability, -3 empty residual (ref:sampling.py:118-146)
BASS_DEV int cl_accept_shaped(const float* qrow, const float* prow, int V, const double* eq, const double* ep,
                              const Shaped& sq, const Shaped& sp, int tok, Pcg64& g, Cl& cl) {
    const double px = sh_prob(sp, prow, ep, tok);
    const double qx = sh_prob(sq, qrow, eq, tok);
    if (px <= 0.0) return -2;
    const double u = pcg64_double(g);
    if (u * px < qx) return -1;
    auto r = [&](int k) {
        const double d = sh_prob(sq, qrow, eq, k) - sh_prob(sp, prow, ep, k);
        return d > 0.0 ? d : 0.0;
    };
    double loc = 0.0;
    for (int k = cl.c0 + threadIdx.x; k < cl.c1; k += blockDim.x) loc += r(k);
    const double R = cl.sum(block_sum(loc, cl.sm.dred));
    if (R <= 0.0) return -3;
    const double u2 = pcg64_double(g);
    return cl_inverse_cdf(V, u2, [&](int k) { return r(k) / R; }, cl);
}

// ------------------------------------------------------------------ kernels
// Every kernel: grid.x = CL_CTAS x rows, cluster (CL_CTAS, 1, 1); the row is
// blockIdx.x / CL_CTAS.  The trailing cl_sync keeps each CTA's shared memory
// alive until the whole cluster is done reading it.

// sampled draft step: proposal ~ shape(row), uniform = RNG(seed, sid, DRAFT, pos).
// With the acceptance harness on (d.align >= 0) the proposal is the keyed
// override token and the row becomes a point mass on it — the reference's
// SyntheticAlignedDraft row form (ref:model.py:379-389: logits -inf except 0
// at y) — so the verify tests and resamples against the distribution the
// proposal was actually drawn from (speculative sampling stays exact when the
// override tokens do not depend on the verify draws).
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_draft_sample_kernel(float* __restrict__ logits, int V, double T, double top_p, uint64_t seed,
                           double* scratch, DraftPick d) {
    __shared__ ClSmem sm;
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x / CL_CTAS;
    Cl cl(sm, V);
    const float* row = logits + (int64_t)i * V;
    double* e = scratch + (int64_t)i * V;
    cl_shape_row(row, V, T, top_p, e, cl);
    const int slot = d.slot[i], pos = d.pos[i];
    Pcg64 g = pcg64_from_key(seed, uint64_t(d.sid[slot]), 0u, uint64_t(pos));
    const double u = pcg64_double(g);
    const Shaped sh = sm.sh;
    const int tok = cl_inverse_cdf(V, u, [&](int k) { return sh_prob(sh, row, e, k); }, cl);
    const int prop = aligned_override(d, slot, pos, V, tok);
    if (threadIdx.x == 0 && cl_rank() == 0) d.proposals[slot * d.pstride + d.j] = prop;
    if (d.align >= 0.0) {
        cl_sync();   // every CTA is done reading the row
        float* w = logits + (int64_t)i * V;
        for (int k = cl.c0 + threadIdx.x; k < cl.c1; k += blockDim.x) w[k] = k == prop ? 0.f : -INFINITY;
    }
    cl_sync();
}

// standalone shaping + sampling (bass_shape_sample)
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_shape_sample_kernel(const float* __restrict__ logits, int V, double T, double top_p,
                           const double* __restrict__ u, double* scratch, int32_t* __restrict__ tok,
                           double* __restrict__ probs) {
    __shared__ ClSmem sm;
    const int i = blockIdx.x / CL_CTAS;
    Cl cl(sm, V);
    const float* row = logits + (int64_t)i * V;
    double* e = scratch + (int64_t)i * V;
    cl_shape_row(row, V, T, top_p, e, cl);
    const Shaped sh = sm.sh;
    if (probs)
        for (int k = cl.c0 + threadIdx.x; k < cl.c1; k += blockDim.x)
            probs[(int64_t)i * V + k] = sh_prob(sh, row, e, k);
    const int t = cl_inverse_cdf(V, u[i], [&](int k) { return sh_prob(sh, row, e, k); }, cl);
    if (threadIdx.x == 0 && cl_rank() == 0) tok[i] = t;
    cl_sync();
}

// standalone accept / resample of (q row, p row, token) pairs (bass_accept)
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_accept_pairs_kernel(const float* __restrict__ ql, const float* __restrict__ pl, int V, double T,
                           double top_p, const int32_t* __restrict__ tok, uint64_t seed,
                           const int64_t* __restrict__ sid, const int64_t* __restrict__ ctr, double* scratch,
                           int32_t* __restrict__ acc, int32_t* __restrict__ corr) {
    __shared__ ClSmem sm;
    const int i = blockIdx.x / CL_CTAS;
    Cl cl(sm, V);
    const float* q = ql + (int64_t)i * V;
    const float* p = pl + (int64_t)i * V;
    double* eq = scratch + (int64_t)i * 2 * V;
    double* ep = eq + V;
    cl_shape_row(q, V, T, top_p, eq, cl);
    const Shaped sq = sm.sh;
    __syncthreads();
    cl_shape_row(p, V, T, top_p, ep, cl);
    const Shaped sp = sm.sh;
    Pcg64 g = pcg64_from_key(seed, uint64_t(sid[i]), 1u, uint64_t(ctr[i]));
    const int c = cl_accept_shaped(q, p, V, eq, ep, sq, sp, tok[i], g, cl);
    if (threadIdx.x == 0 && cl_rank() == 0) {
        acc[i] = c == -1;
        corr[i] = c;
    }
    cl_sync();
}

// Verify, launch 1: shape every main row q (z = 0) and draft row p (z = 1)
// of the step, one cluster per row; e stays in the scratch, the summary in sh.
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_verify_shape_kernel(VerifyArgs a, Shaped* __restrict__ sh) {
    __shared__ ClSmem sm;
    pdl_trigger();
    pdl_wait();
    const int l = a.l, i = blockIdx.y;
    const int j = (a.phase == 2 ? l : 0) + blockIdx.x / CL_CTAS, z = a.phase == 2 ? 1 : blockIdx.z;
    if (a.phase == 1 && z == 1 && j == l) return;   // the bonus draft row comes later (whole cluster)
    Cl cl(sm, a.V);
    const int64_t r = (int64_t)i * (l + 1) + j;
    const float* row = z == 0 ? a.vlog + r * a.V : a.dlog + (int64_t)(j * a.nA + i) * a.V;
    double* e = a.scratch + r * 2 * a.V + (z == 0 ? 0 : a.V);
    cl_shape_row(row, a.V, a.T, a.top_p, e, cl);
    if (threadIdx.x == 0 && cl_rank() == 0) sh[r * 2 + z] = sm.sh;
    cl_sync();
}

// Verify, launch 2: per (j, i) the bonus draw (j = l) and accept / resample
// (ref:engine.py:292-343) — the same RNG streams and draws as the reference.
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_verify_accept_kernel(VerifyArgs a, const Shaped* __restrict__ sh) {
    __shared__ ClSmem sm;
    pdl_trigger();
    pdl_wait();
    const int j = (a.phase == 2 ? a.l : 0) + blockIdx.x / CL_CTAS, i = blockIdx.y, l = a.l;
    Cl cl(sm, a.V);
    const int slot = a.slot[i], pos = a.committed[i] + j;
    const int64_t sid = a.sid[slot];
    const int64_t r = (int64_t)i * (l + 1) + j;
    const float* q = a.vlog + r * a.V;
    const float* p = a.dlog + (int64_t)(j * a.nA + i) * a.V;
    const double* eq = a.scratch + r * 2 * a.V;
    const double* ep = eq + a.V;
    const Shaped sq = sh[r * 2], sp = sh[r * 2 + 1];
    int tok;
    if (j < l) {
        tok = a.proposals[slot * a.pstride + j];
    } else {
        Pcg64 gd = pcg64_from_key(a.seed, uint64_t(sid), 0u, uint64_t(pos));
        const double ub = pcg64_double(gd);
        tok = cl_inverse_cdf(a.V, ub, [&](int k) { return sh_prob(sp, p, ep, k); }, cl);
    }
    Pcg64 g = pcg64_from_key(a.seed, uint64_t(sid), 1u, uint64_t(pos));
    const int c = cl_accept_shaped(q, p, a.V, eq, ep, sq, sp, tok, g, cl);
    if (threadIdx.x == 0 && cl_rank() == 0) {
        a.acc_flag[i * (l + 1) + j] = c == -1;
        a.corr[i * (l + 1) + j] = c;
        if (j == l) a.bonus_tok[i] = tok;
    }
    cl_sync();
}

// regular decoding: pick one token per active sequence (ref:engine.py:151-163)
// and its logprob on the unshaped row; writes proposals[slot][0]
static __global__ void __cluster_dims__(CL_CTAS, 1, 1) __launch_bounds__(CL_THREADS)
    cl_regular_pick_kernel(const float* __restrict__ logits, RegularArgs a) {
    __shared__ ClSmem sm;
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x / CL_CTAS;
    Cl cl(sm, a.V);
    const float* row = logits + (int64_t)i * a.V;
    double* e = a.scratch + (int64_t)i * a.V;
    const ArgMax mx = cl_row_argmax(row, cl);
    double s = 0.0;
    for (int k = cl.c0 + threadIdx.x; k < cl.c1; k += blockDim.x) s += double(expf(row[k] - mx.v));
    const double lse = double(mx.v) + log(cl.sum(block_sum(s, sm.dred)));
    int tok;
    if (a.T == 0.0) {
        tok = mx.i;
    } else {
        cl_shape_row(row, a.V, a.T, a.top_p, e, cl);
        const Shaped sh = sm.sh;
        const int slot = a.slot[i];
        Pcg64 g = pcg64_from_key(a.seed, uint64_t(a.sid[slot]), 1u, uint64_t(a.pos[i]));
        const double u = pcg64_double(g);
        tok = cl_inverse_cdf(a.V, u, [&](int k) { return sh_prob(sh, row, e, k); }, cl);
    }
    if (threadIdx.x == 0 && cl_rank() == 0) {
        a.tok_out[i] = tok;
        a.lp_out[i] = double(row[tok]) - lse;
        a.proposals[a.slot[i] * a.pstride] = tok;
    }
    cl_sync();
}

}  // namespace bass
