// K9: shaping, sampling, accept/resample, bonus, finalize — on device.
//
// Restates ref:sampling.py:69-146 and the per-slot step logic of
// ref:engine.py:243-360 over fp32 logits rows, with probabilities in fp64.
// Shaping keeps the nucleus as "keys above a boundary + ties up to an id",
// found by a 4-pass radix select on the orderable logit key; this equals the
// reference's lexsort((ids, -p)) order because p is monotone in the logit
// and ties in p are ties in the logit.
#pragma once
#include "common.cuh"
#include "rng.cuh"

namespace bass {

constexpr int SM_THREADS = 512;

// thread-local argmax over a row (16-byte loads, 4 in flight), first index on ties
BASS_DEV ArgMax row_argmax_local(const float* __restrict__ row, int V) {
    ArgMax a{-INFINITY, 0x7fffffff};
    if ((V & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int n4 = V >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += blockDim.x) {
            const float4 v = __ldg(r4 + i);
            a = better(a, ArgMax{v.x, 4 * i});
            a = better(a, ArgMax{v.y, 4 * i + 1});
            a = better(a, ArgMax{v.z, 4 * i + 2});
            a = better(a, ArgMax{v.w, 4 * i + 3});
        }
    } else {
        for (int i = threadIdx.x; i < V; i += blockDim.x) a = better(a, ArgMax{row[i], i});
    }
    return a;
}

// thread-local sum of exp(x - m) (fp32 exp, fp64 accumulation)
BASS_DEV double row_sumexp_local(const float* __restrict__ row, int V, float m) {
    double s = 0.0;
    if ((V & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int n4 = V >> 2;
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += blockDim.x) {
            const float4 v = __ldg(r4 + i);
            s += double(expf(v.x - m)) + double(expf(v.y - m)) + double(expf(v.z - m)) + double(expf(v.w - m));
        }
    } else {
        for (int i = threadIdx.x; i < V; i += blockDim.x) s += double(expf(row[i] - m));
    }
    return s;
}

struct Shaped {
    int greedy;      // T == 0: one-hot on argmax
    int argmax;
    double S;        // sum of e_i
    double Kf;       // kept mass in units of e_i / S
    uint32_t ukey;   // boundary key
    int id_lim;      // ties at ukey kept when id <= id_lim
    int keep_all;
};

struct ShapeSmem {
    int cnt[256];
    double mass[256];
    double wmass[SM_THREADS / 32][256];   // per-warp bucket masses (summed in warp order)
    double dred[33];
    float fred[33];
    int ired[33];
    int64_t lred[33];
    Shaped sh;
    int sel, found;
    double before;
};

BASS_DEV bool sh_kept(const Shaped& s, float x, int i) {
    if (s.keep_all) return true;
    const uint32_t k = fkey(x);
    return k > s.ukey || (k == s.ukey && i <= s.id_lim);
}

BASS_DEV double sh_prob(const Shaped& s, const float* row, const double* e, int i) {
    if (s.greedy) return i == s.argmax ? 1.0 : 0.0;
    return sh_kept(s, row[i], i) ? (e[i] / s.S) / s.Kf : 0.0;
}

// Shape one row into `out`.  `e` is a per-row fp64 scratch of length V.
// ref:sampling.py:69-104.  Must be called by all threads of the block.
BASS_DEV void shape_row(const float* __restrict__ row, int V, double T, double top_p,
                        double* __restrict__ e, ShapeSmem& sm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    // argmax / max (first index on ties)
    const ArgMax a = block_argmax(row_argmax_local(row, V), sm.fred, sm.ired);
    if (T == 0.0) {
        if (tid == 0) { sm.sh = Shaped{}; sm.sh.greedy = 1; sm.sh.argmax = a.i; }
        __syncthreads();
        return;
    }
    const double zmax = double(a.v) / T;
    double s = 0.0;
    for (int i = tid; i < V; i += nt) {
        const double ei = exp(double(row[i]) / T - zmax);   // exp(-inf) = 0
        e[i] = ei;
        s += ei;
    }
    const double S = block_sum(s, sm.dred);
    // radix select over the key, descending: find the bucket where the
    // running mass (in descending key order) first reaches top_p.
    uint32_t prefix = 0;
    double before = 0.0;
    int keep_all = 0;
    for (int pass = 0; pass < 4 && !keep_all; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int b = tid; b < 256; b += nt) sm.cnt[b] = 0;
        for (int b = tid; b < (SM_THREADS / 32) * 256; b += nt) (&sm.wmass[0][0])[b] = 0.0;
        __syncthreads();
        // warp-aggregated: lanes hitting the same bucket are summed (lane
        // order) and the group's leader adds it to its warp's private
        // histogram (no fp64 atomics; warps merged in fixed order below, so
        // the masses are deterministic)
        const int lane = tid & 31, wid = tid >> 5;
        for (int i0 = 0; i0 < V; i0 += nt) {   // uniform trip count: whole warps stay converged
            const int i = i0 + tid;
            int b = -1;
            double m = 0.0;
            if (i < V) {
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
            for (int w = 0; w < SM_THREADS / 32; ++w) mb += sm.wmass[w][b];
            sm.mass[b] = mb;
        }
        __syncthreads();
        if (tid == 0) {
            double run = before;
            int sel = -1, last_nonempty = -1;
            for (int b = 255; b >= 0; --b) {
                if (sm.cnt[b] == 0) continue;
                last_nonempty = b;
                if (run + sm.mass[b] >= top_p) { sel = b; break; }
                run += sm.mass[b];
            }
            if (sel < 0) {
                // never reaches top_p: at pass 0 keep everything
                // (searchsorted clamps to n-1); deeper, take the last bucket
                if (pass == 0) { sm.found = 0; }
                else { sel = last_nonempty; double r2 = before;
                       for (int b = 255; b > sel; --b) r2 += sm.mass[b]; run = r2; sm.found = 1; }
            } else {
                sm.found = 1;
            }
            sm.sel = sel;
            sm.before = run;
        }
        __syncthreads();
        if (!sm.found) { keep_all = 1; break; }
        prefix = (prefix << 8) | uint32_t(sm.sel);
        before = sm.before;
        __syncthreads();
    }
    int id_lim = 0x7fffffff;
    if (!keep_all) {
        // ties at the boundary key: same logit -> same probability f
        const int g = sm.cnt[sm.sel];
        const uint32_t ukey = prefix;
        // f of a member (all equal); find one member's e
        __syncthreads();
        if (tid == 0) sm.found = -1;
        __syncthreads();
        for (int i = tid; i < V; i += nt)
            if (fkey(row[i]) == ukey) atomicMax(&sm.found, i);   // any member index
        __syncthreads();
        const double f = e[sm.found] / S;
        if (tid == 0) {
            double run = before;
            int n = 0;
            while (n < g) { run += f; ++n; if (run >= top_p) break; }
            sm.sel = n;          // members (by id) kept
        }
        __syncthreads();
        const int need = sm.sel;
        if (need < g) {
            // id of the need-th member in ascending id order
            const int chunk = (V + nt - 1) / nt, lo = tid * chunk, hi = min(V, lo + chunk);
            int c = 0;
            for (int i = lo; i < hi; ++i) c += fkey(row[i]) == ukey;
            int tot;
            int pre = block_exclusive_scan(c, sm.ired, &tot);
            __syncthreads();
            if (pre < need && pre + c >= need) {
                int cc = pre;
                for (int i = lo; i < hi; ++i)
                    if (fkey(row[i]) == ukey && ++cc == need) { sm.found = i; break; }
            }
            __syncthreads();
            id_lim = sm.found;
        }
        if (tid == 0) { sm.sh.ukey = ukey; }
    }
    __syncthreads();
    Shaped sh{};
    sh.greedy = 0;
    sh.argmax = a.i;
    sh.S = S;
    sh.keep_all = keep_all;
    sh.ukey = keep_all ? 0u : prefix;
    sh.id_lim = id_lim;
    double kf = 0.0;
    for (int i = tid; i < V; i += nt)
        if (sh_kept(sh, row[i], i)) kf += e[i] / S;
    sh.Kf = block_sum(kf, sm.dred);
    if (tid == 0) sm.sh = sh;
    __syncthreads();
}

// First index whose running sum (id order) of w(i) exceeds u * total;
// clamped to V-1 (ref:sampling.py:112-115).  `w` is a callable.
template <typename W>
BASS_DEV int inverse_cdf_block(int V, double u, W w, ShapeSmem& sm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int chunk = (V + nt - 1) / nt, lo = tid * chunk, hi = min(V, lo + chunk);
    double loc = 0.0;
    for (int i = lo; i < hi; ++i) loc += w(i);
    double total;
    const double pre = block_exclusive_scan(loc, sm.dred, &total);
    const double target = u * total;
    // the chosen element always has positive weight (csum[i-1] <= target <
    // csum[i]); every thread proposes its first crossing, the block keeps the
    // smallest, which is robust to the scan's rounding at range borders
    int cand = 0x7fffffff;
    double c = pre;
    for (int i = lo; i < hi; ++i) {
        const double wi = w(i);
        c += wi;
        if (c > target && wi > 0.0) { cand = i; break; }
    }
    // block min of candidates
    ArgMax am{-float(cand), cand};
    am = block_argmax(am, sm.fred, sm.ired);
    const int idx = am.i;
    return idx == 0x7fffffff ? V - 1 : min(idx, V - 1);
}

// ---------------------------------------------------------------- kernels

// per logits row: argmax (first index) and log-sum-exp (fp64 accumulate)
static __global__ void __launch_bounds__(SM_THREADS) row_stats_kernel(const float* __restrict__ logits,
                                                               int V, int32_t* __restrict__ amax,
                                                               double* __restrict__ lse) {
    pdl_trigger();
    pdl_wait();
    __shared__ float fv[33];
    __shared__ int iv[33];
    __shared__ double dv[33];
    const float* row = logits + (int64_t)blockIdx.x * V;
    ArgMax a = block_argmax(row_argmax_local(row, V), fv, iv);
    const double s = block_sum(row_sumexp_local(row, V, a.v), dv);
    if (threadIdx.x == 0) {
        amax[blockIdx.x] = a.i;
        lse[blockIdx.x] = double(a.v) + log(s);      // scipy.special.logsumexp
    }
}

struct DraftPick {               // per active sequence of a draft step
    const int32_t* slot;         // [nA]
    const int64_t* sid;          // sequence ids (by slot)
    const int32_t* pos;          // absolute position of the proposal (by seq)
    int32_t* proposals;          // [slot][pstride]
    int pstride, j;
    // harness override (align < 0: off)
    double align;
    uint64_t align_seed;
    const int32_t* align_tok;    // [slot][max_new]
    const int32_t* prompt_len;   // by slot
    int max_new;
};

BASS_DEV int aligned_override(const DraftPick& d, int slot, int pos, int V, int tok) {
    if (d.align < 0.0) return tok;
    const uint64_t h = splitmix64(d.align_seed ^ splitmix64(uint64_t(d.sid[slot]) * 0x100000001B3ull +
                                                            uint64_t(pos)));
    const double u = double(h >> 11) * (1.0 / 9007199254740992.0);
    const int gi = pos - d.prompt_len[slot];
    if (u < d.align && gi >= 0 && gi < d.max_new) return d.align_tok[slot * d.max_new + gi];
    return int(splitmix64(h) % uint64_t(V));
}

// greedy draft step: proposal = argmax of the sequence's last draft row
static __global__ void __launch_bounds__(SM_THREADS) draft_greedy_kernel(const float* __restrict__ logits,
                                                                  int V, DraftPick d) {
    pdl_trigger();
    pdl_wait();
    __shared__ float fv[33];
    __shared__ int iv[33];
    const int i = blockIdx.x;
    const float* row = logits + (int64_t)i * V;
    const ArgMax a = block_argmax(row_argmax_local(row, V), fv, iv);
    if (threadIdx.x == 0) {
        const int slot = d.slot[i];
        d.proposals[slot * d.pstride + d.j] = aligned_override(d, slot, d.pos[i], V, a.i);
    }
}

// Greedy draft step over P CTAs per row: CTA (i, p) takes the argmax of
// columns [p V/P, (p+1) V/P), parks it, and the row's last-arriving CTA
// combines the P partials (max value, then first index — order-free, so the
// result equals draft_greedy_kernel's bit for bit) and writes the proposal.
// `cnt` [rows] must be zero; the last CTA re-arms it.
constexpr int GREEDY_PARTS = 16;
static __global__ void __launch_bounds__(256) draft_greedy_split_kernel(const float* __restrict__ logits, int V,
                                                                        DraftPick d, float* __restrict__ pv,
                                                                        int* __restrict__ pi, int* __restrict__ cnt) {
    pdl_trigger();
    pdl_wait();
    __shared__ float fv[33];
    __shared__ int iv[33];
    __shared__ bool last;
    const int i = blockIdx.x, part = blockIdx.y, P = gridDim.y;
    const float* row = logits + (int64_t)i * V;
    // 4-aligned column range so the float4 path stays aligned
    const int n4 = V >> 2;
    const int c0 = (int)((int64_t)part * n4 / P) * 4;
    const int c1 = part == P - 1 ? V : (int)((int64_t)(part + 1) * n4 / P) * 4;
    ArgMax a{-INFINITY, 0x7fffffff};
    if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int e4 = c1 >> 2;
#pragma unroll 4
        for (int k = (c0 >> 2) + threadIdx.x; k < e4; k += blockDim.x) {
            const float4 v = __ldcg(r4 + k);
            a = better(a, ArgMax{v.x, 4 * k});
            a = better(a, ArgMax{v.y, 4 * k + 1});
            a = better(a, ArgMax{v.z, 4 * k + 2});
            a = better(a, ArgMax{v.w, 4 * k + 3});
        }
        for (int k = (e4 << 2) + threadIdx.x; k < c1; k += blockDim.x) a = better(a, ArgMax{row[k], k});
    } else {
        for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x) a = better(a, ArgMax{row[k], k});
    }
    a = block_argmax(a, fv, iv);
    if (threadIdx.x == 0) {
        pv[i * P + part] = a.v;
        pi[i * P + part] = a.i;
        __threadfence();
        last = atomicAdd(&cnt[i], 1) == P - 1;
    }
    __syncthreads();
    if (!last) return;
    if (threadIdx.x == 0) {
        __threadfence();
        ArgMax r{-INFINITY, 0x7fffffff};
        for (int q = 0; q < P; ++q) r = better(r, ArgMax{__ldcg(pv + i * P + q), __ldcg(pi + i * P + q)});
        cnt[i] = 0;
        const int slot = d.slot[i];
        d.proposals[slot * d.pstride + d.j] = aligned_override(d, slot, d.pos[i], V, r.i);
    }
}

// sampled draft step: proposal ~ shape(row), uniform = RNG(seed, sid, DRAFT, pos)
static __global__ void __launch_bounds__(SM_THREADS) draft_sample_kernel(const float* __restrict__ logits,
                                                                  int V, double T, double top_p,
                                                                  uint64_t seed, double* scratch,
                                                                  DraftPick d) {
    __shared__ ShapeSmem sm;
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x;
    const float* row = logits + (int64_t)i * V;
    double* e = scratch + (int64_t)blockIdx.x * V;
    shape_row(row, V, T, top_p, e, sm);
    const int slot = d.slot[i], pos = d.pos[i];
    Pcg64 g = pcg64_from_key(seed, uint64_t(d.sid[slot]), 0u, uint64_t(pos));
    const double u = pcg64_double(g);
    const Shaped sh = sm.sh;
    const int tok = inverse_cdf_block(V, u, [&](int k) { return sh_prob(sh, row, e, k); }, sm);
    if (threadIdx.x == 0) d.proposals[slot * d.pstride + d.j] = aligned_override(d, slot, pos, V, tok);
}

// standalone shaping + sampling (bass_shape_sample)
static __global__ void __launch_bounds__(SM_THREADS) shape_sample_kernel(const float* __restrict__ logits,
                                                                  int V, double T, double top_p,
                                                                  const double* __restrict__ u,
                                                                  double* scratch,
                                                                  int32_t* __restrict__ tok,
                                                                  double* __restrict__ probs) {
    __shared__ ShapeSmem sm;
    const float* row = logits + (int64_t)blockIdx.x * V;
    double* e = scratch + (int64_t)blockIdx.x * V;
    shape_row(row, V, T, top_p, e, sm);
    const Shaped sh = sm.sh;
    if (probs)
        for (int k = threadIdx.x; k < V; k += blockDim.x)
            probs[(int64_t)blockIdx.x * V + k] = sh_prob(sh, row, e, k);
    const int t = inverse_cdf_block(V, u[blockIdx.x], [&](int k) { return sh_prob(sh, row, e, k); }, sm);
    if (threadIdx.x == 0) tok[blockIdx.x] = t;
}

// accept / resample given both rows' shaping (see accept_block)
BASS_DEV int accept_shaped(const float* qrow, const float* prow, int V, const double* eq, const double* ep,
                           const Shaped& sq, const Shaped& sp, int tok, Pcg64& g, ShapeSmem& sm);

// accept / resample for one (q row, p row, token, VERIFY generator);
// returns corrected token or -1 when accepted; -2 on zero draft probability.
BASS_DEV int accept_block(const float* qrow, const float* prow, int V, double T, double top_p,
                          double* eq, double* ep, int tok, Pcg64& g, ShapeSmem& sm) {
    shape_row(qrow, V, T, top_p, eq, sm);
    const Shaped sq = sm.sh;
    __syncthreads();
    shape_row(prow, V, T, top_p, ep, sm);
    const Shaped sp = sm.sh;
    return accept_shaped(qrow, prow, V, eq, ep, sq, sp, tok, g, sm);
}

BASS_DEV int accept_shaped(const float* qrow, const float* prow, int V, const double* eq, const double* ep,
                           const Shaped& sq, const Shaped& sp, int tok, Pcg64& g, ShapeSmem& sm) {
    const double px = sh_prob(sp, prow, ep, tok);
    const double qx = sh_prob(sq, qrow, eq, tok);
    if (px <= 0.0) return -2;
    const double u = pcg64_double(g);
    if (u * px < qx) return -1;
    // residual normalize(max(q - p, 0)), sampled with the second draw
    auto r = [&](int k) {
        const double d = sh_prob(sq, qrow, eq, k) - sh_prob(sp, prow, ep, k);
        return d > 0.0 ? d : 0.0;
    };
    double loc = 0.0;
    for (int k = threadIdx.x; k < V; k += blockDim.x) loc += r(k);
    const double R = block_sum(loc, sm.dred);
    if (R <= 0.0) return -3;
    const double u2 = pcg64_double(g);
    return inverse_cdf_block(V, u2, [&](int k) { return r(k) / R; }, sm);
}

static __global__ void __launch_bounds__(SM_THREADS) accept_pairs_kernel(
    const float* __restrict__ ql, const float* __restrict__ pl, int V, double T, double top_p,
    const int32_t* __restrict__ tok, uint64_t seed, const int64_t* __restrict__ sid,
    const int64_t* __restrict__ ctr, double* scratch, int32_t* __restrict__ acc,
    int32_t* __restrict__ corr) {
    __shared__ ShapeSmem sm;
    const int i = blockIdx.x;
    Pcg64 g = pcg64_from_key(seed, uint64_t(sid[i]), 1u, uint64_t(ctr[i]));
    const int c = accept_block(ql + (int64_t)i * V, pl + (int64_t)i * V, V, T, top_p,
                               scratch + (int64_t)i * 2 * V, scratch + (int64_t)i * 2 * V + V, tok[i],
                               g, sm);
    if (threadIdx.x == 0) {
        acc[i] = c == -1;
        corr[i] = c;
    }
}

static __global__ void rng_kernel(int n, uint64_t seed, const int64_t* sid, const int32_t* role,
                           const int64_t* ctr, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Pcg64 g = pcg64_from_key(seed, uint64_t(sid[i]), uint32_t(role[i]), uint64_t(ctr[i]));
    out[2 * i] = pcg64_double(g);
    out[2 * i + 1] = pcg64_double(g);
}

// ------------------------------------------------------ engine step logic

// device -> host, one record per active sequence: a SlotStep header, then
// `estride` emitted token ids (int32, padded to 8 bytes), then `estride`
// logprobs (double); estride = draft limit + 1 (the most a step can emit)
struct SlotStep {
    int32_t accepted, n_emit, reason, err;   // reason: -1 running, 0 eos, 1 length
};
__host__ __device__ inline size_t slot_rec_bytes(int estride) {
    return sizeof(SlotStep) + (((size_t)estride * 4 + 7) & ~(size_t)7) + (size_t)estride * 8;
}
__host__ __device__ inline int32_t* slot_rec_tok(void* rec) { return reinterpret_cast<int32_t*>((char*)rec + sizeof(SlotStep)); }
__host__ __device__ inline double* slot_rec_lp(void* rec, int estride) {
    return reinterpret_cast<double*>((char*)rec + sizeof(SlotStep) + (((size_t)estride * 4 + 7) & ~(size_t)7));
}

struct StepArgs {
    int nA, l, V;
    const int32_t* slot;          // [nA]
    const int32_t* committed;     // [nA] committed length C at step start
    const int32_t* generated;     // [nA] generated count at step start
    const int32_t* proposals;     // [slot][pstride]
    int pstride;
    const float* vlog;            // verify logits [nA*(l+1), V]
    const int32_t* vamax;         // argmax per verify row
    const double* vlse;           // lse per verify row
    int max_new, eos;
    // sampled
    const int32_t* acc_flag;      // [nA*(l+1)]
    const int32_t* corr;          // [nA*(l+1)]
    const int32_t* bonus_tok;     // [nA]
    int greedy;
    char* out;                    // [nA] records of slot_rec_bytes(estride)
    int estride;
};

// accepted prefix + correction / bonus + EOS/length finalize + logprobs
// (ref:engine.py:276-349, _finalize_emitted :103-117, logprob :99-100)
static __global__ void finalize_kernel(StepArgs a) {
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.nA) return;
    const int slot = a.slot[i], l = a.l, rb = i * (l + 1);
    char* rec = a.out + (size_t)i * slot_rec_bytes(a.estride);
    int32_t* em = slot_rec_tok(rec);   // emitted tokens, built in place (<= l + 1)
    int x = 0, n = 0, err = 0;
    for (int j = 0; j < l; ++j) {
        const int t = a.proposals[slot * a.pstride + j];
        if (a.greedy) {
            const int am = a.vamax[rb + j];
            if (t == am) { em[n++] = t; ++x; }
            else { em[n++] = am; break; }
        } else {
            if (a.acc_flag[rb + j]) { em[n++] = t; ++x; }
            else {
                const int c = a.corr[rb + j];
                if (c < 0) err = c;
                em[n++] = c < 0 ? 0 : c;
                break;
            }
        }
    }
    const int remaining = a.max_new - a.generated[i];
    if (x == l) {
        bool eos_hit = false;
        for (int j = 0; j < n; ++j) eos_hit |= (a.eos >= 0 && em[j] == a.eos);
        if (!eos_hit && remaining > l) {
            int b;
            if (a.greedy) b = a.vamax[rb + l];
            else {
                const int c = a.corr[rb + l];
                b = a.acc_flag[rb + l] ? a.bonus_tok[i] : c;
                if (!a.acc_flag[rb + l] && c < 0) { err = c; b = 0; }
            }
            em[n++] = b;
        }
    }
    int reason = -1;
    if (a.eos >= 0) {
        for (int j = 0; j < n; ++j)
            if (em[j] == a.eos) { n = j + 1; reason = 0; break; }
    }
    if (n > remaining) { n = remaining; reason = 1; }
    else if (n == remaining && reason < 0) reason = 1;
    SlotStep& o = *reinterpret_cast<SlotStep*>(rec);
    o.accepted = x;
    o.n_emit = n;
    o.reason = reason;
    o.err = err;
    double* lp = slot_rec_lp(rec, a.estride);
    for (int j = 0; j < n; ++j) lp[j] = double(a.vlog[(int64_t)(rb + j) * a.V + em[j]]) - a.vlse[rb + j];
}

// sampled verify: one CTA per (sequence, position j <= l).  j < l tests the
// proposal against (q_j, p_j); j == l draws the bonus token from the bonus
// draft row and tests it (ref:engine.py:292-343).
struct VerifyArgs {
    int nA, l, V;
    double T, top_p;
    uint64_t seed;
    const int32_t* slot;
    const int64_t* sid;           // by slot
    const int32_t* committed;     // [nA]
    const int32_t* proposals;
    int pstride;
    const float* vlog;            // [nA*(l+1), V]
    const float* dlog;            // draft rows: row (j, i) at dlog + (j*nA + i)*V, j <= l
    double* scratch;              // [nA*(l+1), 2, V]
    int32_t* acc_flag;
    int32_t* corr;
    int32_t* bonus_tok;
};

static __global__ void __launch_bounds__(SM_THREADS) verify_sampled_kernel(VerifyArgs a) {
    __shared__ ShapeSmem sm;
    pdl_trigger();
    pdl_wait();
    const int j = blockIdx.x, i = blockIdx.y, l = a.l;
    const int slot = a.slot[i], pos = a.committed[i] + j;
    const int64_t sid = a.sid[slot];
    const float* q = a.vlog + (int64_t)(i * (l + 1) + j) * a.V;
    const float* p = a.dlog + (int64_t)(j * a.nA + i) * a.V;
    double* eq = a.scratch + (int64_t)(i * (l + 1) + j) * 2 * a.V;
    double* ep = eq + a.V;
    int tok;
    if (j < l) {
        tok = a.proposals[slot * a.pstride + j];
    } else {
        shape_row(p, a.V, a.T, a.top_p, ep, sm);
        const Shaped sp = sm.sh;
        Pcg64 gd = pcg64_from_key(a.seed, uint64_t(sid), 0u, uint64_t(pos));
        const double ub = pcg64_double(gd);
        tok = inverse_cdf_block(a.V, ub, [&](int k) { return sh_prob(sp, p, ep, k); }, sm);
        __syncthreads();
    }
    Pcg64 g = pcg64_from_key(a.seed, uint64_t(sid), 1u, uint64_t(pos));
    const int c = accept_block(q, p, a.V, a.T, a.top_p, eq, ep, tok, g, sm);
    if (threadIdx.x == 0) {
        a.acc_flag[i * (l + 1) + j] = c == -1;
        a.corr[i * (l + 1) + j] = c;
        if (j == l) a.bonus_tok[i] = tok;
    }
}

// Verify, split in two launches so the 2 (l+1) nA row shapings run on as
// many CTAs: (1) shape every main row q (z = 0) and draft row p (z = 1),
// keeping e in the scratch and the Shaped summary in `sh`; (2) per (j, i):
// bonus draw (j = l) and accept / resample — the same arithmetic, RNG
// streams and draws as verify_sampled_kernel.
static __global__ void __launch_bounds__(SM_THREADS) verify_shape_kernel(VerifyArgs a, Shaped* __restrict__ sh) {
    __shared__ ShapeSmem sm;
    pdl_trigger();
    pdl_wait();
    const int j = blockIdx.x, i = blockIdx.y, z = blockIdx.z, l = a.l;
    const int64_t r = (int64_t)i * (l + 1) + j;
    const float* row = z == 0 ? a.vlog + r * a.V : a.dlog + (int64_t)(j * a.nA + i) * a.V;
    double* e = a.scratch + r * 2 * a.V + (z == 0 ? 0 : a.V);
    shape_row(row, a.V, a.T, a.top_p, e, sm);
    if (threadIdx.x == 0) sh[r * 2 + z] = sm.sh;
}

static __global__ void __launch_bounds__(SM_THREADS) verify_accept_kernel(VerifyArgs a,
                                                                          const Shaped* __restrict__ sh) {
    __shared__ ShapeSmem sm;
    pdl_trigger();
    pdl_wait();
    const int j = blockIdx.x, i = blockIdx.y, l = a.l;
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
        tok = inverse_cdf_block(a.V, ub, [&](int k) { return sh_prob(sp, p, ep, k); }, sm);
        __syncthreads();
    }
    Pcg64 g = pcg64_from_key(a.seed, uint64_t(sid), 1u, uint64_t(pos));
    const int c = accept_shaped(q, p, a.V, eq, ep, sq, sp, tok, g, sm);
    if (threadIdx.x == 0) {
        a.acc_flag[i * (l + 1) + j] = c == -1;
        a.corr[i * (l + 1) + j] = c;
        if (j == l) a.bonus_tok[i] = tok;
    }
}

// regular decoding: pick one token per active sequence from its current
// logits row (ref:engine.py:151-163); writes proposals[slot][0] for the next
// forward's token indirection.
struct RegularArgs {
    const int32_t* slot;
    const int64_t* sid;           // by slot
    const int32_t* pos;           // [nA] absolute position of the new token
    int32_t* proposals;
    int pstride;
    int V;
    double T, top_p;
    uint64_t seed;
    double* scratch;
    int32_t* tok_out;
    double* lp_out;
};

static __global__ void __launch_bounds__(SM_THREADS) regular_pick_kernel(const float* __restrict__ logits,
                                                                  RegularArgs a) {
    __shared__ ShapeSmem sm;
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x;
    const float* row = logits + (int64_t)i * a.V;
    double* e = a.scratch + (int64_t)i * a.V;
    // lse of the raw row (logprob uses unshaped logits, ref:engine.py:162)
    const ArgMax mx = block_argmax(row_argmax_local(row, a.V), sm.fred, sm.ired);
    const double s = block_sum(row_sumexp_local(row, a.V, mx.v), sm.dred);
    const double lse = double(mx.v) + log(s);
    int tok;
    if (a.T == 0.0) {
        tok = mx.i;
    } else {
        shape_row(row, a.V, a.T, a.top_p, e, sm);
        const Shaped sh = sm.sh;
        const int slot = a.slot[i];
        Pcg64 g = pcg64_from_key(a.seed, uint64_t(a.sid[slot]), 1u, uint64_t(a.pos[i]));
        const double u = pcg64_double(g);
        tok = inverse_cdf_block(a.V, u, [&](int k) { return sh_prob(sh, row, e, k); }, sm);
    }
    if (threadIdx.x == 0) {
        a.tok_out[i] = tok;
        a.lp_out[i] = double(row[tok]) - lse;
        a.proposals[a.slot[i] * a.pstride] = tok;
    }
}

}  // namespace bass
