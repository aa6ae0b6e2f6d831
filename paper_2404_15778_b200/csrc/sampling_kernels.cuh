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

BASS_DEV bool sh_kept(const Shaped& s, float x, int i) {
    if (s.keep_all) return true;
    const uint32_t k = fkey(x);
    return k > s.ukey || (k == s.ukey && i <= s.id_lim);
}

BASS_DEV double sh_prob(const Shaped& s, const float* row, const double* e, int i) {
    if (s.greedy) return i == s.argmax ? 1.0 : 0.0;
    return sh_kept(s, row[i], i) ? (e[i] / s.S) / s.Kf : 0.0;
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

// Greedy draft step over P CTAs per row: CTA (i, p) takes the argmax of
// columns [p V/P, (p+1) V/P), parks it, and the row's last-arriving CTA
// combines the P partials (max value, then first index — order-free, so the
// result equals a single scan's bit for bit) and writes the proposal.
// `cnt` [rows] must be zero; the last CTA re-arms it.  P = 8 (64 CTAs for
// b = 8; 16 / 32 / 4 / 2 measured equal or slower in the C2 chain,
// profiles/r2/greedy_parts_ab.txt).
constexpr int GREEDY_PARTS = 8;
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
    // device loop: 0 = every row of the step at once; 1 = everything except
    // the bonus draft row (j = l), which 2 handles after its conditional draft
    // forward (ref:engine.py:305-322 runs that forward only when a sequence
    // accepted its whole draft)
    int phase;
};

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

}  // namespace bass
