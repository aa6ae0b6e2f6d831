// Device-resident decode loop (north_star (4); ref:engine.py:237-362,
// draft_control.py:49-69): the per-step planning, bookkeeping and Algorithm 1
// run on the GPU, and one CUDA graph drives every step after the first:
//
//   init ──> WHILE(any sequence active) { SWITCH(l_draft) { step(l) } }
//
// step(l) is one PDL chain captured once per draft length: plan kernel (this
// step's token / position / attention work-list metadata from the device
// state) -> l draft forwards + picks -> verify forward -> row statistics ->
// [sampled shaping, accept / resample] -> finalize -> book kernel (commit the
// emitted tokens, roll the cache lengths back, Algorithm 1, the step trace).
// A select node before the SWITCH and a continue node after it set the two
// graph conditions from the booked state.  The prompt step (ragged prompt
// blocks) is planned on the host and enqueued ahead of the graph; its
// outcome is booked by the same kernel on the device.  The host synchronises
// once per generation.
//
// Fixed shapes per branch: every slot of the batch runs every step (a finished
// sequence's rows are computed and ignored — rows are independent, so the
// active rows' bits do not change), the first draft forward of a step feeds the
// last two committed tokens (the older one rewrites identical K/V), and the
// verify block is the last committed token + l proposals.
#pragma once

#include "sampling_kernels.cuh"

namespace bass {

constexpr int GL_MAXL = 48;           // draft limits above this run the per-step host loop
constexpr int GL_MAXF = GL_MAXL + 2;  // forwards per step: l (+1 sampled bonus) draft + verify

struct DevLoop {                      // device-resident generation state
    int b, l, s, step, err, lmin, active;
    int fixed, incre, mod, limit;
    int maxnew, estride, com_cap, greedy, eos, steps_cap;
    unsigned long long t0;
    long long main_calls, draft_calls;
    int32_t *com;                     // [b][com_cap] committed tokens (prompt + generated)
    int32_t *C, *ngen, *done, *kvm, *kvd;   // [b]
    int32_t *tokens;                  // [b][maxnew]
    double *lps;                      // [b][maxnew]
    int32_t *reason, *cstep;          // [b]
    unsigned long long *tfin;         // [b] globaltimer at completion
    unsigned long long *tstep;        // [steps_cap] globaltimer at the end of each step
    int32_t *tr_l, *tr_acc, *tr_emit, *tr_kv;   // [steps_cap], [steps_cap][b] x 3
    int32_t *tr_bonus;                // [steps_cap] the sampled bonus draft forward ran
    int bonus;                        // ... in the current step
    const char* rec;                  // finalize records of the step ([b] x slot_rec_bytes(estride))
};

// one forward of a step: kind 0 = first draft forward (2 rows / sequence from
// position C - 2), 1 = draft forward j (1 row: proposal j - 1 at C + j - 1),
// 2 = verify (l + 1 rows from C - 1); meta / work: arena offsets (int32)
struct PlanFwd {
    int kind, j, q, meta, work, stride, nq, live;   // live: arena offset of {m_act, r_act}
};
struct PlanArgs {
    int b, l, nf, strategy, ch, split_ch;
    int perm, cperm, gperm;           // arena offsets: slot of sequence index i (active slots first),
                                      // its committed length and generated count
    int pos[GL_MAXL + 1];             // arena offsets of the proposal positions (C + j) per draft j
    PlanFwd f[GL_MAXF];
};

// The step's metadata, mirroring forward_premeta / stream_attention_work
// (runtime.cu, attn_stream.cu) on the host.  No early PDL trigger: every later
// kernel of the step starts after this one completed, so the attention's
// pre-wait loads of its work list see it.
__global__ void __launch_bounds__(1024) loop_plan_kernel(const DevLoop* __restrict__ S, int32_t* __restrict__ ar,
                                                         PlanArgs a) {
    __shared__ int cmax, n_act;
    __shared__ int16_t order[1024];
    const int t = threadIdx.x, b = a.b;
    // sequence order of the step: the active slots first (ascending), then the
    // finished ones, so every forward's live rows are a prefix (GEMM token
    // groups past it exit, the LM head stops there)
    if (t == 0) {
        int k = 0;
        for (int s = 0; s < b; ++s)
            if (!S->done[s]) order[k++] = (int16_t)s;
        n_act = k;
        for (int s = 0; s < b; ++s)
            if (S->done[s]) order[k++] = (int16_t)s;
        cmax = 0;
    }
    __syncthreads();
    const int i = t;                                   // sequence index
    const int slot = i < b ? order[i] : 0;
    const int C = i < b ? S->C[slot] : 0;
    const bool fin = i >= n_act;
    if (i < b && !fin) atomicMax(&cmax, C);   // PAD pads to the longest ACTIVE history
    __syncthreads();
    if (i >= b) return;
    ar[a.perm + i] = slot;
    ar[a.cperm + i] = C;
    ar[a.gperm + i] = S->ngen[slot];
    const int32_t* com = S->com + (size_t)slot * S->com_cap;
    for (int f = 0; f < a.nf; ++f) {
        const PlanFwd F = a.f[f];
        const int q = F.q, M = b * q, n = b;
        const int off = F.kind == 0 ? C - 2 : F.kind == 1 ? C + F.j - 1 : C - 1;
        const int safe = F.kind == 2 ? C - 1 : C - 2;   // rows written before the step began
        int32_t* mt = ar + F.meta;
        for (int t = 0; t < q; ++t) {
            const int r = i * q + t;
            mt[r] = F.kind == 0 ? com[C - 2 + t] : F.kind == 1 ? -F.j : (t == 0 ? com[C - 1] : -t);
            mt[M + r] = slot;
            mt[2 * M + r] = off + t;
        }
        if (i == 0) {
            ar[F.live] = n_act * q;                        // live rows of the forward
            ar[F.live + 1] = F.kind == 2 ? n_act * q : n_act;   // live logit rows
        }
        mt[3 * M + i] = slot;
        mt[3 * M + n + i] = i * q;
        mt[3 * M + 2 * n + i] = q;
        mt[3 * M + 3 * n + i] = off;
        int32_t* lr = mt + 3 * M + 4 * n;
        if (F.kind == 2)
            for (int t = 0; t < q; ++t) lr[i * q + t] = i * q + t;
        else
            lr[i] = i * q + q - 1;
        // attention work items of this sequence (ref:attention.py:96-137; PAD
        // streams every sequence up to the batch's longest history)
        const int pad_last = (F.kind == 0 ? cmax : F.kind == 1 ? cmax + F.j : cmax + a.l) - 1;
        int32_t* w = ar + F.work + (size_t)i * F.stride * 8;
        // a finished sequence's rows are computed and discarded: its attention
        // only sees its first keys (finite values, no history streamed)
        const int aoff = fin ? 0 : off;
        int k = 0;
        // split-major, query tile minor (as stream_items: the tiles of one
        // split share their K/V rows through L2)
        const int last_row = (a.strategy == BASS_PAD && !fin) ? pad_last : aoff + q - 1;
        for (int s = 0; s * a.split_ch < last_row / a.ch + 1; ++s) {
            for (int t0 = 0; t0 < q && k < F.stride; t0 += F.nq) {
                const int last = (a.strategy == BASS_PAD && !fin) ? pad_last : aoff + min(q, t0 + F.nq) - 1;
                const int nch = last / a.ch + 1;
                if (s * a.split_ch >= nch) continue;
                int32_t* it = w + k * 8;
                it[0] = slot; it[1] = i * q; it[2] = q; it[3] = aoff;
                it[4] = t0; it[5] = s; it[6] = min(a.split_ch, nch - s * a.split_ch); it[7] = min(aoff, safe);
                ++k;
            }
        }
        for (; k < F.stride; ++k) {   // idle padding (skipped by the attention's item loop)
            int32_t* it = w + k * 8;
            it[0] = slot; it[1] = i * q; it[2] = q; it[3] = off; it[4] = q; it[5] = 0; it[6] = 0; it[7] = 0;
        }
    }
    for (int j = 0; j <= a.l; ++j) ar[a.pos[j] + i] = C + j;
}

// Bookkeeping of one step from the finalize records (ref:engine.py:344-362):
// emitted tokens / logprobs appended, EOS / length completion, cache lengths
// rolled back to the committed prefix, forward-call counters, the step trace,
// Algorithm 1 over the accepted counts of the slots active at the step start
// (ref:draft_control.py:49-69), and the graph conditions for the next step.
// perm: the slot of each finalize record (the step's sequence order; the
// prompt step's records are in slot order).
__global__ void __launch_bounds__(1024) loop_book_kernel(DevLoop* __restrict__ S, const int32_t* __restrict__ perm) {
    __shared__ int mx, any_active, any_err, n_act;
    __shared__ long long dcalls;
    pdl_wait();
    const int q = threadIdx.x, b = S->b, l = S->l, step = S->step;
    const int i = q < b ? perm[q] : q;   // this thread's slot
    if (i == 0) {
        mx = 0;
        any_active = 0;
        any_err = 0;
        n_act = 0;
        dcalls = 0;
    }
    __syncthreads();
    const unsigned long long now = gtimer();
    const bool tr = step < S->steps_cap;
    if (i < b && !S->done[i]) {
        const char* rec = S->rec + (size_t)q * slot_rec_bytes(S->estride);
        const SlotStep& o = *reinterpret_cast<const SlotStep*>(rec);
        const int32_t* tok = slot_rec_tok(const_cast<char*>(rec));
        const double* lp = slot_rec_lp(const_cast<char*>(rec), S->estride);
        if (o.err) atomicMin(&any_err, o.err);
        atomicMax(&mx, o.accepted);
        atomicAdd(&n_act, 1);
        const int C = S->C[i], g = S->ngen[i], n = o.n_emit;
        // the bonus draft forward counts per eligible slot (sampled, all accepted)
        if (!S->greedy && o.accepted == l && n >= 1) {
            bool eos_core = false;
            for (int j = 0; j < min(n, l); ++j) eos_core |= (S->eos >= 0 && tok[j] == S->eos);
            if (!eos_core && S->maxnew - g > l) atomicAdd((unsigned long long*)&dcalls, 1ull);
        }
        for (int j = 0; j < n; ++j) {
            S->tokens[(size_t)i * S->maxnew + g + j] = tok[j];
            S->lps[(size_t)i * S->maxnew + g + j] = lp[j];
            S->com[(size_t)i * S->com_cap + C + j] = tok[j];
        }
        const int C2 = C + n;
        S->C[i] = C2;
        S->ngen[i] = g + n;
        // the step appended l + 1 verify rows from C - 1 and nd draft rows from
        // C (as the host loop counts them); roll both back to C2 - 1 (ref:engine.py:358-360)
        const int nd = l + (S->greedy ? 0 : 1);
        S->kvm[i] = min(C + l, C2 - 1);
        S->kvd[i] = min(C + nd - 1, C2 - 1);
        if (o.reason >= 0) {
            S->done[i] = 1;
            S->reason[i] = o.reason;
            S->cstep[i] = step + 1;
            S->tfin[i] = now;
        } else {
            atomicOr(&any_active, 1);
        }
        if (tr) {
            S->tr_acc[(size_t)step * b + i] = o.accepted;
            S->tr_emit[(size_t)step * b + i] = n;
        }
    } else if (i < b && tr) {
        S->tr_acc[(size_t)step * b + i] = -1;
        S->tr_emit[(size_t)step * b + i] = -1;
    }
    __syncthreads();
    if (i < b && tr) S->tr_kv[(size_t)step * b + i] = S->C[i];
    if (q != 0) return;
    S->main_calls += n_act;
    S->draft_calls += (long long)n_act * l + dcalls;
    if (tr) {
        S->tr_l[step] = l;
        S->tstep[step] = now;
        S->tr_bonus[step] = S->bonus;
    }
    S->bonus = 0;
    int ln = l, sn = S->s;
    if (!S->fixed && n_act > 0) {   // Algorithm 1
        if (mx == l) {
            ln = min(l + S->incre, S->limit);
            sn = 0;
        } else {
            const int shrink = l - (l + S->mod - 1) / S->mod - S->s;
            ln = max(max(1, mx), shrink);
            sn = 1;
        }
    }
    S->l = ln;
    S->s = sn;
    S->step = step + 1;
    S->active = any_active;
    if (any_err) S->err = any_err;
}

// device time at the start of the generation (before the prompt step)
__global__ void loop_stamp_kernel(DevLoop* __restrict__ S) { S->t0 = gtimer(); }
// sampled steps: run the bonus draft forward only when an active sequence
// accepted its whole draft (ref:engine.py:305-322; the accept flags of rows
// j < l are final here).  perm: the step's sequence order.
__global__ void loop_bonus_cond_kernel(DevLoop* __restrict__ S, const int32_t* __restrict__ acc_flag,
                                       const int32_t* __restrict__ perm, int l,
                                       cudaGraphConditionalHandle h_bonus) {
    __shared__ int any;
    pdl_wait();
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    const int i = threadIdx.x;
    if (i < S->b && !S->done[perm[i]]) {
        bool all = true;
        for (int j = 0; j < l; ++j) all &= acc_flag[i * (l + 1) + j] != 0;
        if (all) atomicOr(&any, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        S->bonus = any;
        cudaGraphSetConditional(h_bonus, any ? 1u : 0u);
    }
}

// first node of the graph: the loop condition after the prompt step
__global__ void loop_init_kernel(DevLoop* __restrict__ S, cudaGraphConditionalHandle h_loop) {
    int act = 0;
    for (int i = 0; i < S->b; ++i) act |= !S->done[i];
    S->active = act;
    cudaGraphSetConditional(h_loop, act ? 1u : 0u);
}
// first node of a loop iteration: the branch (draft length) of this step
__global__ void loop_select_kernel(const DevLoop* __restrict__ S, cudaGraphConditionalHandle h_len) {
    cudaGraphSetConditional(h_len, (unsigned)(S->l - S->lmin));
}
// last node of a loop iteration: continue while a sequence is active and no step failed
__global__ void loop_continue_kernel(const DevLoop* __restrict__ S, cudaGraphConditionalHandle h_loop) {
    cudaGraphSetConditional(h_loop, (S->active && !S->err) ? 1u : 0u);
}

}  // namespace bass
