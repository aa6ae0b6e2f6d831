// Device-computed decode loops: batched speculative decoding
// (ref:engine.py:200-385) and regular decoding (ref:engine.py:120-197).
//
// The host keeps only bookkeeping (committed tokens, cache lengths, the
// Algorithm-1 state); every forward, every draft pick (greedy or sampled),
// the verify accept/resample pass, the bonus token, EOS/length finalize and
// the logprobs run on the GPU.  One device->host read per step returns the
// per-slot outcome (accepted count, emitted tokens, logprobs, finish flag).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "runtime.h"
#include "cluster_sampling.cuh"

using namespace bass;

struct bass_engine {
    bass_ctx* ctx = nullptr;          // kept so destroy never touches a freed model
    bass_model* main = nullptr;
    bass_model* draft = nullptr;
    bass_kv* kv_main = nullptr;
    bass_kv* kv_draft = nullptr;
    int n_slots = 0, cap = 0;
    int strategy = BASS_RAGGED;
    int n_alloc = 0;                  // slots the per-slot buffers are sized for
    int pstride = 1;                  // proposal row stride of the current generation (draft limit + 1)
    DevBuf proposals;                 // [n_slots][pstride] draft proposals (token ids; never leave the device)
    DevBuf vlog, dlog, vamax, vlse, accf, corr, bonus, scratch, slotbuf, stepbuf, align_tok, arena, pick, shaped;
    char* step_host = nullptr;        // pinned: per-step slot records (slot_rec_bytes)
    size_t step_host_cap = 0;
    int32_t* props() { return (int32_t*)proposals.p; }
};

namespace {

using clk = std::chrono::steady_clock;

double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

template <typename F>
int guarded_e(bass_engine* e, F&& f) {
    bass_ctx* c = e ? e->main->ctx : nullptr;
    try {
        f();
        return BASS_OK;
    } catch (const Error& x) {
        if (c) c->err = x.what();
        return x.code;
    } catch (const std::exception& x) {
        if (c) c->err = x.what();
        return BASS_ERR_STATE;
    }
}

void launched(bass_ctx* c) {
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(BASS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

void up(bass_ctx* c, void* dev, const void* src, size_t bytes) {
    void* h = c->staging.take(bytes);
    if (!h) {
        c->sync();
        h = c->staging.take(bytes);
        if (!h) throw Error(BASS_ERR_MEMORY, "staging arena too small");
    }
    std::memcpy(h, src, bytes);
    BASS_CUDA(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += (int64_t)bytes;
}

// Algorithm 1 (ref:draft_control.py:49-69)
struct Controller {
    int fixed, l, s, incre, mod, limit;
    int length() const { return fixed ? fixed : l; }
    int max_length() const { return fixed ? fixed : limit; }
    void observe(const std::vector<int>& acc) {
        if (fixed || acc.empty()) return;
        int mx = 0;
        for (int a : acc) mx = std::max(mx, a);
        if (mx == l) {
            l = std::min(l + incre, limit);
            s = 0;
        } else {
            int ln = l - (l + mod - 1) / mod - s;
            l = std::max(std::max(1, mx), ln);
            s = 1;
        }
    }
};

struct Request {
    int b;
    std::vector<std::vector<int32_t>> prompts;
    std::vector<int64_t> sid;
};

Request parse(const bass_gen_request* r, int V) {
    Request q;
    BASS_REQUIRE(r->batch >= 1, "batch size must be >= 1");
    BASS_REQUIRE(r->max_new_tokens >= 1, "max_new_tokens must be >= 1");
    q.b = r->batch;
    for (int i = 0; i < r->batch; ++i) {
        const int a = r->prompt_offsets[i], z = r->prompt_offsets[i + 1];
        BASS_REQUIRE(z > a, "every prompt needs at least one token");
        q.prompts.emplace_back(r->prompt_tokens + a, r->prompt_tokens + z);
        for (int t : q.prompts.back()) BASS_REQUIRE(t >= 0 && t < V, "token id outside vocab");
        q.sid.push_back(r->sequence_ids ? r->sequence_ids[i] : i);
        BASS_REQUIRE(q.sid.back() >= 0, "sequence ids must be non-negative");
    }
    BASS_REQUIRE(r->top_p > 0.0 && r->top_p <= 1.0, "top_p must be in (0, 1]");
    BASS_REQUIRE(r->temperature >= 0.0, "temperature must be >= 0");
    return q;
}

}  // namespace

extern "C" {

int bass_engine_create(bass_model* mm, bass_kv* mkv, bass_model* dm, bass_kv* dkv, bass_engine** out) {
    *out = nullptr;
    bass_engine tmp;
    tmp.main = mm;
    return guarded_e(&tmp, [&] {
        BASS_REQUIRE(dm == nullptr || dm->ctx == mm->ctx, "main and draft must share a context");
        BASS_REQUIRE(mkv && mkv->m == mm, "main cache must belong to the main model");
        BASS_REQUIRE(dm == nullptr || (dkv && dkv->m == dm), "draft cache must belong to the draft model");
        bass_engine* e = new bass_engine();
        e->ctx = mm->ctx;
        e->main = mm;
        e->draft = dm;
        e->kv_main = mkv;
        e->kv_draft = dkv;
        e->n_slots = dkv ? std::min(mkv->n_slots, dkv->n_slots) : mkv->n_slots;
        e->cap = dkv ? std::min(mkv->cap, dkv->cap) : mkv->cap;
        e->n_alloc = std::max(mkv->n_slots, dkv ? dkv->n_slots : 0);
        *out = e;
    });
}

int bass_engine_destroy(bass_engine* e) {
    if (!e) return BASS_OK;
    cudaStreamSynchronize(e->ctx->stream);
    if (e->step_host) cudaFreeHost(e->step_host);
    for (DevBuf* b : {&e->proposals, &e->vlog, &e->dlog, &e->vamax, &e->vlse, &e->accf, &e->corr, &e->bonus, &e->scratch,
                      &e->slotbuf, &e->stepbuf, &e->align_tok, &e->arena, &e->pick, &e->shaped})
        b->release();
    delete e;
    return BASS_OK;
}

int bass_engine_set_strategy(bass_engine* e, int strategy) {
    return guarded_e(e, [&] {
        BASS_REQUIRE(strategy >= BASS_PAD && strategy <= BASS_RAGGED, "unknown strategy");
        e->strategy = strategy;
    });
}

// ------------------------------------------------------------------ spec
int bass_spec_generate(bass_engine* e, const bass_gen_request* r, bass_gen_result* res) {
    return guarded_e(e, [&] {
        BASS_REQUIRE(e->draft != nullptr, "speculative decoding needs a draft model");
        bass_model& M = *e->main;
        bass_model& D = *e->draft;
        bass_ctx* c = M.ctx;
        cudaStream_t st = c->stream;
        const int V = M.g.vocab_size;
        BASS_REQUIRE(D.g.vocab_size == V, "vocab mismatch: main " + std::to_string(V) + " vs draft " +
                                              std::to_string(D.g.vocab_size));
        Request q = parse(r, V);
        const int b = q.b;
        BASS_REQUIRE(b <= e->n_slots, "batch exceeds engine slots");
        Controller ctl{r->ctl_fixed, r->l0, r->s0, r->incre, r->mod, r->limit};
        if (!r->ctl_fixed) {
            BASS_REQUIRE(r->l0 >= 1 && r->l0 <= r->limit, "l0 must be in [1, limit]");
            BASS_REQUIRE(r->s0 == 0 || r->s0 == 1, "s must be 0 or 1");
            BASS_REQUIRE(r->incre >= 0 && r->mod >= 1 && r->limit >= 1, "incre >= 0, mod >= 1, limit >= 1 required");
        }
        const int limit = ctl.max_length();
        BASS_REQUIRE(limit >= 1, "draft limit must be >= 1");
        // the keyed acceptance override replaces proposals by point masses; a
        // sampled verify would then divide by a zero draft probability
        BASS_REQUIRE(r->align < 0.0 || r->temperature == 0.0, "the keyed acceptance override (align) needs greedy decoding");
        const int max_seq = std::min(M.g.max_seq_len, D.g.max_seq_len);
        for (auto& p : q.prompts)
            BASS_REQUIRE((int)p.size() + r->max_new_tokens + limit <= max_seq,
                         "context overflow: prompt (" + std::to_string(p.size()) + ") + max_new_tokens (" +
                             std::to_string(r->max_new_tokens) + ") + draft limit (" + std::to_string(limit) +
                             ") exceeds max_seq_len " + std::to_string(max_seq));
        for (auto& p : q.prompts)
            BASS_REQUIRE((int)p.size() + r->max_new_tokens + limit <= e->cap, "context exceeds cache capacity");
        const bool greedy = r->temperature == 0.0;
        const int maxnew = r->max_new_tokens;

        // per-slot device tables: sequence id (int64), prompt length (by slot)
        char* slot_tab = (char*)e->slotbuf.need((size_t)e->n_slots * 12, st);
        std::vector<int64_t> sids(e->n_slots, 0);
        std::vector<int32_t> plens(e->n_slots, 0);
        for (int s = 0; s < b; ++s) {
            sids[s] = q.sid[s];
            plens[s] = (int32_t)q.prompts[s].size();
        }
        up(c, slot_tab, sids.data(), sids.size() * 8);
        up(c, slot_tab + (size_t)e->n_slots * 8, plens.data(), plens.size() * 4);
        const int64_t* d_sid = (const int64_t*)slot_tab;
        const int32_t* d_plen = (const int32_t*)(slot_tab + (size_t)e->n_slots * 8);
        // proposals [slot][limit + 1] and the per-step slot records (<= limit + 1 tokens each)
        e->pstride = limit + 1;
        e->proposals.need((size_t)e->n_alloc * e->pstride * 4, st);
        const int estride = limit + 1;
        const size_t rec = slot_rec_bytes(estride);
        if (e->step_host_cap < (size_t)b * rec) {
            c->sync();
            if (e->step_host) cudaFreeHost(e->step_host);
            e->step_host = nullptr;
            e->step_host_cap = 0;
            BASS_CUDA(cudaMallocHost((void**)&e->step_host, (size_t)b * rec));
            e->step_host_cap = (size_t)b * rec;
        }
        const int32_t* d_align = nullptr;
        if (r->align >= 0.0) {
            BASS_REQUIRE(r->align_tokens != nullptr, "align_tokens required when align >= 0");
            int32_t* at = (int32_t*)e->align_tok.need((size_t)b * maxnew * 4, st);
            BASS_CUDA(cudaMemcpyAsync(at, r->align_tokens, (size_t)b * maxnew * 4, cudaMemcpyHostToDevice, st));
            c->h2d_bytes += (int64_t)b * maxnew * 4;
            d_align = at;
        }
        // the caches continue from their current lengths (fresh providers: 0,
        // so step 1's blocks carry the whole prompt, ref:engine.py:248, 268)
        for (int s = 0; s < b; ++s)
            BASS_REQUIRE(e->kv_main->len[s] < (int)q.prompts[s].size() + 0 &&
                             e->kv_draft->len[s] < (int)q.prompts[s].size(),
                         "cached context longer than the prompt");

        std::vector<std::vector<int32_t>> com(b);
        for (int s = 0; s < b; ++s) com[s] = q.prompts[s];
        std::vector<int> ngen(b, 0), done(b, 0);
        for (int s = 0; s < b; ++s) {
            res->n_tokens[s] = 0;
            res->finish_reason[s] = -1;
            res->completion_step[s] = 0;
            res->finish_wall_s[s] = 0.0;
        }
        int64_t main_calls = 0, draft_calls = 0;
        double host_enqueue_s = 0.0, sync_wait_s = 0.0;
        int step = 0;
        const auto t0 = clk::now();
        const int Lmax = limit + 1;
        // device buffers sized for the worst step
        float* vlog = (float*)e->vlog.need((size_t)b * Lmax * V * 4, st);
        float* dlog = (float*)e->dlog.need((size_t)Lmax * b * V * 4, st);
        int32_t* vamax = (int32_t*)e->vamax.need((size_t)b * Lmax * 4, st);
        double* vlse = (double*)e->vlse.need((size_t)b * Lmax * 8, st);
        int32_t* accf = (int32_t*)e->accf.need((size_t)b * Lmax * 4, st);
        int32_t* corr = (int32_t*)e->corr.need((size_t)b * Lmax * 4, st);
        int32_t* btok = (int32_t*)e->bonus.need((size_t)b * 4, st);
        double* scratch = greedy ? nullptr : (double*)e->scratch.need((size_t)b * Lmax * 2 * V * 8, st);
        char* step_dev = (char*)e->stepbuf.need((size_t)b * rec, st);
        // split greedy draft pick: partials [b][P] {value, index} + per-row arrival counters (zeroed here,
        // re-armed by the kernel)
        float* pick_v = (float*)e->pick.need((size_t)b * (2 * GREEDY_PARTS + 1) * 4, st);
        int* pick_i = (int*)(pick_v + (size_t)b * GREEDY_PARTS);
        int* pick_cnt = pick_i + (size_t)b * GREEDY_PARTS;
        BASS_CUDA(cudaMemsetAsync(pick_cnt, 0, (size_t)b * 4, st));

        // any error inside a step (CUDA, a zero draft probability, an empty
        // residual) rolls both caches back to the committed prefix first, so
        // the providers stay usable (ref:engine.py:358-360 invariant)
        try {
            while (true) {
                std::vector<int> A;
                for (int s = 0; s < b; ++s)
                    if (!done[s]) A.push_back(s);
                if (A.empty()) break;
                ++step;
                const auto ts = clk::now();
                const int l = ctl.length(), nA = (int)A.size();
                // ---- the step's metadata in ONE upload (one PDL chain from the
                // first draft kernel to finalize): per-active tables (slot,
                // committed C, generated count), every draft forward's and the
                // verify forward's batch metadata, the draft positions per j.  All
                // of it is known on the host before the step's first kernel.
                const int nd = l + (greedy ? 0 : 1);   // draft forwards (sampled: + the bonus row)
                std::vector<Batch> dbt(nd);
                Batch vbt;
                std::vector<int32_t> ar(3 * nA);
                for (int i = 0; i < nA; ++i) {
                    ar[i] = A[i];
                    ar[nA + i] = (int32_t)com[A[i]].size();
                    ar[2 * nA + i] = ngen[A[i]];
                }
                std::vector<PreMetaOff> doff(nd);
                std::vector<size_t> pos_off(nd);
                PreMetaOff voff;
                {
                    std::vector<int> dl(nA);
                    std::vector<int32_t> dsafe(nA), vsafe(nA);   // cache lengths at the step's upload
                    for (int i = 0; i < nA; ++i) {
                        dl[i] = dsafe[i] = e->kv_draft->len[A[i]];
                        vsafe[i] = e->kv_main->len[A[i]];
                    }
                    for (int j = 0; j < nd; ++j) {
                        Batch& bt = dbt[j];
                        for (int i = 0; i < nA; ++i) {
                            const int s = A[i];
                            if (j == 0) {
                                const int C = (int)com[s].size();
                                BASS_REQUIRE(dl[i] < C, "draft cache ahead of committed prefix");
                                bt.add_seq(s, dl[i], com[s].data() + dl[i], C - dl[i]);
                            } else {
                                const int32_t ind = -j;   // proposals[s][j-1]
                                bt.add_seq(s, dl[i], &ind, 1);
                            }
                            bt.logit_rows.push_back(bt.rows() - 1);
                            dl[i] += bt.qn[i];
                        }
                        doff[j] = forward_premeta(D, bt, e->strategy, dsafe, ar);
                        ar.resize((ar.size() + 7) & ~(size_t)7, 0);
                        pos_off[j] = ar.size();
                        for (int i = 0; i < nA; ++i) ar.push_back((int32_t)com[A[i]].size() + j);
                    }
                    std::vector<int32_t> blk;
                    for (int i = 0; i < nA; ++i) {
                        const int s = A[i];
                        const int ml = e->kv_main->len[s];
                        blk.assign(com[s].begin() + ml, com[s].end());
                        for (int j = 0; j < l; ++j) blk.push_back(-(j + 1));
                        vbt.add_seq(s, ml, blk.data(), (int)blk.size());
                        for (int j = 0; j <= l; ++j) vbt.logit_rows.push_back(vbt.rows() - (l + 1) + j);
                    }
                    voff = forward_premeta(M, vbt, e->strategy, vsafe, ar);
                }
                int32_t* dar = (int32_t*)e->arena.need(ar.size() * 4, st);
                up(c, dar, ar.data(), ar.size() * 4);
                const int32_t* d_slot = dar;
                const int32_t* d_com = dar + nA;
                const int32_t* d_gen = dar + 2 * nA;

                // ---------------------------------------------- draft phase
                for (int j = 0; j < nd; ++j) {
                    const Batch& bt = dbt[j];
                    float* out = dlog + (size_t)j * nA * V;
                    const PreMeta pm = premeta_at(dar, doff[j]);
                    forward(D, *e->kv_draft, bt, e->strategy, out, e->props(), e->pstride, &pm);
                    for (int i = 0; i < nA; ++i) e->kv_draft->len[A[i]] += bt.qn[i];
                    if (j == l) break;   // sampled bonus row: no pick here
                    draft_calls += nA;
                    const int32_t* d_pos = dar + pos_off[j];
                    DraftPick dp{d_slot, d_sid, d_pos, e->props(), e->pstride, j,
                                 r->align, r->align_seed, d_align, d_plen, maxnew};
                    ProfScope prof(c, BASS_PROF_SAMPLE, (double)nA * V * 4);
                    if (greedy) BASS_CUDA(launch_pdl(draft_greedy_split_kernel, dim3(nA, GREEDY_PARTS), dim3(256), 0, st,
                                                     (const float*)out, V, dp, pick_v, pick_i, pick_cnt));
                    else cl_draft_sample_kernel<<<nA * CL_CTAS, CL_THREADS, 0, st>>>(out, V, r->temperature, r->top_p, r->seed,
                                                                         scratch, dp);
                    launched(c);
                }
                // ---------------------------------------------- verify
                {
                    const Batch& bt = vbt;
                    const PreMeta pm = premeta_at(dar, voff);
                    forward(M, *e->kv_main, bt, e->strategy, vlog, e->props(), e->pstride, &pm);
                    for (int i = 0; i < nA; ++i) e->kv_main->len[A[i]] += bt.qn[i];
                    main_calls += nA;
                }
                const int R = nA * (l + 1);
                {
                    ProfScope prof(c, BASS_PROF_SAMPLE, (double)R * V * 4);
                    BASS_CUDA(launch_pdl(row_stats_kernel, dim3(R), dim3(SM_THREADS), 0, st, (const float*)vlog, V, vamax,
                                         vlse));
                }
                launched(c);
                if (!greedy) {
                    VerifyArgs va{nA, l, V, r->temperature, r->top_p, r->seed, d_slot, d_sid, d_com,
                                  e->props(), e->pstride, vlog, dlog, scratch, accf, corr, btok};
                    ProfScope prof(c, BASS_PROF_SAMPLE, (double)R * V * 8);
                    Shaped* shp = (Shaped*)e->shaped.need((size_t)nA * (l + 1) * 2 * sizeof(Shaped), st);
                    cl_verify_shape_kernel<<<dim3((l + 1) * CL_CTAS, nA, 2), CL_THREADS, 0, st>>>(va, shp);
                    launched(c);
                    cl_verify_accept_kernel<<<dim3((l + 1) * CL_CTAS, nA), CL_THREADS, 0, st>>>(va, shp);
                    launched(c);
                }
                StepArgs sa{nA, l, V, d_slot, d_com, d_gen, e->props(), e->pstride, vlog, vamax, vlse,
                            maxnew, r->eos_token, accf, corr, btok, greedy ? 1 : 0, step_dev, estride};
                BASS_CUDA(launch_pdl(finalize_kernel, dim3((nA + 63) / 64), dim3(64), 0, st, sa));
                launched(c);
                c->d2h_bytes += (int64_t)(nA * rec);
                BASS_CUDA(cudaMemcpyAsync(e->step_host, step_dev, (size_t)nA * rec, cudaMemcpyDeviceToHost, st));
                const auto t_enq = clk::now();
                host_enqueue_s += secs(ts, t_enq);
                c->sync();
                sync_wait_s += secs(t_enq, clk::now());
                const double now = secs(t0, clk::now());
                // ---------------------------------------------- bookkeeping
                std::vector<int> acc(nA);
                if (res->step_draft_len && step <= res->max_steps) {
                    res->step_draft_len[step - 1] = l;
                    res->step_wall_s[step - 1] = secs(ts, clk::now());
                }
                for (int i = 0; i < nA; ++i) {
                    const int s = A[i];
                    char* orec = e->step_host + (size_t)i * rec;
                    const SlotStep& o = *reinterpret_cast<const SlotStep*>(orec);
                    const int32_t* o_tok = slot_rec_tok(orec);
                    const double* o_lp = slot_rec_lp(orec, estride);
                    if (o.err == -2)
                        throw Error(BASS_ERR_VALUE, "draft token has zero draft probability");
                    if (o.err == -3) throw Error(BASS_ERR_VALUE, "residual is empty: q <= p everywhere");
                    acc[i] = o.accepted;
                    // reference counts the bonus draft forward per eligible slot
                    if (!greedy && o.accepted == l && o.n_emit >= 1) {
                        bool eos_in_core = false;
                        for (int j = 0; j < std::min(o.n_emit, l); ++j)
                            eos_in_core |= (r->eos_token >= 0 && o_tok[j] == r->eos_token);
                        if (!eos_in_core && maxnew - ngen[s] > l) ++draft_calls;
                    }
                    for (int j = 0; j < o.n_emit; ++j) {
                        res->tokens[(size_t)s * maxnew + ngen[s] + j] = o_tok[j];
                        res->logprobs[(size_t)s * maxnew + ngen[s] + j] = o_lp[j];
                        com[s].push_back(o_tok[j]);
                    }
                    ngen[s] += o.n_emit;
                    if (o.reason >= 0) {
                        done[s] = 1;
                        res->finish_reason[s] = o.reason;
                        res->completion_step[s] = step;
                        res->finish_wall_s[s] = now;
                    }
                    const int target = (int)com[s].size() - 1;   // ref:engine.py:358-360
                    e->kv_main->len[s] = std::min(e->kv_main->len[s], target);
                    e->kv_draft->len[s] = std::min(e->kv_draft->len[s], target);
                    if (res->step_accepted && step <= res->max_steps) {
                        res->step_accepted[(size_t)(step - 1) * b + s] = o.accepted;
                        res->step_emitted[(size_t)(step - 1) * b + s] = o.n_emit;
                    }
                }
                if (res->step_accepted && step <= res->max_steps)
                    for (int s = 0; s < b; ++s) {
                        if (done[s] && res->completion_step[s] != step) {
                            res->step_accepted[(size_t)(step - 1) * b + s] = -1;
                            res->step_emitted[(size_t)(step - 1) * b + s] = -1;
                        }
                        res->step_kv_len[(size_t)(step - 1) * b + s] = (int32_t)com[s].size();
                    }
                ctl.observe(acc);
            }
        } catch (...) {
            for (int s = 0; s < b; ++s) {
                const int target = (int)com[s].size() - 1;
                e->kv_main->len[s] = std::min(e->kv_main->len[s], target);
                e->kv_draft->len[s] = std::min(e->kv_draft->len[s], target);
            }
            throw;
        }
        for (int s = 0; s < b; ++s) res->n_tokens[s] = ngen[s];
        res->n_steps = step;
        res->main_forward_calls = main_calls;
        res->draft_forward_calls = draft_calls;
        res->wall_s = secs(t0, clk::now());
        res->final_l_draft = ctl.l;
        res->final_s = ctl.s;
        res->host_enqueue_s = host_enqueue_s;
        res->sync_wait_s = sync_wait_s;
    });
}

// --------------------------------------------------------------- regular
int bass_regular_generate(bass_engine* e, const bass_gen_request* r, bass_gen_result* res) {
    return guarded_e(e, [&] {
        bass_model& M = *e->main;
        bass_ctx* c = M.ctx;
        cudaStream_t st = c->stream;
        const int V = M.g.vocab_size;
        Request q = parse(r, V);
        const int b = q.b, maxnew = r->max_new_tokens;
        BASS_REQUIRE(b <= e->n_slots, "batch exceeds engine slots");
        for (auto& p : q.prompts)
            BASS_REQUIRE((int)p.size() + maxnew <= M.g.max_seq_len,
                         "prompt (" + std::to_string(p.size()) + ") + max_new_tokens (" + std::to_string(maxnew) +
                             ") exceeds max_seq_len " + std::to_string(M.g.max_seq_len));
        for (auto& p : q.prompts) BASS_REQUIRE((int)p.size() + maxnew <= e->cap, "context exceeds cache capacity");
        const bool greedy = r->temperature == 0.0;
        int64_t* slot_tab = (int64_t*)e->slotbuf.need((size_t)e->n_slots * 8, st);
        std::vector<int64_t> sids(e->n_slots, 0);
        for (int s = 0; s < b; ++s) sids[s] = q.sid[s];
        up(c, slot_tab, sids.data(), sids.size() * 8);
        e->pstride = 1;   // proposals[slot][0]: the token picked for the next forward
        e->proposals.need((size_t)e->n_alloc * 4, st);
        for (int s = 0; s < b; ++s)
            BASS_REQUIRE(e->kv_main->len[s] == 0, "sequence " + std::to_string(s) + " already has cached context");
        float* cur = (float*)e->vlog.need((size_t)b * V * 4, st);
        double* scratch = greedy ? nullptr : (double*)e->scratch.need((size_t)b * V * 8, st);
        int32_t* per = (int32_t*)e->stepbuf.need((size_t)b * 4 * 4 + (size_t)b * 16, st);
        int32_t* d_slot = per;
        int32_t* d_pos = per + b;
        int32_t* d_tok = per + 2 * b;
        double* d_lp = (double*)(per + 4 * b);
        std::vector<int> ngen(b, 0), done(b, 0);
        for (int s = 0; s < b; ++s) {
            res->n_tokens[s] = 0;
            res->finish_reason[s] = -1;
            res->completion_step[s] = 0;
        }
        const auto t0 = clk::now();
        // prefill all slots in one ragged block (row-independent == per-slot prefill)
        {
            Batch bt;
            for (int s = 0; s < b; ++s) {
                bt.add_seq(s, 0, q.prompts[s].data(), (int)q.prompts[s].size());
                bt.logit_rows.push_back(bt.rows() - 1);
            }
            forward(M, *e->kv_main, bt, e->strategy, cur, nullptr, 0);
            for (int s = 0; s < b; ++s) e->kv_main->len[s] = (int)q.prompts[s].size();
        }
        int64_t main_calls = b;
        std::vector<int> A;
        for (int s = 0; s < b; ++s) A.push_back(s);
        int step = 0;
        std::vector<int32_t> htok(b);
        std::vector<double> hlp(b);
        while (!A.empty()) {
            ++step;
            const auto ts = clk::now();
            const int nA = (int)A.size();
            std::vector<int32_t> h(2 * nA);
            for (int i = 0; i < nA; ++i) {
                h[i] = A[i];
                h[nA + i] = (int32_t)q.prompts[A[i]].size() + ngen[A[i]];
            }
            up(c, d_slot, h.data(), nA * 4);
            up(c, d_pos, h.data() + nA, nA * 4);
            RegularArgs ra{d_slot, slot_tab, d_pos, e->props(), e->pstride, V, r->temperature,
                           r->top_p, r->seed, scratch, d_tok, d_lp};
            {
                ProfScope prof(c, BASS_PROF_SAMPLE, (double)nA * V * 4);
                cl_regular_pick_kernel<<<nA * CL_CTAS, CL_THREADS, 0, st>>>(cur, ra);
            }
            launched(c);
            c->d2h_bytes += (int64_t)nA * 12;
            BASS_CUDA(cudaMemcpyAsync(htok.data(), d_tok, nA * 4, cudaMemcpyDeviceToHost, st));
            BASS_CUDA(cudaMemcpyAsync(hlp.data(), d_lp, nA * 8, cudaMemcpyDeviceToHost, st));
            c->sync();
            std::vector<int> surv;
            for (int i = 0; i < nA; ++i) {
                const int s = A[i];
                res->tokens[(size_t)s * maxnew + ngen[s]] = htok[i];
                res->logprobs[(size_t)s * maxnew + ngen[s]] = hlp[i];
                ++ngen[s];
                int why = -1;
                if (r->eos_token >= 0 && htok[i] == r->eos_token) why = 0;
                else if (ngen[s] >= maxnew) why = 1;
                if (why >= 0) {
                    done[s] = 1;
                    res->finish_reason[s] = why;
                } else {
                    surv.push_back(s);
                }
            }
            if (!surv.empty()) {
                Batch bt;
                const int32_t ind = -1;
                for (int s : surv) {
                    bt.add_seq(s, e->kv_main->len[s], &ind, 1);
                    bt.logit_rows.push_back(bt.rows() - 1);
                }
                forward(M, *e->kv_main, bt, e->strategy, cur, e->props(), e->pstride);
                for (int s : surv) e->kv_main->len[s] += 1;
                main_calls += (int64_t)surv.size();
            }
            const double now = secs(t0, clk::now());
            for (int s : A)
                if (done[s] && res->completion_step[s] == 0) {
                    res->completion_step[s] = step;
                    res->finish_wall_s[s] = now;
                }
            if (res->step_draft_len && step <= res->max_steps) {
                res->step_draft_len[step - 1] = 0;
                res->step_wall_s[step - 1] = secs(ts, clk::now());
                for (int s = 0; s < b; ++s) {
                    const bool act = std::find(A.begin(), A.end(), s) != A.end();
                    res->step_accepted[(size_t)(step - 1) * b + s] = act ? 0 : -1;
                    res->step_emitted[(size_t)(step - 1) * b + s] = act ? 1 : -1;
                    res->step_kv_len[(size_t)(step - 1) * b + s] = (int32_t)q.prompts[s].size() + ngen[s];
                }
            }
            A = surv;
        }
        for (int s = 0; s < b; ++s) res->n_tokens[s] = ngen[s];
        res->n_steps = step;
        res->main_forward_calls = main_calls;
        res->draft_forward_calls = 0;
        res->wall_s = secs(t0, clk::now());
    });
}

}  // extern "C"
