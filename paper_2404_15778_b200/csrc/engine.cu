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
#include <cstdio>
#include <cstdlib>

#include <array>
#include <numeric>

#include "runtime.h"
#include "cluster_sampling.cuh"
#include "loop_graph.cuh"

using namespace bass;

// the captured device-resident decode loop of one request shape (loop_graph.cuh)
// a context's algorithmic counters {launches, bytes, flops} per kernel class
using AlgoVec = std::array<double, 3 * BASS_PROF_N>;
static AlgoVec algo_take(const bass_ctx* c) {
    AlgoVec v;
    for (int x = 0; x < BASS_PROF_N; ++x) {
        v[3 * x] = (double)c->algo_n[x];
        v[3 * x + 1] = c->algo_bytes[x];
        v[3 * x + 2] = c->algo_flops[x];
    }
    return v;
}
static void algo_set(bass_ctx* c, const AlgoVec& v) {
    for (int x = 0; x < BASS_PROF_N; ++x) {
        c->algo_n[x] = (int64_t)v[3 * x];
        c->algo_bytes[x] = v[3 * x + 1];
        c->algo_flops[x] = v[3 * x + 2];
    }
}
static AlgoVec algo_sub(const AlgoVec& a, const AlgoVec& b) {
    AlgoVec v;
    for (int i = 0; i < 3 * BASS_PROF_N; ++i) v[i] = a[i] - b[i];
    return v;
}

struct LoopGraph {
    std::vector<double> key;          // every scalar / pointer baked into its kernels
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int lmin = 1, lmax = 1;
    // per branch (l - lmin): launches and algorithmic {launches, bytes, flops} per
    // kernel class of one step, recorded while capturing (attention excluded:
    // its bytes depend on the lengths and are counted from the step trace)
    std::vector<int64_t> launches, launches_b;   // _b: the conditional bonus part (sampled)
    std::vector<AlgoVec> algo, algo_b;
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        exec = nullptr;
        graph = nullptr;
        key.clear();
    }
};

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
    // device-resident loop (BASS_LOOP_DEVICE): state, plan arena, the graph
    int loop_mode = BASS_LOOP_DEVICE;
    DevBuf loopbuf, looparena;
    LoopGraph lg;
    int64_t graph_builds = 0;
    int last_mode = BASS_LOOP_HOST, last_syncs = 0;
    std::string graph_fallback;       // why the last generation fell back to the host loop ("" if it did not)
    char* loop_host = nullptr;        // pinned read-back of the device loop state
    size_t loop_host_cap = 0;
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
    e->lg.reset();
    if (e->loop_host) cudaFreeHost(e->loop_host);
    for (DevBuf* b : {&e->loopbuf, &e->looparena, &e->proposals, &e->vlog, &e->dlog, &e->vamax, &e->vlse, &e->accf, &e->corr, &e->bonus, &e->scratch,
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

int bass_engine_set_loop(bass_engine* e, int mode) {
    return guarded_e(e, [&] {
        BASS_REQUIRE(mode == BASS_LOOP_HOST || mode == BASS_LOOP_DEVICE, "unknown loop mode");
        e->loop_mode = mode;
    });
}

int bass_engine_loop_info(const bass_engine* e, int32_t* last_mode, int32_t* last_syncs, int64_t* graph_builds) {
    if (!e) return BASS_ERR_STATE;
    if (last_mode) *last_mode = e->last_mode;
    if (last_syncs) *last_syncs = e->last_syncs;
    if (graph_builds) *graph_builds = e->graph_builds;
    return BASS_OK;
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
        // the keyed acceptance override: greedy replaces the proposal token;
        // sampled also turns the draft row into a point mass on it
        // (cl_draft_sample_kernel), so the verify never sees a zero draft probability
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

        // ------------------------------------------------------------------
        // device-resident loop (loop_graph.cuh): the prompt step is planned on
        // the host and enqueued as usual, its outcome booked on the device, and
        // every later step runs from one CUDA graph; one synchronisation per
        // generation
        bool use_graph = e->loop_mode == BASS_LOOP_DEVICE && model_uses_stream_attention(M) &&
                               model_uses_stream_attention(D) && !c->profile && !c->trace_buf &&
                               limit <= GL_MAXL && b <= 1024;
        e->last_mode = use_graph ? BASS_LOOP_DEVICE : BASS_LOOP_HOST;
        e->last_syncs = 0;
        const int g_lmin = ctl.fixed ? ctl.fixed : 1, g_lmax = ctl.fixed ? ctl.fixed : limit;
        const int g_nbr = g_lmax - g_lmin + 1;
        const int com_cap = e->cap, steps_cap = maxnew + 2;
        // DevLoop + arrays in one device buffer (offsets)
        auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
        size_t o_end = al(sizeof(DevLoop));
        auto lay = [&](size_t n) { const size_t r0 = o_end; o_end += al(n); return r0; };
        const size_t o_com = lay((size_t)b * com_cap * 4), o_C = lay((size_t)b * 4), o_ngen = lay((size_t)b * 4),
                     o_done = lay((size_t)b * 4), o_kvm = lay((size_t)b * 4), o_kvd = lay((size_t)b * 4),
                     o_tok = lay((size_t)b * maxnew * 4), o_lp = lay((size_t)b * maxnew * 8),
                     o_reason = lay((size_t)b * 4), o_cstep = lay((size_t)b * 4), o_tfin = lay((size_t)b * 8),
                     o_tstep = lay((size_t)steps_cap * 8), o_trl = lay((size_t)steps_cap * 4),
                     o_tracc = lay((size_t)steps_cap * b * 4), o_tremit = lay((size_t)steps_cap * b * 4),
                     o_trkv = lay((size_t)steps_cap * b * 4), o_ident = lay((size_t)b * 4),
                     o_trb = lay((size_t)steps_cap * 4);
        const size_t g_total = o_end;
        char* dbase = nullptr;
        DevLoop* dS = nullptr;
        DevLoop hs{};
        double g_t_start = 0.0;
        auto graph_setup = [&]() {   // before the prompt step's first kernel
            dbase = (char*)e->loopbuf.need(g_total, st);
            dS = reinterpret_cast<DevLoop*>(dbase);
            std::vector<char> h(g_total, 0);
            hs.b = b; hs.l = ctl.length(); hs.s = ctl.s; hs.step = 0; hs.err = 0; hs.lmin = g_lmin; hs.active = 1;
            hs.fixed = ctl.fixed; hs.incre = ctl.incre; hs.mod = ctl.mod; hs.limit = ctl.limit;
            hs.maxnew = maxnew; hs.estride = estride; hs.com_cap = com_cap; hs.greedy = greedy ? 1 : 0;
            hs.eos = r->eos_token; hs.steps_cap = steps_cap;
            auto P32 = [&](size_t off) { return (int32_t*)(dbase + off); };
            hs.com = P32(o_com); hs.C = P32(o_C); hs.ngen = P32(o_ngen); hs.done = P32(o_done);
            hs.kvm = P32(o_kvm); hs.kvd = P32(o_kvd); hs.tokens = P32(o_tok); hs.lps = (double*)(dbase + o_lp);
            hs.reason = P32(o_reason); hs.cstep = P32(o_cstep);
            hs.tfin = (unsigned long long*)(dbase + o_tfin); hs.tstep = (unsigned long long*)(dbase + o_tstep);
            hs.tr_l = P32(o_trl); hs.tr_acc = P32(o_tracc); hs.tr_emit = P32(o_tremit); hs.tr_kv = P32(o_trkv);
            hs.tr_bonus = P32(o_trb);
            hs.rec = step_dev;
            std::memcpy(h.data(), &hs, sizeof(hs));
            auto H32 = [&](size_t off) { return (int32_t*)(h.data() + off); };
            for (int s = 0; s < b; ++s) {
                BASS_REQUIRE((int)com[s].size() <= com_cap, "device loop: prompt longer than the cache");
                std::memcpy(H32(o_com) + (size_t)s * com_cap, com[s].data(), com[s].size() * 4);
                H32(o_C)[s] = (int32_t)com[s].size();
                H32(o_kvm)[s] = e->kv_main->len[s];
                H32(o_kvd)[s] = e->kv_draft->len[s];
                H32(o_reason)[s] = -1;
                H32(o_ident)[s] = s;
            }
            BASS_CUDA(cudaMemcpyAsync(dbase, h.data(), g_total, cudaMemcpyHostToDevice, st));
            c->h2d_bytes += (int64_t)g_total;
            g_t_start = secs(t0, clk::now());
            loop_stamp_kernel<<<1, 1, 0, st>>>(dS);   // device time of the generation start
            launched(c);
        };
        // capture the loop graph (once per request shape; again when a workspace moved)
        auto graph_capture = [&]() {
            const int max_len = std::min(e->cap, max_seq);
            struct Branch {
                PlanArgs pa;
                std::vector<Batch> bts;   // shapes only (the device writes the values)
            };
            std::vector<Branch> brs(g_nbr);
            size_t arena_ints = 0;
            for (int k = 0; k < g_nbr; ++k) {
                const int l = g_lmin + k, nd = l + (greedy ? 0 : 1);
                Branch& B = brs[k];
                PlanArgs& pa = B.pa;
                std::memset(&pa, 0, sizeof(pa));
                pa.b = b; pa.l = l; pa.strategy = e->strategy;
                pa.ch = stream_chunk_len(); pa.split_ch = stream_split_chunks();
                size_t off = 0;
                auto take = [&](size_t n) { off = (off + 7) & ~(size_t)7; const size_t r0 = off; off += n; return (int)r0; };
                auto add_fwd = [&](int kind, int j, int qq) {
                    PlanFwd& F = pa.f[pa.nf++];
                    F.kind = kind; F.j = j; F.q = qq;
                    const int Mr = b * qq, R = kind == 2 ? Mr : b;
                    F.meta = take((size_t)3 * Mr + 4 * b + R);
                    F.nq = stream_nq_for(qq);
                    F.stride = stream_items_per_seq(qq, max_len);
                    F.work = take((size_t)b * F.stride * 8);
                    F.live = take(2);
                    Batch bt;
                    std::vector<int32_t> dummy(qq, 0);
                    for (int s = 0; s < b; ++s) {
                        bt.add_seq(s, 0, dummy.data(), qq);
                        if (kind == 2)
                            for (int t = 0; t < qq; ++t) bt.logit_rows.push_back(s * qq + t);
                        else
                            bt.logit_rows.push_back(s * qq + qq - 1);
                    }
                    B.bts.push_back(std::move(bt));
                };
                add_fwd(0, 0, 2);
                for (int j = 1; j < nd; ++j) add_fwd(1, j, 1);
                add_fwd(2, 0, l + 1);
                for (int j = 0; j <= l; ++j) pa.pos[j] = take((size_t)b);
                pa.perm = take((size_t)b);
                pa.cperm = take((size_t)b);
                pa.gperm = take((size_t)b);
                arena_ints = std::max(arena_ints, off);
            }
            int32_t* ar = (int32_t*)e->looparena.need(arena_ints * 4 + 256, st);
            Shaped* shp = greedy ? nullptr : (Shaped*)e->shaped.need((size_t)b * Lmax * 2 * sizeof(Shaped), st);
            std::vector<double> key = {(double)b, (double)greedy, (double)e->strategy, r->temperature, r->top_p,
                                       (double)r->seed, (double)r->eos_token, (double)maxnew, r->align,
                                       (double)r->align_seed, (double)g_lmin, (double)g_lmax, (double)estride,
                                       (double)e->pstride, (double)max_len, (double)devbuf_epoch()};
            const size_t k_epoch = key.size() - 1;
            for (const void* p : {(const void*)dbase, (const void*)ar, (const void*)vlog, (const void*)dlog,
                                  (const void*)vamax, (const void*)vlse, (const void*)accf, (const void*)corr,
                                  (const void*)btok, (const void*)scratch, (const void*)step_dev, (const void*)pick_v,
                                  (const void*)e->props(), (const void*)d_sid, (const void*)d_plen,
                                  (const void*)d_align, (const void*)shp, (const void*)M.wblob, (const void*)D.wblob,
                                  (const void*)e->kv_main->k, (const void*)e->kv_draft->k})
                key.push_back((double)(uintptr_t)p);
            LoopGraph& G = e->lg;
            if (G.key == key && G.exec) return;
            G.reset();
            G.lmin = g_lmin;
            G.lmax = g_lmax;
            G.launches.assign(g_nbr, 0);
            G.algo.assign(g_nbr, {});
            G.launches_b.assign(g_nbr, 0);
            G.algo_b.assign(g_nbr, {});
            // capture on a private stream (the caller's stream may still run the
            // prompt step); every launch helper uses ctx->stream
            cudaStream_t cs;
            BASS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            struct Restore {   // also on an exception: end a dangling capture, drop the partial graph
                bass_ctx* c;
                cudaStream_t st, cs;
                LoopGraph& g;
                bool ok = false;
                ~Restore() {
                    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
                    if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
                        cudaGraph_t dangling = nullptr;
                        cudaStreamEndCapture(cs, &dangling);
                    }
                    c->stream = st;
                    cudaStreamDestroy(cs);
                    if (!ok) g.reset();
                    cudaGetLastError();
                }
            } restore{c, st, cs, G};
            c->stream = cs;
            BASS_CUDA(cudaGraphCreate(&G.graph, 0));
            cudaGraphConditionalHandle h_loop, h_len;
            BASS_CUDA(cudaGraphConditionalHandleCreate(&h_loop, G.graph, 0, 0));
            // init -> WHILE(h_loop) { select -> SWITCH(h_len) { step(l) } -> continue }
            auto knode = [&](cudaGraphNode_t* out, cudaGraph_t g, const cudaGraphNode_t* dep, void* fn, void** args) {
                cudaKernelNodeParams kp = {};
                kp.func = fn;
                kp.gridDim = dim3(1);
                kp.blockDim = dim3(1);
                kp.kernelParams = args;
                BASS_CUDA(cudaGraphAddKernelNode(out, g, dep, dep ? 1 : 0, &kp));
            };
            cudaGraphNode_t n_init, n_while, n_sel, n_switch, n_cond;
            void* a_init[] = {(void*)&dS, (void*)&h_loop};
            knode(&n_init, G.graph, nullptr, (void*)loop_init_kernel, a_init);
            cudaGraphNodeParams wp = {};
            wp.type = cudaGraphNodeTypeConditional;
            wp.conditional.handle = h_loop;
            wp.conditional.type = cudaGraphCondTypeWhile;
            wp.conditional.size = 1;
            BASS_CUDA(cudaGraphAddNode(&n_while, G.graph, &n_init, 1, &wp));
            cudaGraph_t body = wp.conditional.phGraph_out[0];
            BASS_CUDA(cudaGraphConditionalHandleCreate(&h_len, body, 0, 0));
            void* a_sel[] = {(void*)&dS, (void*)&h_len};
            knode(&n_sel, body, nullptr, (void*)loop_select_kernel, a_sel);
            cudaGraphNodeParams sw = {};
            sw.type = cudaGraphNodeTypeConditional;
            sw.conditional.handle = h_len;
            sw.conditional.type = cudaGraphCondTypeSwitch;
            sw.conditional.size = (unsigned)g_nbr;
            BASS_CUDA(cudaGraphAddNode(&n_switch, body, &n_sel, 1, &sw));
            void* a_cond[] = {(void*)&dS, (void*)&h_loop};
            knode(&n_cond, body, &n_switch, (void*)loop_continue_kernel, a_cond);
            // branches, largest draft length first (workspaces only grow)
            for (int k = g_nbr - 1; k >= 0; --k) {
                const int l = g_lmin + k, nd = l + (greedy ? 0 : 1), R = b * (l + 1);
                Branch& B = brs[k];
                const int64_t l0 = c->launches;
                const AlgoVec a0 = algo_take(c);
                cudaGraph_t bg = sw.conditional.phGraph_out[k];
                cudaGraphConditionalHandle h_bonus{};
                if (!greedy) BASS_CUDA(cudaGraphConditionalHandleCreate(&h_bonus, bg, 0, 0));
                BASS_CUDA(cudaStreamBeginCaptureToGraph(cs, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
                loop_plan_kernel<<<1, ((b + 31) / 32) * 32, 0, cs>>>(dS, ar, B.pa);
                launched(c);
                const int32_t* perm = ar + B.pa.perm;
                const int32_t* cperm = ar + B.pa.cperm;
                const int32_t* gperm = ar + B.pa.gperm;
                // the draft forwards j < l; sampled: the bonus row's forward (j = l)
                // is conditional, after the verify (below)
                for (int j = 0; j < l; ++j) {
                    const PlanFwd& F = B.pa.f[j];
                    PreMeta pm{ar + F.meta, ar + F.work, true, F.stride, max_len, ar + F.live, ar + F.live + 1};
                    float* out = dlog + (size_t)j * b * V;
                    forward(D, *e->kv_draft, B.bts[j], e->strategy, out, e->props(), e->pstride, &pm);
                    DraftPick dp{perm, d_sid, ar + B.pa.pos[j], e->props(), e->pstride, j,
                                 r->align, r->align_seed, d_align, d_plen, maxnew};
                    ProfScope prof(c, BASS_PROF_SAMPLE, (double)b * V * 4);
                    if (greedy)
                        BASS_CUDA(launch_pdl(draft_greedy_split_kernel, dim3(b, GREEDY_PARTS), dim3(256), 0, cs,
                                             (const float*)out, V, dp, pick_v, pick_i, pick_cnt));
                    else
                        cl_draft_sample_kernel<<<b * CL_CTAS, CL_THREADS, 0, cs>>>(out, V, r->temperature, r->top_p,
                                                                                  r->seed, scratch, dp);
                    launched(c);
                }
                {
                    const PlanFwd& F = B.pa.f[nd];
                    PreMeta pm{ar + F.meta, ar + F.work, true, F.stride, max_len, ar + F.live, ar + F.live + 1};
                    forward(M, *e->kv_main, B.bts[nd], e->strategy, vlog, e->props(), e->pstride, &pm);
                }
                {
                    ProfScope prof(c, BASS_PROF_SAMPLE, (double)R * V * 4);
                    BASS_CUDA(launch_pdl(row_stats_kernel, dim3(R), dim3(SM_THREADS), 0, cs, (const float*)vlog, V,
                                         vamax, vlse));
                }
                launched(c);
                if (!greedy) {
                    VerifyArgs va{b, l, V, r->temperature, r->top_p, r->seed, perm, d_sid, cperm,
                                  e->props(), e->pstride, vlog, dlog, scratch, accf, corr, btok, 1};
                    {
                        ProfScope prof(c, BASS_PROF_SAMPLE, (double)R * V * 8);
                        cl_verify_shape_kernel<<<dim3((l + 1) * CL_CTAS, b, 2), CL_THREADS, 0, cs>>>(va, shp);
                        launched(c);
                        cl_verify_accept_kernel<<<dim3(l * CL_CTAS, b), CL_THREADS, 0, cs>>>(va, shp);
                        launched(c);
                    }
                    BASS_CUDA(launch_pdl(loop_bonus_cond_kernel, dim3(1), dim3(((b + 31) / 32) * 32), 0, cs, dS,
                                         (const int32_t*)accf, perm, l, h_bonus));
                    launched(c);
                    // IF(a sequence accepted its whole draft) { bonus draft forward,
                    // shape its row, draw + accept the bonus token }: end this
                    // capture, hang the conditional node after its last node,
                    // capture the body, then resume the chain after the node
                    cudaStreamCaptureStatus cst;
                    const cudaGraphNode_t* dp0 = nullptr;
                    size_t ndp = 0;
                    BASS_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &dp0, &ndp));
                    std::vector<cudaGraphNode_t> deps(dp0, dp0 + ndp);
                    cudaGraph_t part = nullptr;
                    BASS_CUDA(cudaStreamEndCapture(cs, &part));
                    cudaGraphNodeParams ip = {};
                    ip.type = cudaGraphNodeTypeConditional;
                    ip.conditional.handle = h_bonus;
                    ip.conditional.type = cudaGraphCondTypeIf;
                    ip.conditional.size = 1;
                    cudaGraphNode_t n_if;
                    BASS_CUDA(cudaGraphAddNode(&n_if, bg, deps.data(), deps.size(), &ip));
                    const int64_t lb0 = c->launches;
                    const AlgoVec b0 = algo_take(c);
                    BASS_CUDA(cudaStreamBeginCaptureToGraph(cs, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                            cudaStreamCaptureModeRelaxed));
                    {
                        const PlanFwd& F = B.pa.f[l];
                        PreMeta pm{ar + F.meta, ar + F.work, true, F.stride, max_len, ar + F.live, ar + F.live + 1};
                        forward(D, *e->kv_draft, B.bts[l], e->strategy, dlog + (size_t)l * b * V, e->props(),
                                e->pstride, &pm);
                        VerifyArgs vb = va;
                        vb.phase = 2;
                        ProfScope prof(c, BASS_PROF_SAMPLE, (double)b * V * 8);
                        cl_verify_shape_kernel<<<dim3(CL_CTAS, b, 1), CL_THREADS, 0, cs>>>(vb, shp);
                        launched(c);
                        cl_verify_accept_kernel<<<dim3(CL_CTAS, b), CL_THREADS, 0, cs>>>(vb, shp);
                        launched(c);
                    }
                    cudaGraph_t body = nullptr;
                    BASS_CUDA(cudaStreamEndCapture(cs, &body));
                    G.launches_b[k] = c->launches - lb0;
                    G.algo_b[k] = algo_sub(algo_take(c), b0);
                    BASS_CUDA(cudaStreamBeginCaptureToGraph(cs, bg, &n_if, nullptr, 1, cudaStreamCaptureModeRelaxed));
                }
                StepArgs sa{b, l, V, perm, cperm, gperm, e->props(), e->pstride, vlog, vamax, vlse,
                            maxnew, r->eos_token, accf, corr, btok, greedy ? 1 : 0, step_dev, estride};
                BASS_CUDA(launch_pdl(finalize_kernel, dim3((b + 63) / 64), dim3(64), 0, cs, sa));
                launched(c);
                BASS_CUDA(launch_pdl(loop_book_kernel, dim3(1), dim3(((b + 31) / 32) * 32), 0, cs, dS, perm));
                launched(c);
                cudaGraph_t got = nullptr;
                BASS_CUDA(cudaStreamEndCapture(cs, &got));
                G.launches[k] = c->launches - l0 - G.launches_b[k];
                G.algo[k] = algo_sub(algo_sub(algo_take(c), a0), G.algo_b[k]);
                // capture is not execution: its accounting is replayed per executed step
                c->launches = l0;
                algo_set(c, a0);
            }
            (void)n_cond;
            BASS_CUDA(cudaGraphInstantiate(&G.exec, G.graph, 0));
            restore.ok = true;
            key[k_epoch] = (double)devbuf_epoch();   // (moves only when a workspace grew while capturing)
            G.key = key;
            ++e->graph_builds;
        };
        // after the prompt step's finalize: book it, run the graph, one sync, read back
        auto graph_finish = [&]() {
            // the prompt step's records are in slot order (every slot active)
            BASS_CUDA(launch_pdl(loop_book_kernel, dim3(1), dim3(((b + 31) / 32) * 32), 0, st, dS,
                                 (const int32_t*)(dbase + o_ident)));
            launched(c);
            const auto tq = clk::now();
            graph_capture();
            BASS_CUDA(cudaGraphLaunch(e->lg.exec, st));
            if (e->loop_host_cap < g_total) {   // pinned: the read-back stays asynchronous
                if (e->loop_host) cudaFreeHost(e->loop_host);
                e->loop_host = nullptr;
                e->loop_host_cap = 0;
                BASS_CUDA(cudaMallocHost((void**)&e->loop_host, g_total));
                e->loop_host_cap = g_total;
            }
            char* back_p = e->loop_host;
            BASS_CUDA(cudaMemcpyAsync(back_p, dbase, g_total, cudaMemcpyDeviceToHost, st));
            c->d2h_bytes += (int64_t)g_total;
            const auto tw = clk::now();
            host_enqueue_s += secs(tq, tw);
            c->sync();
            e->last_syncs += 1;
            sync_wait_s += secs(tw, clk::now());
            const LoopGraph& G = e->lg;
            const DevLoop& fs = *reinterpret_cast<const DevLoop*>(back_p);
            auto B32 = [&](size_t off) { return (const int32_t*)(back_p + off); };
            const unsigned long long* tstep = (const unsigned long long*)(back_p + o_tstep);
            const unsigned long long* tfin = (const unsigned long long*)(back_p + o_tfin);
            const int n_steps = fs.step;
            BASS_REQUIRE(n_steps <= steps_cap, "device loop: step trace overflow");
            // accounting of the graph steps (2..n): branch launches / work, attention from the trace
            std::vector<int32_t> Cprev(b);
            for (int s = 0; s < b; ++s) Cprev[s] = B32(o_trkv)[s];   // committed length after step 1
            const int H_m = M.g.n_head, dh_m = M.g.d_head, H_d = D.g.n_head, dh_d = D.g.d_head;
            const double es_m = (double)M.esize, es_d = (double)D.esize;
            for (int k = 1; k < n_steps; ++k) {
                const int l = B32(o_trl)[k], bi = l - G.lmin;
                const bool bon = !greedy && B32(o_trb)[k];   // the conditional bonus draft forward ran
                const int nd = l + (bon ? 1 : 0);
                c->launches += G.launches[bi] + 3 + (bon ? G.launches_b[bi] : 0);   // + select / continue / while
                for (int x = 0; x < BASS_PROF_N; ++x) {
                    c->algo_n[x] += (int64_t)(G.algo[bi][3 * x] + (bon ? G.algo_b[bi][3 * x] : 0.0));
                    c->algo_bytes[x] += G.algo[bi][3 * x + 1] + (bon ? G.algo_b[bi][3 * x + 1] : 0.0);
                    c->algo_flops[x] += G.algo[bi][3 * x + 2] + (bon ? G.algo_b[bi][3 * x + 2] : 0.0);
                }
                double ab = 0.0, af = 0.0;
                auto att = [&](int L, int H, int dh, double es, int off, int qq) {
                    ab += L * (2.0 * H * (off + qq) * dh + 2.0 * H * qq * dh) * es;
                    af += L * 4.0 * H * dh * qq * (off + 0.5 * (qq + 1));
                };
                for (int s = 0; s < b; ++s) {
                    if (B32(o_tracc)[(size_t)k * b + s] < 0) continue;   // finished before this step
                    const int C0 = Cprev[s];
                    att(D.g.n_layer, H_d, dh_d, es_d, C0 - 2, 2);
                    for (int j = 1; j < nd; ++j) att(D.g.n_layer, H_d, dh_d, es_d, C0 + j - 1, 1);
                    att(M.g.n_layer, H_m, dh_m, es_m, C0 - 1, l + 1);
                    Cprev[s] = B32(o_trkv)[(size_t)k * b + s];
                }
                c->algo_n[BASS_PROF_ATTN] += (int64_t)(nd * D.g.n_layer + M.g.n_layer);
                c->algo_bytes[BASS_PROF_ATTN] += ab;
                c->algo_flops[BASS_PROF_ATTN] += af;
            }
            // results into the host state and the caller's arrays
            for (int s = 0; s < b; ++s) {
                const int C = B32(o_C)[s];
                const int32_t* cm = B32(o_com) + (size_t)s * com_cap;
                com[s].assign(cm, cm + C);
                ngen[s] = B32(o_ngen)[s];
                done[s] = B32(o_done)[s];
                e->kv_main->len[s] = B32(o_kvm)[s];
                e->kv_draft->len[s] = B32(o_kvd)[s];
                std::memcpy(res->tokens + (size_t)s * maxnew, B32(o_tok) + (size_t)s * maxnew, (size_t)maxnew * 4);
                std::memcpy(res->logprobs + (size_t)s * maxnew, (const double*)(back_p + o_lp) + (size_t)s * maxnew,
                            (size_t)maxnew * 8);
                if (done[s]) {
                    res->finish_reason[s] = B32(o_reason)[s];
                    res->completion_step[s] = B32(o_cstep)[s];
                    res->finish_wall_s[s] = g_t_start + (double)(tfin[s] - fs.t0) * 1e-9;
                }
            }
            if (res->step_draft_len)
                for (int k = 0; k < n_steps && k < res->max_steps; ++k) {
                    res->step_draft_len[k] = B32(o_trl)[k];
                    res->step_wall_s[k] = (double)(tstep[k] - (k == 0 ? fs.t0 : tstep[k - 1])) * 1e-9;
                    for (int s = 0; s < b; ++s) {
                        res->step_accepted[(size_t)k * b + s] = B32(o_tracc)[(size_t)k * b + s];
                        res->step_emitted[(size_t)k * b + s] = B32(o_tremit)[(size_t)k * b + s];
                        res->step_kv_len[(size_t)k * b + s] = B32(o_trkv)[(size_t)k * b + s];
                    }
                }
            // the device counted every step, the prompt step included (the host
            // enqueue of that step counted it too)
            main_calls = fs.main_calls;
            draft_calls = fs.draft_calls;
            if (!ctl.fixed) {   // a fixed controller keeps the caller's (unused) state
                ctl.l = fs.l;
                ctl.s = fs.s;
            }
            step = n_steps;
            if (fs.err == -2) throw Error(BASS_ERR_VALUE, "draft token has zero draft probability");
            if (fs.err == -3) throw Error(BASS_ERR_VALUE, "residual is empty: q <= p everywhere");
            if (fs.err) throw Error(BASS_ERR_STATE, "device loop error " + std::to_string(fs.err));
        };

        // any error inside a step (CUDA, a zero draft probability, an empty
        // residual) rolls both caches back to the committed prefix first, so
        // the providers stay usable (ref:engine.py:358-360 invariant)
        try {
            if (use_graph) {
                forward_prepare(M);
                forward_prepare(D);
                graph_setup();
                // capture (or reuse) the loop graph before the prompt step, so a
                // driver without conditional graph nodes falls back to the host
                // loop before any step is committed to the device path
                try {
                    graph_capture();
                } catch (const Error& ex) {
                    use_graph = false;
                    e->last_mode = BASS_LOOP_HOST;
                    e->graph_fallback = ex.what();
                }
            }
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
                if (use_graph) {   // the prompt step's outcome is booked on the device; the graph runs the rest
                    graph_finish();
                    break;
                }
                c->d2h_bytes += (int64_t)(nA * rec);
                BASS_CUDA(cudaMemcpyAsync(e->step_host, step_dev, (size_t)nA * rec, cudaMemcpyDeviceToHost, st));
                const auto t_enq = clk::now();
                host_enqueue_s += secs(ts, t_enq);
                c->sync();
                e->last_syncs += 1;
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
