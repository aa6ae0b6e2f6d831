// Host-side runtime objects behind the C ABI (include/bass.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bass.h"
#include "model_kernels.cuh"


namespace bass {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BASS_CUDA(call)                                                                    \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess)                                                             \
            throw ::bass::Error(BASS_ERR_CUDA, std::string(#call) + ": " +                 \
                                                   cudaGetErrorString(_e));                \
    } while (0)

#define BASS_REQUIRE(cond, msg)                                                            \
    do {                                                                                   \
        if (!(cond)) throw ::bass::Error(BASS_ERR_VALUE, (msg));                           \
    } while (0)

// Bump allocator over pinned host memory for per-forward metadata.  Async
// H2D copies may still read an earlier region, so it is only reset at a
// stream synchronisation point.
struct Staging {
    char* base = nullptr;
    size_t cap = 0, used = 0;
    void* take(size_t n);
};

// Device buffer that grows (after a stream sync) when a larger size is needed.
// Every growth bumps a process-wide epoch (devbuf_epoch): a captured CUDA graph
// records it and is re-captured when any workspace it references may have moved.
uint64_t devbuf_epoch();
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    std::vector<void*> retired;   // outgrown while a stream capture referenced them
    void* need(size_t n, cudaStream_t s);
    void release();
};

}  // namespace bass

// Per-kernel-class device timing (CUDA events on the launching stream) with
// the algorithmic bytes / flops of every timed launch; resolved at syncs.
enum { BASS_PROF_GEMM = 0, BASS_PROF_ATTN = 1, BASS_PROF_NORM = 2, BASS_PROF_SAMPLE = 3, BASS_PROF_N = 4 };

struct bass_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int64_t launches = 0;
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    bass::Staging staging;
    bass::DevBuf scr_meta, scr_work, scr_po, scr_pml;   // standalone attention entry points
    // profiling
    bool profile = false;
    struct Pending { int cls; cudaEvent_t a, b; double bytes, flops; };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    double prof_ms[BASS_PROF_N] = {}, prof_bytes[BASS_PROF_N] = {}, prof_flops[BASS_PROF_N] = {};
    int64_t prof_n[BASS_PROF_N] = {};
    // algorithmic work of every launch (counted without events)
    double algo_bytes[BASS_PROF_N] = {}, algo_flops[BASS_PROF_N] = {};
    int64_t algo_n[BASS_PROF_N] = {};
    cudaEvent_t ev();
    void resolve();
    void sync();
    // timeline trace (bass_trace_enable): records of {t0, t1, smid, tag}
    unsigned long long* trace_buf = nullptr;
    long long trace_cap = 0, trace_n = 0;
    int trace_seq = 0;
    bass::TraceArg trace(int grid, int cls) {   // tag = kernel class | launch sequence << 4
        if (!trace_buf || trace_n + grid > trace_cap) return bass::TraceArg{nullptr, 0, 0};
        bass::TraceArg t{trace_buf, trace_n, cls | (trace_seq++ << 4)};
        trace_n += grid;
        return t;
    }
};
// trace tags (kernel classes)
enum { BASS_TR_GEMM = 1, BASS_TR_ATTN = 2, BASS_TR_NORM = 3, BASS_TR_COMBINE = 4 };

namespace bass {
// Algorithmic-work accounting around one launch (always on: launch count,
// bytes, flops per kernel class) plus a CUDA-event timer when ctx->profile.
struct ProfScope {
    bass_ctx* c;
    int cls;
    double bytes, flops;
    cudaEvent_t a = nullptr;
    ProfScope(bass_ctx* c_, int cls_, double bytes_, double flops_ = 0)
        : c(c_), cls(cls_), bytes(bytes_), flops(flops_) {
        c->algo_n[cls] += 1;
        c->algo_bytes[cls] += bytes_;
        c->algo_flops[cls] += flops_;
        if (c->profile) {
            a = c->ev();
            cudaEventRecord(a, c->stream);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = c->ev();
            cudaEventRecord(b, c->stream);
            c->pending.push_back({cls, a, b, bytes, flops});
        }
    }
};
}  // namespace bass

struct bass_layer {
    float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
    void *wqkv, *wo, *wfc, *wproj;   // output-major [N, K]
    double *sqkv, *so, *sfc, *sproj; // BASS_INT8: per-output-channel weight scales
};

struct bass_model {
    bass_ctx* ctx = nullptr;
    bass_geometry g{};
    int dtype = BASS_BF16;
    int gemm_mode = BASS_GEMM_AUTO;
    bool packed = false;             // GEMM weights in the packed tile layout (bf16, d % 64 == 0)
    size_t esize = 2;                // activation / embedding / KV element size (int8 models: bf16)
    size_t wsize = 2;                // GEMM weight element size (int8 models: 1)
    double* sblob = nullptr;         // BASS_INT8: all per-channel weight scales
    double* shead = nullptr;
    bool int8() const { return dtype == BASS_INT8; }
    void* wblob = nullptr;           // all matrices, one allocation
    float* fblob = nullptr;          // LN params
    int64_t weight_bytes = 0;
    void *tok_emb = nullptr, *pos_emb = nullptr, *head = nullptr;
    float *lnf_g = nullptr, *lnf_b = nullptr;
    std::vector<bass_layer> layers;
    // workspace (grown on demand)
    bass::DevBuf x, h, q, ctxb, f, hs, meta, part_o, part_ml, logits_tmp;
    bass::DevBuf lnstats;            // {sum, sum^2} per (128-column tile, row) for folded LayerNorms
    bass::DevBuf lnfold;             // per layer: c, e of LN1 -> QKV and LN2 -> FC (c = W g, e = W b)
    bool lnfold_valid = false;       // recomputed after any weight / LN parameter change
    void* tc_state = nullptr;        // tcgen05 split-K GEMM descriptors (gemm_tc.cu)
    bass::DevBuf attn_work;          // stream-attention work list of the current forward
    bass::DevBuf xq, xs;             // BASS_INT8: per-token int8 GEMM input and its scales
    const int32_t* dev_rows = nullptr;   // device-planned forward: live row count of the next GEMMs (PreMeta::m_act)
};

struct bass_kv {
    bass_model* m = nullptr;
    bass_ctx* ctx = nullptr;          // kept so destroy never touches a freed model
    int n_slots = 0, cap = 0;
    void *k = nullptr, *v = nullptr;  // [L][slot][H][cap][dh]
    std::vector<int32_t> len;
    size_t layer_elems() const {
        return (size_t)n_slots * m->g.n_head * cap * m->g.d_head;
    }
};

namespace bass {

// One ragged forward described on the host; metadata is uploaded by forward().
struct Batch {
    std::vector<int32_t> tok, row_slot, row_pos;      // per row
    std::vector<int32_t> slot, q0, qn, off;           // per sequence
    std::vector<int32_t> logit_rows;                  // rows whose logits are wanted
    void add_seq(int s, int offset, const int32_t* toks, int n);
    int rows() const { return (int)tok.size(); }
};

// Step-level metadata staging: the per-forward metadata (rows, sequences,
// logit rows, attention work list) of every forward of a speculative step is
// laid out in one host arena and uploaded with ONE copy before the step's
// first kernel, so the step's kernels form a single PDL chain (a host->device
// copy between kernels is a full stream barrier).
struct PreMeta {
    const int32_t* meta = nullptr;   // device: the forward's meta block
    const void* work = nullptr;      // device: stream-attention work list (nullptr: forward uploads its own)
    // device-planned forward (the device-resident decode loop, engine.cu):
    // the meta block and the work list are written on the device by the
    // step's plan kernel, so the host knows only the shapes.  The work list
    // holds n_seq regions of work_stride items (idle items pad a region);
    // every history is shorter than max_len.
    bool dev = false;
    int work_stride = 0, max_len = 0;
    // live rows of this forward (the active sequences come first): GEMM token
    // groups past m_act exit at once, the LM head stops at r_act logit rows
    const int32_t* m_act = nullptr;
    const int32_t* r_act = nullptr;
};
struct PreMetaOff {
    size_t meta = 0, work = 0;       // offsets into the arena (int32 units, 32-byte aligned)
    bool has_work = false;
};
// append forward(m, b)'s metadata to the host arena `h`.  safe[i]: sequence
// i's K/V rows below it were written before the upload (earlier steps) — the
// attention may load them before its dependency wait.
PreMetaOff forward_premeta(const bass_model& m, const Batch& b, int strategy, const std::vector<int32_t>& safe,
                           std::vector<int32_t>& h);
inline PreMeta premeta_at(const int32_t* dev_arena, const PreMetaOff& o) {
    return PreMeta{dev_arena + o.meta, o.has_work ? (const void*)(dev_arena + o.work) : nullptr};
}

// the forward's attention runs the persistent tcgen05 stream kernel (bf16 /
// int8 models, d_head 64 or 128): the precondition of device-planned forwards
bool model_uses_stream_attention(const bass_model& m);

// the model's lazily computed per-upload state (folded-LayerNorm constants),
// on the context stream; call before capturing forwards into a CUDA graph
void forward_prepare(bass_model& m);

// Run `b` through model m over cache kv; logits [logit_rows, V] fp32 -> logits_out (device).
// `pre`: metadata already on the device (forward_premeta + one upload).
void forward(bass_model& m, bass_kv& kv, const Batch& b, int strategy, float* logits_out,
             const int32_t* proposals, int pstride, const PreMeta* pre = nullptr);

// GEMM dispatch (SIMT or tcgen05) — Y = X W^T with a fused epilogue.
// `packed`: W is in the packed tile layout (packed_index) — the model's own
// weights; raw [N, K] pointers (bass_gemm) pass false.  `norm`: LayerNorm
// fused into X (tcgen05 path only; see TcNorm).
struct TcNorm;
void gemm(bass_model& m, int mode, const void* X, const void* W, int M, int N, int K,
          const Epi& e, bool packed, const TcNorm* norm = nullptr);

// tcgen05 GEMM (gemm_tc.cu); returns false when the shape is unsupported.
bool tc_gemm_supported(const bass_model& m, int N, int K);
// LayerNorm folded into a tcgen05 GEMM: X = bf16(x * g) (written by the
// previous residual epilogue / the embedding), row mean / rstd from the
// {sum, sum^2} per (128-column tile, row) they emitted, c = W g, e = W b.
struct TcNorm {
    const float* stats;
    const float* c;
    const float* e;
    float* kmean;      // row means (see forward()), updated by the consumer
    int stat_tiles;
};
// sx / sw (W8A8 models): per-token / per-channel scales; X, W int8 (W packed)
void tc_gemm(bass_model& m, int mode, const void* X, const void* W, int M, int N, int K,
             const Epi& e, bool packed, const TcNorm* norm = nullptr, const double* sx = nullptr,
             const double* sw = nullptr);
void tc_release(bass_model& m);
// per-model split-count override for one (N, K) projection shape (0: the default rule)
void tc_set_split(bass_model& m, int N, int K, int splits);
// pack n_mat contiguous [N, K] bf16 matrices into the packed layout (dst: n_mat * packed_rows(N) * K)
void pack_weights(cudaStream_t st, const void* src, void* dst, int N, int K, int n_mat);

// tcgen05 attention (attn_stream.cu).  A plan (work list + Q tensor map) is
// built once per forward and reused by every layer.
struct AttnPlan {
    bool valid = false;
    bool stream = false;                 // streaming flash-decoding kernel (attn_stream.cu)
    bool needs_combine = false;          // some row spans more than one 1024-key split
    int max_len = 0;                     // longest history + block (stream kernel: stage count choice)
    int max_q = 0;                       // longest block (new rows of one sequence)
    int NQ = 0, pad_len = 0, strategy = 0, H = 0, dh = 128, cap = 0, n_slots = 0, mc = 0, tmem_cols = 32;
    std::vector<int> first;
    void* work = nullptr;
    CUtensorMap tq;
};
bool tc_attention_supported(int dtype, int dh);
// streaming tcgen05 attention (attn_stream.cu): the default bf16 d_head=128 path
int stream_split_len();
void stream_attention_plan(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots,
                           const std::vector<int32_t>& slot, const std::vector<int32_t>& qn,
                           const std::vector<int32_t>& off, int H, int dh, int cap, DevBuf& work_buf,
                           AttnPlan& plan, const void* pre_work = nullptr);
// the stream attention's work list for a batch (what stream_attention_plan uploads)
void stream_attention_work(int strategy, const std::vector<int32_t>& slot, const std::vector<int32_t>& qn,
                           const std::vector<int32_t>& off, const std::vector<int32_t>& safe,
                           std::vector<int32_t>& w);
void stream_attention_run(bass_ctx* ctx, const AttnPlan& plan, const void* kc, const void* vc, const Seqs& seqs_dev,
                          float* part_o, float* part_ml, void* out);
// device-planned variant (PreMeta::dev): work list written on the device
void stream_attention_plan_dev(bass_ctx* ctx, int strategy, const void* q, int M, int n_slots,
                               const std::vector<int32_t>& qn, int H, int dh, int cap, const void* work,
                               int work_stride, int max_len, AttnPlan& plan);
// work-list geometry shared with the device planner: query-tile width for a
// block of q rows, 128-key chunk length, chunks per split, and the items one
// sequence of q rows needs when its history is shorter than max_len
int stream_nq_for(int q);
int stream_chunk_len();
int stream_split_chunks();
int stream_items_per_seq(int q, int max_len);
}  // namespace bass
