/*
 * bass.h — C ABI of the B200-native BASS hot path (libbass.so).
 *
 * Drop-in boundary.  The reference (a pure-Python package, `batchspec`)
 * has no FFI; its hot path is reached through Python objects.  Each entry
 * point below replaces one reference interface, cited as ref:<file>:<line>
 * under /root/reference/pkg/src/batchspec/.  The Python package
 * `paper_2404_15778_b200` binds these with ctypes and re-exposes the
 * reference's Python API.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types;
 *   - every function returns BASS_OK (0) or a negative error class; the
 *     message is available from bass_last_error(ctx);
 *   - "host" arrays are read synchronously; "dev" pointers are device
 *     memory on the context's device;
 *   - all work is enqueued on the context's stream; a context is not
 *     thread-safe (one context per GPU per process, ref SPEC.md:96).
 */
#ifndef BASS_H
#define BASS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BASS_OK            0
#define BASS_ERR_VALUE    -1   /* maps to the reference's ValueError        */
#define BASS_ERR_CUDA     -2
#define BASS_ERR_MEMORY   -3
#define BASS_ERR_STATE    -4

/* weight/activation dtype.  BASS_INT8: W8A8 — the reference's quantized
 * inference path (ref:quant.py:55-129, model.py:135-143, 160-164, 219-222):
 * int8 per-output-channel weights, per-token int8 activations into every
 * linear layer, int8 x int8 -> s32 tensor-core GEMMs dequantized in the
 * epilogue, q/k/v fake-quantized per (token, head); embeddings, residual
 * stream, attention and KV cache as in the bf16 path. */
enum { BASS_BF16 = 0, BASS_F32 = 1, BASS_INT8 = 2 };
enum { BASS_PAD = 0, BASS_SPLIT = 1, BASS_RAGGED = 2 };  /* ref:attention.py:30-32 (+ragged work list) */
/* decode-loop driver of bass_spec_generate: DEVICE (default) runs every step
 * after the first (prompt) step from one CUDA graph — the step planning,
 * bookkeeping and Algorithm 1 on the GPU, one host synchronisation per
 * generation; HOST plans each step on the host and reads its outcome back
 * (one synchronisation per step).  Both give identical results.  DEVICE falls
 * back to HOST where it does not apply (fp32 models, d_head outside {64, 128},
 * draft limit > 48, timeline tracing or per-kernel event profiling on). */
enum { BASS_LOOP_HOST = 0, BASS_LOOP_DEVICE = 1 };
enum { BASS_GEMM_AUTO = 0, BASS_GEMM_SIMT = 1, BASS_GEMM_TC = 2 };
enum { BASS_ROLE_DRAFT = 0, BASS_ROLE_VERIFY = 1 };      /* ref:sampling.py:20-22 */

typedef struct bass_ctx bass_ctx;
typedef struct bass_model bass_model;
typedef struct bass_kv bass_kv;
typedef struct bass_engine bass_engine;

/* ref:model.py:36-62 ModelConfig */
typedef struct {
    int32_t n_layer, n_head, d_model, d_head, vocab_size, max_seq_len;
} bass_geometry;

/* tensor ids for bass_model_set_weight (ref:model.py:73-95) */
enum {
    BASS_W_TOK_EMB = 0, BASS_W_POS_EMB, BASS_W_LN1_G, BASS_W_LN1_B,
    BASS_W_WQ, BASS_W_WK, BASS_W_WV, BASS_W_WO, BASS_W_LN2_G, BASS_W_LN2_B,
    BASS_W_FC, BASS_W_PROJ, BASS_W_LNF_G, BASS_W_LNF_B, BASS_W_HEAD
};

int         bass_version(void);
int         bass_device_arch(int device);              /* e.g. 100 for sm_100 */
int         bass_ctx_create(int device, bass_ctx** out);
int         bass_ctx_destroy(bass_ctx* ctx);
int         bass_ctx_set_stream(bass_ctx* ctx, void* cuda_stream);
int         bass_ctx_sync(bass_ctx* ctx);
const char* bass_last_error(const bass_ctx* ctx);
/* number of kernels this context has launched so far (for gpu_launches) */
int64_t     bass_ctx_launches(const bass_ctx* ctx);
/* host<->device bytes this context has copied (per-step metadata, results) */
int         bass_ctx_transfer_bytes(const bass_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* per-kernel-class device timing with CUDA events on the context stream:
 * class 0 GEMM, 1 attention, 2 norm/embed, 3 sampling/accept.  enable resets
 * the counters; read returns launches, total ms, algorithmic bytes, flops. */
int         bass_ctx_profile(bass_ctx* ctx, int enable);
int         bass_ctx_profile_read(bass_ctx* ctx, int cls, int64_t* launches,
                                  double* ms, double* bytes, double* flops);
/* cumulative algorithmic work of every launch of a class since the context
 * was created (no events, no overhead): launches, bytes, flops.  The bench's
 * roofline divides these by the traced in-chain kernel time. */
int         bass_ctx_algo_read(bass_ctx* ctx, int cls, int64_t* launches,
                               double* bytes, double* flops);

/* Model weights live in device memory owned by the model.
 * Replaces ModelWeights/init_model (ref:model.py:87-132). */
int bass_model_create(bass_ctx* ctx, const bass_geometry* g, int dtype,
                      bass_model** out);
int bass_model_destroy(bass_model* m);
/* host fp32 values in the REFERENCE layout (input-major [in,out] for
 * matrices, ref:model.py:160-164); converted to dtype and stored
 * output-major on device.  n must equal the tensor's element count. */
int bass_model_set_weight(bass_model* m, int tensor, int layer,
                          const float* host, int64_t n);
/* the inverse: one tensor back to host fp32 in the reference layout (the
 * device values, e.g. bf16-rounded) — checkpoint save (ref:checkpoint.py:65-79) */
int bass_model_get_weight(const bass_model* m, int tensor, int layer,
                          float* host, int64_t n);
/* device-side N(0, std) init for benchmark-scale models (ref init is
 * N(0,0.02) on the fp32 grid, ref:model.py:106-132); LN gains 1, biases 0 */
int bass_model_init_random(bass_model* m, uint64_t seed, float std);
/* BASS_INT8 models: the quantized payload of one matrix in the reference
 * layout ([in, out] int8, ref:quant.py:55-63 QuantTensor.payload) and its
 * per-output-channel scales ([out] fp64, QuantTensor.scales). */
int bass_model_get_qweight(const bass_model* m, int tensor, int layer,
                           int8_t* payload_host, double* scales_host, int64_t n);
int bass_model_set_gemm(bass_model* m, int gemm_mode);
/* split-K count of the tcgen05 GEMM for one (N, K) projection shape of this
 * model (1..8; 0 restores the default rule of gemm_tc.cu choose_splits).
 * Splits are a function of the shape only, never of M (row bits stay
 * batch-invariant); this is the per-model tuning hook. */
int bass_model_set_split(bass_model* m, int N, int K, int splits);
int64_t bass_model_weight_bytes(const bass_model* m);

/* Ragged KV cache: per (layer, slot, head) contiguous [capacity, d_head]
 * rows; lengths are per slot.  Replaces RaggedKvCache (ref:kv_cache.py:23-128). */
int bass_kv_create(bass_model* m, int n_slots, int capacity, bass_kv** out);
int bass_kv_destroy(bass_kv* kv);
int bass_kv_lengths(const bass_kv* kv, int32_t* out_host);         /* ref:kv_cache.py:118-120 */
int bass_kv_truncate(bass_kv* kv, int n, const int32_t* slots_host,
                     const int32_t* lens_host);                    /* ref:kv_cache.py:93-104 */

/* One ragged forward: ref:model.py:177-246 forward_block.
 * Sequence i extends slot slots[i] with tokens[cu_q[i] .. cu_q[i+1]).
 * rows_mode 0: logits for every new row ([cu_q[n], V]);
 * rows_mode 1: logits for the last row of each sequence ([n, V]).
 * logits_host: fp32 host buffer, written before return. */
int bass_forward_ragged(bass_model* m, bass_kv* kv, int n_seq,
                        const int32_t* slots_host, const int32_t* cu_q_host,
                        const int32_t* tokens_host, int strategy,
                        int rows_mode, float* logits_host);

/* Standalone projection GEMM with the forward's kernels (tests / microbench):
 * Y[M, N] (fp32) = X[M, K] . W[N, K]^T with X, W in the model's dtype, all
 * device pointers; gemm_mode BASS_GEMM_SIMT, BASS_GEMM_TC (tcgen05 on the raw
 * [N, K] weights) or 3 (tcgen05 on a copy repacked into the model's packed
 * tile layout — the forward's own path, incl. the serial split-K kernel for
 * M > 256).  ref:model.py:160-164 (_linear), output-major weights. */
int bass_gemm(bass_model* m, int gemm_mode, int M, int N, int K,
              const void* x_dev, const void* w_dev, float* y_dev);
/* Integer-accumulate GEMM with the fused dequantizing epilogue
 * (ref:quant.py:98-123 int_gemm_dequant, without bias / residual):
 * out[t, c] = (sum_i a[t, i] w[i, c]) * sa[t] * sw[c] on the tcgen05
 * kind::i8 path.  Host arrays: a [M, K] int8 (per-token payload), sa [M],
 * w [K, N] int8 in the reference layout (per-channel payload), sw [N];
 * out [M, N] fp32.  K % 128 == 0, N >= 128. */
int bass_int_gemm_dequant(bass_ctx* ctx, int M, int N, int K,
                          const int8_t* a_host, const double* sa_host,
                          const int8_t* w_host, const double* sw_host,
                          float* out_host);

/* microbenchmark: `reps` back-to-back launches; launch i uses weight copy
 * i % n_w (w_dev holds n_w contiguous [N, K] copies); device time per launch
 * from CUDA events on the context stream.  gemm_mode 3: tcgen05 on copies
 * repacked into the packed tile layout bf16 models use for their weights. */
int bass_gemm_bench(bass_model* m, int gemm_mode, int M, int N, int K,
                    const void* x_dev, const void* w_dev, float* y_dev,
                    int reps, int n_w, double* ms_per_launch);

/* Standalone ragged attention (ref:attention.py:140-154 attend), for the
 * C4 sweep and kernel parity.  Layouts (device, dtype = BASS_BF16|F32):
 *   q, out : [cu_q[n], n_head, d_head]
 *   k, v   : [n_seq, n_head, kv_stride, d_head]  (sequence i uses entry i)
 * sequence i has cu_q[i+1]-cu_q[i] queries at positions offsets[i]+t and
 * attends keys [0, offsets[i]+t]. */
int bass_attention(bass_ctx* ctx, int strategy, int dtype, int n_seq,
                   int n_head, int d_head, const int32_t* cu_q_host,
                   const int32_t* offsets_host, const void* q_dev,
                   const void* k_dev, const void* v_dev, int kv_stride,
                   void* out_dev);

/* microbenchmark of the bf16 tcgen05 attention (d_head 64 or 128) as the
 * forward runs it: one plan, then `reps` back-to-back launches (+ split
 * combine); launch i reads K/V copy i % n_kv (k_dev / v_dev hold n_kv
 * contiguous [n_seq, n_head, kv_stride, d_head] copies, so > L2 defeats
 * caching).  Device time per call from CUDA events on the context stream. */
int bass_attention_bench(bass_ctx* ctx, int strategy, int n_seq, int n_head, int d_head,
                         const int32_t* cu_q_host, const int32_t* offsets_host,
                         const void* q_dev, const void* k_dev, const void* v_dev,
                         int kv_stride, int n_kv, void* out_dev, int reps,
                         double* ms_per_call);

/* Timeline trace (diagnostics): with `records` > 0, every CTA of the
 * GEMM / attention / LayerNorm launches that follow writes one record
 * {t_start_ns, t_end_ns, smid, tag} (globaltimer) until the buffer is full;
 * 0 disables.  bass_trace_read copies the records out and rewinds. */
int bass_trace_enable(bass_ctx* ctx, int64_t records);
int bass_trace_read(bass_ctx* ctx, uint64_t* host, int64_t max_records, int64_t* n_out);

/* Device RNG parity: uniforms u[2i], u[2i+1] = first two draws of
 * default_rng(SeedSequence((seed, sid[i], role[i], ctr[i]))).random()
 * (ref:sampling.py:53-66).  Host arrays in, host array out. */
int bass_rng_uniforms(bass_ctx* ctx, int n, uint64_t seed,
                      const int64_t* sid, const int32_t* role,
                      const int64_t* ctr, double* out_host);

/* Shaping + inverse-CDF sampling on device (ref:sampling.py:69-115):
 * rows of fp32 logits (host), one uniform per row (host); writes the
 * sampled token per row and (optionally) the shaped probabilities. */
int bass_shape_sample(bass_ctx* ctx, int n_rows, int vocab,
                      const float* logits_host, double temperature,
                      double top_p, const double* u_host,
                      int32_t* tok_out_host, double* probs_out_host);

/* Accept / resample (ref:sampling.py:118-146) for n independent cases:
 * q_logits/p_logits [n, V] fp32 (host), draft tokens, keys for the
 * VERIFY-role generator.  Writes accepted (0/1) and corrected token
 * (-1 when accepted). */
int bass_accept(bass_ctx* ctx, int n, int vocab, const float* q_logits_host,
                const float* p_logits_host, double temperature, double top_p,
                const int32_t* tok_host, uint64_t seed, const int64_t* sid_host,
                const int64_t* ctr_host, int32_t* accepted_out,
                int32_t* corrected_out);

/* ---------------- device-resident decode (ref:engine.py:120-385) -------- */

typedef struct {
    int32_t  batch;
    const int32_t* prompt_tokens;      /* concatenated prompts             */
    const int32_t* prompt_offsets;     /* [batch+1]                         */
    int32_t  max_new_tokens;
    double   temperature, top_p;
    int32_t  eos_token;                /* -1: none                          */
    uint64_t seed;
    const int64_t* sequence_ids;       /* [batch]; NULL -> slot index       */
    /* draft-length controller (ref:draft_control.py:17-108) */
    int32_t  ctl_fixed;                /* 0 adaptive (Algorithm 1), else fixed length */
    int32_t  l0, incre, mod, limit;    /* l0 = current l_draft of the controller       */
    int32_t  s0;                       /* current shrink flag s of the controller      */
    /* benchmark harness: draft proposals overridden per (sid, pos) by a keyed
     * hash — the main model's greedy token (align_tokens, [batch, max_new])
     * with probability align, else a hash token.  align < 0 disables. */
    double   align;
    uint64_t align_seed;
    const int32_t* align_tokens;
} bass_gen_request;

typedef struct {
    int32_t* tokens;          /* [batch, max_new_tokens]                      */
    double*  logprobs;        /* [batch, max_new_tokens]                      */
    int32_t* n_tokens;        /* [batch]                                      */
    int32_t* finish_reason;   /* [batch] 0 eos, 1 length                      */
    int32_t* completion_step; /* [batch]                                      */
    double*  finish_wall_s;   /* [batch] seconds since call start             */
    int32_t  max_steps;       /* capacity of the trace arrays                 */
    int32_t  n_steps;
    int32_t* step_draft_len;  /* [max_steps]                                  */
    int32_t* step_accepted;   /* [max_steps, batch], -1 for inactive slots    */
    int32_t* step_emitted;    /* [max_steps, batch] emitted count, -1 inactive */
    int32_t* step_kv_len;     /* [max_steps, batch] committed length           */
    double*  step_wall_s;     /* [max_steps]                                   */
    int64_t  main_forward_calls, draft_forward_calls;
    double   wall_s;
    int32_t  final_l_draft, final_s;
    double   host_enqueue_s;  /* host time spent building/launching steps      */
    double   sync_wait_s;     /* host time blocked on the per-step read-back    */
} bass_gen_result;

/* The engine drives the providers' own caches (main_kv / draft_kv), as the
 * reference's decode loop mutates its providers' caches (ref:engine.py:358-360).
 * draft_model/draft_kv may be NULL for regular decoding only. */
int bass_engine_create(bass_model* main_model, bass_kv* main_kv,
                       bass_model* draft_model, bass_kv* draft_kv,
                       bass_engine** out);
int bass_engine_destroy(bass_engine* e);
int bass_engine_set_strategy(bass_engine* e, int strategy);
int bass_engine_set_loop(bass_engine* e, int loop_mode);
/* how the last bass_spec_generate ran: BASS_LOOP_HOST / DEVICE, its host
 * synchronisations, and how many times this engine captured a loop graph */
int bass_engine_loop_info(const bass_engine* e, int32_t* last_mode, int32_t* last_syncs,
                          int64_t* graph_builds);
int bass_spec_generate(bass_engine* e, const bass_gen_request* req,
                       bass_gen_result* res);        /* ref:engine.py:200-385 */
int bass_regular_generate(bass_engine* e, const bass_gen_request* req,
                          bass_gen_result* res);     /* ref:engine.py:120-197 */

#ifdef __cplusplus
}
#endif
#endif /* BASS_H */
