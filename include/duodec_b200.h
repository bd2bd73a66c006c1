/*
 * duodec_b200.h — C ABI of the B200-native DuoDecoding target path.
 *
 * This is the drop-in seam below the reference's model/verifier contract
 * (reference = DuoDecoding C++ library under proj/ of arxiv 2503.00784).
 * Every entry point names the reference interface it replaces:
 *
 *   dd_prefill / dd_score   <- ModelSpec::forward / forward_scored
 *                              (proj/include/duodec/model.hpp:57-65) as used by
 *                              scored_with_next + target_step
 *                              (proj/src/engine.cpp:36-43, 145-157)
 *   dd_verify               <- verify_prefix / verify_bundle / sps_verify
 *                              (proj/include/duodec/verify.hpp:43-44, 53-54, 66-68;
 *                              proj/src/verify.cpp:41-107) plus the per-draw
 *                              RandomStream schedule (proj/include/duodec/random.hpp:16-26)
 *   dd_kv_truncate          <- the verified-prefix commit/truncate of
 *                              apply_verification (proj/src/engine.cpp:62-106)
 *   dd_time_pass            <- the target half of calibrate (proj/src/engine.cpp:534-578)
 *   dd_engine_run           <- run_vanilla / run_sps / run_duo
 *                              (proj/include/duodec/engine.hpp:102-116)
 *   dd_calibrate            <- calibrate + choose_budget (engine.hpp:118-126)
 *
 * Conventions: no exceptions cross this boundary; every int-returning call
 * returns 0 on success and a negative DD_E* code otherwise, with a message
 * available from dd_last_error().  A dd_ctx owns one CUDA stream on one GPU
 * and is not thread-safe: it is driven only from the target-role thread, as
 * the reference drives ModelSpec::forward only from the engine thread
 * (engine.cpp:458-478).  There is no CPU fallback: creating a context on a
 * machine without a Blackwell (sm_100) GPU fails with DD_E_CUDA.
 */
#ifndef DUODEC_B200_H
#define DUODEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DD_OK 0
#define DD_E_ARG (-1)      /* ConfigError / invalid argument            */
#define DD_E_CUDA (-2)     /* CUDA / driver failure (includes "no GPU") */
#define DD_E_STATE (-3)    /* call sequence violated (e.g. no pass yet) */
#define DD_E_CAPACITY (-4) /* KV cache or pass width exceeded           */

typedef struct dd_ctx dd_ctx;
typedef struct dd_draft dd_draft;

/* Llama-family shape (the target; the CPU draft uses the same struct). */
typedef struct dd_model_desc {
    int n_layers;
    int d_model;
    int n_heads;
    int n_kv_heads;
    int head_dim;
    int ffn_dim;
    int vocab;
    float rms_eps;    /* 1e-5 for Llama-2 */
    float rope_theta; /* 1e4 for Llama-2  */
    int max_seq;      /* KV capacity in tokens */
    int page_size;    /* tokens per KV page (0 -> 16) */
    int precision;    /* DD_PREC_*; target only (the CPU draft ignores it) */
} dd_model_desc;

/* Target arithmetic (north star: "per-position target logits match within a
 * stated bf16 tolerance (fp32-accumulate mode within 1e-4 relative)").
 * BF16: bf16 weights, activations and KV, fp32 accumulation (the fast path).
 * FP32ACC: activations carried as bf16 hi + lo pairs into two tcgen05 MMAs
 * per k-step (one TMEM accumulator), fp32 KV cache and fp32 attention; one
 * launch per GEMM / attention, tensor_parallel size 1, max_seq <= 49152. */
#define DD_PREC_BF16 0
#define DD_PREC_FP32ACC 1

/* Synthetic random-init weights with an optional planted shared bigram
 * (SURVEY.md §7 hard part 1): a fraction `alpha` of tokens t get the LM-head
 * row of pi(t) aligned with their embedding, in target and draft alike. */
typedef struct dd_plant_desc {
    uint64_t plant_seed; /* permutation pi and planted set                   */
    double alpha;        /* fraction of planted tokens (0 = pure random init) */
    float gain;          /* planted logit gain                                */
    float emb_std;       /* embedding std (0 -> 0.02)                         */
} dd_plant_desc;

/* ------------------------------------------------------------ target ctx */
int dd_ctx_create(const dd_model_desc* desc, int cuda_device, dd_ctx** out);
void dd_ctx_destroy(dd_ctx* ctx);
const char* dd_last_error(const dd_ctx* ctx); /* ctx may be NULL: global error */

/* Tensor parallelism (BASELINE config 5: 70B-shape TP=8; the
 * reference has no multi-GPU target, this replaces its single ModelSpec
 * forward with a Megatron-split one).  Rank tp_rank of tp_size holds
 * n_heads/tp_size q heads, n_kv_heads/tp_size kv heads, ffn_dim/tp_size FFN
 * features and a 128-row-aligned slice of the LM head; the embedding and the
 * residual stream are replicated.  dd_weights_init generates the rank's
 * slice of the same full model for any tp_size.  Before the first pass the
 * ranks connect their exchange buffers: one process per GPU exports a CUDA
 * IPC handle (dd_tp_export), gathers all tp_size handles in rank order over
 * the host (e.g. torch.distributed all_gather_object) and calls
 * dd_tp_connect; a single process driving every rank calls
 * dd_tp_connect_local.  Every rank must then issue the same sequence of
 * passes (dd_prefill / dd_score with the same widths): each pass ends with
 * the full logits on every rank and dd_verify runs redundantly with the same
 * seed and counter.  The CUDA-event timing helpers (dd_time_pass, ...) are
 * single-rank only. */
#define DD_TP_HANDLE_BYTES 64
int dd_ctx_create_tp(const dd_model_desc* desc, int cuda_device, int tp_rank, int tp_size,
                     dd_ctx** out);
int dd_tp_export(dd_ctx* ctx, void* ipc_handle /* DD_TP_HANDLE_BYTES */);
int dd_tp_connect(dd_ctx* ctx, const void* ipc_handles /* tp_size x DD_TP_HANDLE_BYTES */);
int dd_tp_connect_local(dd_ctx* const* ctxs, int n);

/* Generate all weights on the device from (weight_seed, plant); bit-identical
 * to the CPU oracle's generator (oracle/llama_ref.c). plant may be NULL. */
int dd_weights_init(dd_ctx* ctx, uint64_t weight_seed, const dd_plant_desc* plant);

/* Append n tokens to the KV cache without producing logits (chunked). */
int dd_prefill(dd_ctx* ctx, const int32_t* tokens, int n);

/* One scored pass: append w (<= 256) tokens at positions n_cached.. and
 * compute fp32 logits for all w rows (kept on the device).  Row i is the
 * target's next-token logits after tokens[i], i.e. forward_scored rows plus
 * the trailing p_next row of scored_with_next. */
int dd_score(dd_ctx* ctx, const int32_t* tokens, int w);

int dd_kv_len(const dd_ctx* ctx, int* n_cached);
/* Roll the cache back to n_valid tokens (KV rollback after a rejection). */
int dd_kv_truncate(dd_ctx* ctx, int n_valid);
/* In-place compaction (north star (c)): move cache slots src_pos[i] ->
 * dst_pos[i] for every layer, K and V, in one launch; dst strictly
 * increasing with dst <= src, n <= 256 (keeps an accepted branch contiguous
 * after its rejected siblings are dropped; the caller then truncates). */
int dd_kv_compact(dd_ctx* ctx, const int32_t* src_pos, const int32_t* dst_pos, int n);

/* Copy logits rows [row0, row0+rows) of the last pass to host memory. */
int dd_read_logits(dd_ctx* ctx, float* host, int row0, int rows);

/* Draft next-token distributions for the tail rows (fp32, rows x vocab). The
 * copy runs on a side stream and overlaps the next dd_score. */
int dd_upload_q(dd_ctx* ctx, const float* q_rows, int rows, int vocab);

#define DD_MODE_DUO 0     /* verify_prefix (tail) then verify_bundle          */
#define DD_MODE_SPS 1     /* sps_verify                                        */
#define DD_MODE_VANILLA 2 /* sample(p, next_uniform) — run_vanilla step        */

typedef struct dd_verify_args {
    int mode;
    int tail_len;       /* L: rows of the last pass tested against the tail  */
    int n_firsts;       /* s: bundle first tokens (duo)                      */
    int32_t firsts[16]; /* bundle first tokens in bundle order               */
    uint64_t seed;      /* verify RandomStream seed                          */
    uint64_t counter;   /* draws already consumed on entry                   */
    double temperature; /* > 0, used unless greedy                           */
    int greedy;         /* one-hot target at argmax (lowest id on ties)      */
    int q_onehot;       /* draft q rows are one-hot on the drafted tokens     */
} dd_verify_args;

typedef struct dd_verify_out {
    int prefix_all_accepted; /* duo: tail fully accepted (or empty)           */
    int reject_index;        /* duo/sps: first rejected position, -1 if none  */
    int resample;            /* duo: residual resample token                  */
    int bundle_accepted;     /* duo                                           */
    int seq_index;           /* duo: accepted bundle sequence                 */
    int fallback;            /* duo: token drawn when every sequence rejected */
    int sps_accepted;        /* sps: accepted draft length                    */
    int next_token;          /* sps: resample or bonus; vanilla: sampled token*/
    int n_draws;             /* uniforms consumed                              */
    int pad;                 /* internal: completion sequence of the result   */
    uint64_t counter_out;    /* counter + n_draws                              */
} dd_verify_out;

/* Fused logits -> softmax -> speculative-sampling acceptance on the last
 * L+1 rows of the last pass (tail tokens = last L tokens of that pass). */
int dd_verify(dd_ctx* ctx, const dd_verify_args* args, dd_verify_out* out);

/* Same acceptance kernel fed with host fp64 probability rows (L+1 x vocab) and
 * explicit tail tokens instead of logits — the path used to run the
 * reference's Markov-table models through the GPU verifier. */
int dd_verify_probs(dd_ctx* ctx, const double* p_rows, const int32_t* tail_tokens,
                    int vocab, const dd_verify_args* args, dd_verify_out* out);

/* Median device time (CUDA events) of a scored pass of width w. */
int dd_time_pass(dd_ctx* ctx, int w, int trials, float* median_ms);

/* Per-kernel device time breakdown of one pass of width w on the per-launch
 * path (ms, by class: 0 gemm, 1 attention, 2 epilogues/norms, 3 total). */
int dd_profile_pass(dd_ctx* ctx, int w, float* ms4);

/* Device time of the per-launch path's GEMM launches of one pass of width w
 * (4 per layer plus the LM head, back to back, fused epilogues included),
 * median of `trials`. */
int dd_time_gemms(dd_ctx* ctx, int w, int trials, float* median_ms, int* launches);

/* Weighted stream-K partition of the persistent pass kernel: times every SM's
 * weight streaming over a few decode passes and gives each SM a share
 * proportional to its speed (opt-in: DD_PASS_BALANCE=1 runs it from
 * dd_weights_init). Must precede the first scored pass. */
int dd_pass_balance(dd_ctx* ctx);

/* Algorithmic weight bytes streamed by one pass (excludes the gathered
 * embedding), for the roofline. */
uint64_t dd_pass_weight_bytes(const dd_ctx* ctx);

/* ------------------------------------------------------------ test seams */
/* Raw bf16 bits of a generated weight tensor (which: 0 embedding, 1 LM head,
 * 2 fused qkv, 3 o-proj, 4 fused gate/up, 5 down) for bit-exact checks
 * against the oracle generator. n = element count expected. */
int dd_read_weights(dd_ctx* ctx, int which, int layer, uint16_t* host, size_t n);
/* Standalone run of the skinny tcgen05 GEMM: Y[w][n_out] = X[w][k] . W[n_out][k]^T
 * (bf16 bits in, fp32 out; n_out % 128 == 0, k % 64 == 0, w <= 256). */
int dd_test_gemm(const uint16_t* W, const uint16_t* X, int n_out, int k, int w, float* Y);

/* Debug: per-CTA globaltimer timeline (8 u64 per CTA: start, setup, first
 * stage, last MMA issued, accumulator done, end, -, smid) of one launch of
 * layer-0 GEMM `which` (0 qkv, 1 o, 2 gate/up, 3 down, 4 LM head). */
int dd_debug_gemm_trace(dd_ctx* ctx, int which, int w, uint64_t* trace, int max_ctas,
                        int* n_ctas);

/* Debug: per-CTA stamps of every GEMM launch of one pass sequence (stride =
 * 8 * ctas_per_launch u64 per launch). */
int dd_debug_pass_trace(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_launch,
                        int* ctas_per_launch);

/* Debug: one decode pass (w <= 16) of the persistent pass kernel with per-CTA,
 * per-phase globaltimer stamps, trace[cta][phase][12] (weight producer start,
 * inputs ready, MMA done, epilogue done, ..., last flag published, ...,
 * smid in slot 10 of phase 0), followed when max_entries allows by per-tile
 * publish times; n_phases = embed + 5 per layer + head. */
int dd_debug_pass_timeline(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_phases);

/* Debug: one prefill pass (49..128 tokens) with per-CTA stamps of its
 * tokens-on-M GEMM launches, trace[launch][148][8]. */
int dd_debug_prefill_trace(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_launch);

/* Debug: mapped host int[148][8] of per-CTA progress words of the pass kernel
 * (hang diagnosis; pointer stays valid for the process). */
void* dd_debug_pass_progress(void);

/* ------------------------------------------------------------ CPU draft */
int dd_draft_create(const dd_model_desc* desc, uint64_t weight_seed, const dd_plant_desc* plant,
                    int n_threads, const int* cpus, int n_cpus, dd_draft** out);
void dd_draft_destroy(dd_draft* d);
/* Next-token logits (fp32, vocab) after the given context (KV reused). */
int dd_draft_logits(dd_draft* d, const int32_t* ctx_tokens, int n, float* logits);
/* Median wall time of one single-token draft forward (calibrate denominator). */
int dd_draft_time_token(dd_draft* d, int trials, float* median_ms);
/* The draft's q(. | ctx) (fp32, vocab) with the temperature / greedy rule
 * applied (one-hot at the lowest-id argmax when greedy); returns the argmax
 * in *argmax.  Test seam for the drafting parity tests. */
int dd_draft_dist(dd_draft* d, const int32_t* ctx_tokens, int n, double temperature, int greedy,
                  float* q, int* argmax);
/* draft_dynamic (proj/src/drafting.cpp:71-136) as run by the engine's draft
 * worker: sequences are written back to back into tokens (capacity budget),
 * their lengths into seq_len (capacity max_sequences); *counter is the draft
 * RandomStream counter, advanced in place.  Test seam (bit-exact against the
 * reference's drafting). */
int dd_draft_dynamic(dd_draft* d, const int32_t* ctx_tokens, int n, int budget,
                     int max_sequences, double temperature, int greedy, uint64_t seed,
                     uint64_t* counter, int32_t* tokens, int32_t* seq_len, int* n_seqs,
                     double* threshold, int* forwards);

/* ------------------------------------------------------------ engine */
#define DD_BUDGET_FIXED 0
#define DD_BUDGET_CALIBRATED 1

typedef struct dd_engine_config { /* EngineConfig (engine.hpp:43-60) */
    int mode;           /* DD_MODE_*                                           */
    int budget;         /* gamma                                               */
    int max_sequences;  /* s_max                                               */
    int max_new_tokens; /* L                                                   */
    double temperature; /* > 0; ignored when greedy                            */
    int greedy;         /* one-hot target and draft (argmax, lowest-id ties)   */
    uint64_t draft_seed;
    uint64_t verify_seed;
    int budget_policy;  /* DD_BUDGET_*                                         */
    int budget_hard_cap;
    int calib_probe_len;
    int calib_trials;
    int threaded;       /* DuoExecution::threaded (1) / sequential (0)         */
    /* WorkerHooks (engine.hpp:36-41, engine.cpp:430-432, 455-466): when
     * jitter_max_us > 0, sleep a pseudo-random 0..jitter_max_us microseconds
     * (splitmix64 of jitter_seed, iteration and role) before each draft step
     * and each target step -- the determinism tests' scheduling jitter. */
    uint64_t jitter_seed;
    int jitter_max_us;
} dd_engine_config;

typedef struct dd_iteration_record { /* IterationRecord (engine.hpp:62-70) */
    double draft_ms;
    double target_ms;
    double verify_ms;
    double comm_ms;
    int tokens_processed;
    int sequence_count;
    int accepted;
    int width; /* scored-pass width W = 1 + tail */
} dd_iteration_record;

typedef struct dd_generation_result { /* GenerationResult (engine.hpp:72-78) */
    int32_t* tokens;    /* caller buffer, capacity max_tokens              */
    int max_tokens;
    int n_tokens;
    dd_iteration_record* iterations; /* caller buffer, capacity max_iterations */
    int max_iterations;
    int n_iterations;
    double ttft_ms;
    double total_ms;
    double tps;
    double prefill_ms;
    int budget_used;
    double device_ms;      /* CUDA-event time on the target stream, start->end */
    uint64_t h2d_bytes;    /* host->device bytes copied during the run        */
    uint64_t d2h_bytes;    /* device->host bytes copied during the run        */
    uint64_t gpu_launches; /* kernels launched (graph nodes counted)          */
    double device_ttft_ms; /* CUDA-event time start -> end of iteration 1     */
} dd_generation_result;

/* Run one generation: target on the GPU (ctx), draft on host cores (draft,
 * may be NULL for vanilla).  prompt is a host buffer. */
int dd_engine_run(dd_ctx* ctx, dd_draft* draft, const dd_engine_config* cfg,
                  const int32_t* prompt, int n_prompt, dd_generation_result* out);
/* The same generation on a connected tensor-parallel group driven by one
 * process (ctxs[r] is rank r): every pass is issued to all ranks, acceptance
 * runs on rank 0, rollback on all.  Needs a fixed budget policy. */
int dd_engine_run_tp(dd_ctx* const* ctxs, int n, dd_draft* draft, const dd_engine_config* cfg,
                     const int32_t* prompt, int n_prompt, dd_generation_result* out);

/* calibrate(): median GPU scored pass at probe_len over median CPU draft
 * token; *budget = choose_budget(c) capped at hard_cap. */
int dd_calibrate(dd_ctx* ctx, dd_draft* draft, int probe_len, int trials, int hard_cap,
                 double* cost_coefficient, int* budget);

#ifdef __cplusplus
}
#endif

#endif /* DUODEC_B200_H */
