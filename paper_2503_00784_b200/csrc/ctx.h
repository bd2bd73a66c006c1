// dd_ctx: the target-role context behind the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/duodec_b200.h"
#include "gemm.h"
#include "model.h"
#include "pass.h"
#include "plant.h"
#include "tp.h"

namespace dd {

struct LayerW {
    __nv_bfloat16* qkv = nullptr;  // [q_dim + 2 kv_dim, d]
    __nv_bfloat16* o = nullptr;    // [d, q_dim]
    __nv_bfloat16* gu = nullptr;   // [2 ffn, d]  (gate rows, then up rows)
    __nv_bfloat16* dn = nullptr;   // [d, ffn]
    // all four stored pre-tiled (common.cuh tiled_offset) for 16 KiB bulk loads
};

constexpr int kPsRing = 32;  // pinned PassState staging: a 4K-token prefill enqueues without blocking

}  // namespace dd

struct dd_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    cudaEvent_t q_ready = nullptr;
    cudaEvent_t ps_done[dd::kPsRing] = {};
    dd::ModelDims m{};  // this rank's shard: local heads, FFN features, head (vocabulary) rows
    int vocab = 0;      // full vocabulary (tokens, logits, acceptance)
    // tensor parallelism (tp.h); tp_size 1 = unsharded
    int tp_rank = 0, tp_size = 1;
    int pass_ctas = 148;  // persistent pass kernel grid (148 / N when N TP ranks share one GPU)
    std::vector<int> tp_v0;        // vocabulary split, [tp_size + 1]
    void* tp_xbuf = nullptr;       // symmetric exchange buffer (flags | partials | local logits)
    dd::TpLayout tp_lay{};
    dd::TpPeers tp_peers{};        // every rank's exchange buffer (device pointers)
    bool tp_connected = false;
    std::vector<void*> tp_opened;  // IPC-opened peer buffers
    int max_seq = 0, page_size = 16, n_pages = 0;
    bool weights_ready = false, use_graphs = true;

    __nv_bfloat16* emb = nullptr;
    __nv_bfloat16* head = nullptr;
    std::vector<dd::LayerW> layers;
    float* gain_ones = nullptr;

    float* x = nullptr;             // [256, d] fp32 residual stream
    __nv_bfloat16* h = nullptr;     // [256, d] normed GEMM input
    float* q = nullptr;             // [256, q_dim] fp32 roped queries
    __nv_bfloat16* o = nullptr;     // [256, q_dim] attention output
    __nv_bfloat16* a = nullptr;     // [256, ffn] SwiGLU output
    float* ws = nullptr;            // split-K partials
    int* counters = nullptr;        // per-tile split arrival counters
    float* ss = nullptr;            // [256][d/128] deferred-RMSNorm sum-of-squares partials
    float* logits = nullptr;        // [256, vocab]
    CUtensorMap map_h, map_o, map_a;
    CUtensorMap map_h128, map_o128, map_a128;  // 128-row boxes (prefill GEMM)
    CUtensorMap map_kv;  // KV pool rows (head_dim 128), page_size-row boxes (prefill attention)
    bool has_map_kv = false;
    // fp32-accumulate mode (DD_PREC_FP32ACC): lo halves of the GEMM inputs and
    // an fp32 KV pool; every pass runs the per-launch path
    bool fp32acc = false;
    __nv_bfloat16 *h_lo = nullptr, *o_lo = nullptr, *a_lo = nullptr;
    CUtensorMap map_h_lo, map_o_lo, map_a_lo;
    float* kv_f32 = nullptr;
    int32_t* d_compact_dst = nullptr;  // dd_kv_compact destination slots
    dd::GemmPlan wide_plans[5] = {};
    float* ws_wide = nullptr;       // prefill GEMM stream-K partials

    __nv_bfloat16* kv_pool = nullptr;
    int32_t* page_table = nullptr;
    float* rope_cos = nullptr;
    float* rope_sin = nullptr;

    dd::PassState* d_ps = nullptr;
    dd::PassState* h_ps = nullptr;  // pinned ring
    int ps_slot = 0;

    double* row_m = nullptr;
    double* row_sum = nullptr;
    int* row_argmax = nullptr;
    unsigned* ticket = nullptr;
    dd_verify_out* d_out = nullptr;
    dd_verify_out* h_out = nullptr;      // mapped pinned: written by the acceptance kernel
    dd_verify_out* h_out_dev = nullptr;  // its device alias
    int verify_seq = 0;
    float* q_rows = nullptr;
    float* h_q_stage = nullptr;
    int q_rows_valid = 0;
    int32_t* d_tail = nullptr;
    double* d_probs = nullptr;
    size_t probs_cap = 0;

    // persistent pass kernel (pass.cu)
    bool use_pass_kernel = true;     // DD_PASS_KERNEL=0: one launch per GEMM / attention
    int epoch = 0;                   // pass sequence number (flag value)
    int* pass_flags = nullptr;       // [flags][kFlagReplicas] x 128-byte lines
    size_t pass_flag_count = 0;
    int* sk_prefix_d = nullptr;      // weighted stream-K partition by SM rank (or null)
    int* rank_of_smid_d = nullptr;
    int* attn_rank_d = nullptr;  // [pass_ctas] attention item order (pass.cu), rebuilt with the phase tables
    int attn_rank_ctas = 0;
    std::vector<int> sk_prefix_h;
    std::vector<int*> pass_begins;   // device begin tables of the phase tables
    float* pass_ws = nullptr;        // 2 x stream-K partials (alternating GEMM phases)
    int* pass_counters = nullptr;    // 2 x [512] segment arrival counters
    size_t pass_ws_half = 0;         // floats per half
    float* attn_part = nullptr;      // attention chunk-group partials
    int* attn_cnt = nullptr;
    std::map<int, dd::PassPhase*> pass_phases;  // key: w * 2 + want_logits (device arrays)
    std::map<int, int> pass_nphases;

    int n_cached = 0;
    int last_w = 0;  // width of the last scored pass with logits (0 = none)
    std::map<int, dd::GemmPlan> plans;
    std::map<int, cudaGraphExec_t> graphs;
    std::string err;
    // accounting for dd_engine_run
    uint64_t h2d_bytes = 0, d2h_bytes = 0, launches = 0;
    std::map<int, int> graph_kernels;  // kernels per captured pass graph
    cudaEvent_t t_start = nullptr, t_end = nullptr, t_first = nullptr;
};

// engine-side helpers (target.cu)
int ctx_mark(dd_ctx* ctx, int which);      // record start (0) / end (1) / first-iteration (2)
double ctx_elapsed_ms(dd_ctx* ctx, int which);  // start -> end (1) or first (2); syncs

int ctx_fail(dd_ctx* ctx, int code, const std::string& msg);
int run_pass(dd_ctx* ctx, const int32_t* tokens, int w, bool want_logits);
