// Host interface of the skinny tcgen05 weight-streaming GEMM (see gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "model.h"

namespace dd {

// Epilogue applied once per 128-row tile to the fully reduced fp32 result.
enum GemmEpilogue {
    kEpiStore = 0,     // out[t][row] = y                      (LM-head logits, tests)
    kEpiResidual = 1,  // out[t][row] += y                     (o-proj, down-proj)
    kEpiSwiGLU = 2,    // rows interleaved in 64-blocks gate|up -> out_bf[t][f] = silu(g)*u
    kEpiQkvRope = 3,   // RoPE q/k, q -> q_out fp32, k/v -> paged bf16 KV cache
};

struct GemmEpiParams {
    int kind;
    int* counters;          // [tiles] zero-initialised; reset by the last segment
    float* out;             // kEpiStore / kEpiResidual: [w][n_out]
    __nv_bfloat16* out_bf;  // kEpiSwiGLU: [w][n_out / 2]
    const PassState* ps;    // kEpiQkvRope
    const float* rope_cos;
    const float* rope_sin;
    float* q_out;
    __nv_bfloat16* kv_pool;
    const int32_t* page_table;
    int page_size, layer;
    ModelDims m;
    // Deferred RMSNorm.  W.(x*r*g) == r * (W.(x*g)) with r = rsqrt(mean(x^2)+eps),
    // so a residual-producing GEMM writes u = bf16(x*g) and, per token, the sum of
    // squares of its 128 updated rows (ss_out[t][tile]); the consuming GEMM sums
    // those partials in tile order, forms r per token and scales its fp32
    // accumulator before its own epilogue.  No normalisation kernel or pass.
    __nv_bfloat16* u_out;  // kEpiResidual: [w][n_out] bf16(x * gain), or nullptr
    const float* gain;     // [n_out] RMSNorm gain
    float* ss_out;         // kEpiResidual: [w][tiles]
    const float* ss_in;    // consumer: [w][ss_tiles] partials, or nullptr (no scale)
    int ss_tiles;
    float eps;
    int norm_d;            // d of the normalised row
    // fp32-accumulate mode (DD_PREC_FP32ACC): the consumer GEMM reads its
    // activations as bf16 hi + lo pairs (two MMAs into one accumulator), so
    // producers also write lo = bf16(v - hi); K / V go to an fp32 cache.
    __nv_bfloat16* lo_out; // kEpiResidual: u_lo; kEpiSwiGLU: a_lo; or nullptr
    float* kv_f32;         // kEpiQkvRope: fp32 KV pool (same addressing), or nullptr
};

struct GemmArgs {
    int n_out;      // weight rows (output features), multiple of 128
    int k;          // reduction length, multiple of 64
    int w;          // valid tokens
    int nt;         // padded token count: multiple of 16, <= 256
    int tiles;      // n_out / 128
    int nkb;        // k / 64
    int stages;     // smem ring depth
    int max_seg;    // max stream-K segments per tile (workspace stride)
    int tmem_buf;   // TMEM columns per accumulator buffer (2 buffers)
    int prefetch;   // L2 prefetch distance in k-blocks beyond the ring
    int interleave; // timing experiment: lockstep-sequential weight addresses
    int split;      // 1: activations are hi + lo bf16 pairs (fp32-accumulate mode)
    float* ws;      // [tiles][max_seg][w][128] fp32 segment partials
    GemmEpiParams epi;
    unsigned long long* trace;  // debug: 8 globaltimer stamps per CTA, or nullptr
};

struct GemmPlan {
    int tiles, nkb;
    int ctas;        // persistent CTAs (one per SM)
    int stages;
    int max_seg;
    int tmem_cols;   // allocation (2 buffers)
    int smem_bytes;
};

// Row-major [rows, cols] bf16 tensor map with 64-column boxes, 128B swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_rows);

// split: fp32-accumulate mode (two activation boxes per stage)
GemmPlan plan_gemm(int n_out, int k, int nt, int split = 0);

// workspace floats needed by a plan at width w
size_t gemm_ws_floats(const GemmPlan& p, int w);

// debug seam: per-CTA timeline of one launch (see dd_debug_gemm_trace)
void gemm_set_trace(unsigned long long* buf);

// w_tiled: weights in the pre-tiled layout of common.cuh (tiled_offset).
// Launched with programmatic dependent launch: the kernel streams its first
// weight stages before waiting on the previous kernel in the stream.
// map_x_lo (fp32-accumulate mode only): the lo halves of the activations;
// the plan must have been made with split = 1.
cudaError_t launch_gemm(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x, int n_out, int k,
                        int w, int nt, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                        cudaStream_t stream, const CUtensorMap* map_x_lo = nullptr);

// Prefill GEMM (gemm_wide.cu): tokens on M (<= 128, one TMEM lane each),
// 256 weight rows on N; map_x128 has 128-row boxes.  n_out % 256 == 0.
GemmPlan plan_gemm_wide(int n_out, int k, int sm_avail = 148 /* kNumSMs */);
size_t gemm_wide_ws_floats(const GemmPlan& p);
// debug seam: per-CTA stamps of every following wide launch at buf + launch * 8 * 148
void gemm_wide_set_trace(unsigned long long* buf);
cudaError_t launch_gemm_wide(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x128, int n_out, int k,
                             int w, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                             cudaStream_t stream);

// Multi-tile prefill GEMM (gemm_wide.cu): w <= kMaxPrefillTokens tokens in
// 128-token tiles x 256-row weight tiles, full K per unit (no stream-K).
cudaError_t launch_gemm_prefill(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x128, int n_out, int k,
                                int w, const GemmEpiParams& epi, cudaStream_t stream);

}  // namespace dd
