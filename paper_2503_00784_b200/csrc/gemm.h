// Host interface of the skinny tcgen05 GEMM (see gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "model.h"

namespace dd {

// Epilogue applied by the last-arriving CTA of each 128-row tile after it has
// reduced the split-K partials in split order (deterministic).
enum GemmEpilogue {
    kEpiStore = 0,     // out[t][row] = y                      (LM-head logits, tests)
    kEpiResidual = 1,  // out[t][row] += y                     (o-proj, down-proj)
    kEpiSwiGLU = 2,    // rows interleaved in 64-blocks gate|up -> out_bf[t][f] = silu(g)*u
    kEpiQkvRope = 3,   // RoPE q/k, q -> q_out fp32, k/v -> paged bf16 KV cache
};

struct GemmEpiParams {
    int kind;
    int* counters;          // [tiles] zero-initialised; reset by the last CTA
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
};

struct GemmArgs {
    int n_out;         // weight rows (output features), multiple of 128
    int k;             // reduction length, multiple of 64
    int w;             // valid tokens (columns stored)
    int nt;            // padded token count: multiple of 16, <= 256
    int kb_per_split;  // 64-wide k-blocks per split
    int splits;
    int stages;        // smem ring depth
    float* ws;         // [splits][w][n_out] fp32 partial sums
    GemmEpiParams epi;
};

struct GemmPlan {
    int tiles;
    int splits;
    int kb_per_split;
    int stages;
    int smem_bytes;
};

// Row-major [rows, cols] bf16 tensor map with 64-column boxes, 128B swizzle.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_rows);

GemmPlan plan_gemm(int n_out, int k, int nt);

cudaError_t launch_gemm(const CUtensorMap* map_w, const CUtensorMap* map_x, int n_out, int k,
                        int w, int nt, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                        cudaStream_t stream);

}  // namespace dd
