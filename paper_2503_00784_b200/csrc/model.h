// Target model description, synthetic-weight recipe and the device-side
// kernels of one verification pass (see model.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/duodec_b200.h"

namespace dd {

// Tensor ids fed to derive_seed(weight_seed, id) for every generated matrix;
// the CPU oracle (oracle/llama_ref.c) uses the same table.
enum TensorKind { kWq = 0, kWk = 1, kWv = 2, kWo = 3, kWg = 4, kWu = 5, kWd = 6 };
constexpr uint64_t kTensorEmb = 0;
constexpr uint64_t kTensorHead = 1;
__host__ __device__ inline uint64_t tensor_id(int layer, int kind) {
    return 2 + static_cast<uint64_t>(layer) * 8 + static_cast<uint64_t>(kind);
}

struct ModelDims {
    int n_layers, d, n_heads, n_kv_heads, head_dim, ffn, vocab;
    float eps, rope_theta;
    __host__ __device__ int q_dim() const { return n_heads * head_dim; }
    __host__ __device__ int kv_dim() const { return n_kv_heads * head_dim; }
    __host__ __device__ int qkv_rows() const { return q_dim() + 2 * kv_dim(); }
};

// Per-pass state shared by every kernel of a pass (device memory, updated by a
// single small H2D copy before each pass so captured graphs stay valid).
constexpr int kMaxPassTokens = 256;      // scored passes (logits rows)
constexpr int kPrefillChunk = 128;       // prompt chunking of tensor-parallel / fp32acc contexts
constexpr int kMaxPrefillTokens = 2048;  // one prefill pass (gemm_prefill_kernel): weights streamed once
struct PassState {
    int n_cached;  // tokens already in the KV cache (absolute position of row 0)
    int w;         // tokens in this pass
    int epoch;     // pass sequence number (dataflow flags of the persistent pass kernel)
    int pad;
    int32_t tokens[kMaxPrefillTokens];  // only the first w are uploaded
};

// ---------------------------------------------------------------- kernels
// Which block of the full generated tensor a (sharded) matrix holds: logical
// element (row0 + r) * cols + col0 + c (cols == 0: the block's own width).
struct SrcWindow {
    uint64_t row0 = 0, col0 = 0, cols = 0;
};
// row0: first physical row; tiled: write the pre-tiled GEMM layout (common.cuh)
void launch_init_matrix(__nv_bfloat16* dst, uint64_t rows, uint64_t cols, uint64_t seed,
                        float amp, cudaStream_t s, uint64_t row0 = 0, int tiled = 1,
                        SrcWindow src = {});
// rows: head rows held (vocabulary rows v0 .. v0 + rows - 1)
void launch_init_head(__nv_bfloat16* head, const __nv_bfloat16* emb, const int32_t* plant_src,
                      uint64_t rows, uint64_t d, uint64_t seed, float amp, float plant_coef,
                      cudaStream_t s, uint64_t v0 = 0);
void launch_fill_f32(float* dst, size_t n, float v, cudaStream_t s);

// h_lo (fp32-accumulate mode): bf16(x*g - h), or nullptr
void launch_embed_norm(const PassState* ps, int w, const __nv_bfloat16* emb, const float* gain,
                       int d, float eps, float* x, __nv_bfloat16* h, float* ss, cudaStream_t s,
                       __nv_bfloat16* h_lo = nullptr);
constexpr int kMaxF32AttnKeys = 48 * 1024;  // fp32acc mode: scores of one query row in shared memory
// fp32-accumulate mode attention (attention_f32.cu): fp32 q, fp32 paged KV,
// fp32 softmax on CUDA cores; writes o as bf16 hi + lo halves.
int launch_attention_f32(const PassState* ps, int w, const ModelDims& m, const float* q,
                         const float* kv_f32, const int32_t* page_table, int page_size,
                         int layer, int max_keys, __nv_bfloat16* o, __nv_bfloat16* o_lo,
                         cudaStream_t s);
// Split-KV tensor-core attention with a cluster/DSMEM merge (attention.cu);
// returns 0, or nonzero for an unsupported head_dim / launch failure.
int launch_attention(const PassState* ps, int w, const ModelDims& m, const float* q,
                     const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                     int layer, __nv_bfloat16* o, cudaStream_t s, int ranks = 8);
// Long-prompt prefill attention (head_dim 128: tcgen05, 128-query tiles, K/V
// pages staged by TMA through `map_kv` = the pool as [rows of head_dim] bf16
// with (64-dim x page_size) SW128 boxes; otherwise mma.sync, 64-query tiles).
int launch_attention_prefill(const PassState* ps, int w, const ModelDims& m, const float* q,
                             const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                             int layer, __nv_bfloat16* o, cudaStream_t s, const CUtensorMap* map_kv);
void launch_rmsnorm(int w, const float* x, int d, const float* gain, float eps, __nv_bfloat16* h,
                    cudaStream_t s);
void launch_init_matrix_interleaved(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                    uint64_t seed, float amp, int offset, cudaStream_t s,
                                    uint64_t src_row0 = 0);
// src / dst: device arrays of n slot moves, dst strictly increasing, dst <= src
void launch_kv_compact(__nv_bfloat16* kv_pool, float* kv_f32, const int32_t* page_table,
                       int page_size, const ModelDims& m, const int32_t* src_pos_d,
                       const int32_t* dst_pos_d, int n, cudaStream_t s);

// KV pool addressing: pool[page][layer][k|v][kv_head][page_size][head_dim]
__host__ __device__ inline size_t kv_offset(const ModelDims& m, int page_size, int page,
                                            int layer, int kv, int head, int slot) {
    return ((((static_cast<size_t>(page) * m.n_layers + layer) * 2 + kv) * m.n_kv_heads + head) *
                page_size +
            slot) *
           m.head_dim;
}

}  // namespace dd
