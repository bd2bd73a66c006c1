// Device kernels of one target verification pass (everything except the
// tcgen05 GEMM): synthetic weight generation, embedding gather + RMSNorm,
// split-K reductions fused with RoPE + paged-KV append, residual + RMSNorm,
// SwiGLU, and decode-style attention over the paged bf16 KV cache.
//
// Numerics (mirrored by oracle/llama_ref.c):
//   residual stream x: fp32; GEMM inputs h / o / a: bf16 (round-to-nearest);
//   GEMM accumulate fp32; q kept fp32 after RoPE; K, V stored bf16;
//   attention scores/softmax fp32; logits fp32.
#include "common.cuh"
#include "model.h"

namespace dd {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Small kernels of the pass are launched normally (they start once the
// preceding GEMM has completed) but trigger launch_dependents immediately, so
// the following weight-streaming GEMM (launched with programmatic dependent
// launch) becomes resident and fetches its first weight stages while they run.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
    kernel<<<grid, block, smem, s>>>(static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------ weights
// Element (r, c) of a rows x cols block is logical element
// (src.row0 + r) * src.cols + src.col0 + c of the full generated tensor (the
// whole tensor when unsharded, one rank's rows or columns under tensor
// parallelism), written to physical row row0 + r of a pre-tiled matrix with
// `cols` columns.
__global__ void init_matrix_kernel(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                   uint64_t seed, float amp, uint64_t row0, int tiled,
                                   SrcWindow src) {
    const uint64_t n = rows * cols;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = e / cols, c = e % cols;
        const uint64_t le = (src.row0 + r) * (src.cols ? src.cols : cols) + src.col0 + c;
        const __nv_bfloat16 v = __float2bfloat16_rn(__fmul_rn(weight_unit(seed, le), amp));
        dst[tiled ? tiled_offset(row0 + r, c, cols) : (row0 + r) * cols + c] = v;
    }
}

void launch_init_matrix(__nv_bfloat16* dst, uint64_t rows, uint64_t cols, uint64_t seed,
                        float amp, cudaStream_t s, uint64_t row0, int tiled, SrcWindow src) {
    init_matrix_kernel<<<kNumSMs * 8, 256, 0, s>>>(dst, rows, cols, seed, amp, row0, tiled, src);
}

// Logical row r of a [rows, cols] tensor stored at physical row
// (r / 64) * 128 + offset + r % 64: the gate/up interleave that lets one
// 128-row GEMM tile hold matching gate and up features (SwiGLU epilogue).
__global__ void init_matrix_il_kernel(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                      uint64_t seed, float amp, int offset, uint64_t src_row0) {
    const uint64_t n = rows * cols;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = e / cols, c = e % cols;
        const uint64_t pr = (r / 64) * 128 + offset + r % 64;
        const uint64_t le = (src_row0 + r) * cols + c;
        dst[tiled_offset(pr, c, cols)] = __float2bfloat16_rn(__fmul_rn(weight_unit(seed, le), amp));
    }
}

void launch_init_matrix_interleaved(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                    uint64_t seed, float amp, int offset, cudaStream_t s,
                                    uint64_t src_row0) {
    init_matrix_il_kernel<<<kNumSMs * 8, 256, 0, s>>>(dst, rows, cols, seed, amp, offset, src_row0);
}

// LM head: random rows plus, for planted tokens t, row pi(t) += coef * E[t].
// plant_src[v] = t (or -1) with pi(t) = v.  Local row r is vocabulary row v0 + r.
__global__ void init_head_kernel(__nv_bfloat16* head, const __nv_bfloat16* emb,
                                 const int32_t* plant_src, uint64_t rows, uint64_t d,
                                 uint64_t seed, float amp, float coef, uint64_t v0) {
    const uint64_t n = rows * d;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = e / d, i = e % d, v = v0 + r;
        float w = __fmul_rn(weight_unit(seed, v * d + i), amp);
        const int32_t t = plant_src ? plant_src[v] : -1;
        if (t >= 0) w = __fmaf_rn(coef, __bfloat162float(emb[static_cast<uint64_t>(t) * d + i]), w);
        head[tiled_offset(r, i, d)] = __float2bfloat16_rn(w);
    }
}

void launch_init_head(__nv_bfloat16* head, const __nv_bfloat16* emb, const int32_t* plant_src,
                      uint64_t rows, uint64_t d, uint64_t seed, float amp, float plant_coef,
                      cudaStream_t s, uint64_t v0) {
    init_head_kernel<<<kNumSMs * 8, 256, 0, s>>>(head, emb, plant_src, rows, d, seed, amp,
                                                 plant_coef, v0);
}

__global__ void fill_f32_kernel(float* dst, size_t n, float v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] = v;
}
void launch_fill_f32(float* dst, size_t n, float v, cudaStream_t s) {
    fill_f32_kernel<<<64, 256, 0, s>>>(dst, n, v);
}

// ------------------------------------------------------------ helpers
// Block-wide sum over 256 threads with a fixed tree (deterministic).
__device__ __forceinline__ float block_sum_256(float v, float* red) {
    v = warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float t = lane < 8 ? red[lane] : 0.0f;
    t = warp_sum(t);
    return t;  // valid in every thread
}

// x (fp32, d) -> h = bf16(x * (1/sqrt(mean(x^2)+eps)) * g)
__device__ __forceinline__ void rmsnorm_row(const float* x, const float* gain, int d, float eps,
                                            __nv_bfloat16* h, float* red) {
    float ss = 0.0f;
    for (int i = threadIdx.x; i < d; i += 256) ss = __fmaf_rn(x[i], x[i], ss);
    const float tot = block_sum_256(ss, red);
    const float r = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(tot, static_cast<float>(d)), eps));
    for (int i = threadIdx.x; i < d; i += 256)
        h[i] = __float2bfloat16_rn(__fmul_rn(__fmul_rn(x[i], r), gain[i]));
}

// ------------------------------------------------------------ embed + norm
__global__ void embed_norm_kernel(const PassState* ps, const __nv_bfloat16* emb,
                                  const float* gain, int d, float eps, float* x,
                                  __nv_bfloat16* h, float* ss, __nv_bfloat16* h_lo) {
    // x = E[tok]; deferred RMSNorm producer: h = bf16(x * g) and per-128-row
    // sums of squares ss[t][d/128] (same tree as the GEMM residual epilogue)
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    const int tok = ps->tokens[t];
    const int tiles = d / 128;
    for (int base = 0; base < tiles; base += 2) {  // d % 256 == 0: uniform trip count
        const int tile = base + (threadIdx.x >> 7);
        const int i = tile * 128 + (threadIdx.x & 127);
        const float v = __bfloat162float(emb[static_cast<size_t>(tok) * d + i]);
        x[static_cast<size_t>(t) * d + i] = v;
        const float uv = __fmul_rn(v, gain[i]);
        const __nv_bfloat16 hi = __float2bfloat16_rn(uv);
        h[static_cast<size_t>(t) * d + i] = hi;
        if (h_lo) h_lo[static_cast<size_t>(t) * d + i] = __float2bfloat16_rn(__fsub_rn(uv, __bfloat162float(hi)));
        float sq = __fmul_rn(v, v);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
        __shared__ float part[8][4];
        const int lw = (threadIdx.x & 127) >> 5, grp = threadIdx.x >> 7;
        if ((threadIdx.x & 31) == 0) part[grp][lw] = sq;
        __syncthreads();
        if ((threadIdx.x & 127) == 0)
            ss[static_cast<size_t>(t) * tiles + tile] =
                __fadd_rn(__fadd_rn(part[grp][0], part[grp][1]), __fadd_rn(part[grp][2], part[grp][3]));
        __syncthreads();
    }
    (void)eps;
}

void launch_embed_norm(const PassState* ps, int w, const __nv_bfloat16* emb, const float* gain,
                       int d, float eps, float* x, __nv_bfloat16* h, float* ss, cudaStream_t s,
                       __nv_bfloat16* h_lo) {
    launch_pdl(embed_norm_kernel, dim3(w), dim3(256), 0, s, ps, emb, gain, d, eps, x, h, ss, h_lo);
}

// ------------------------------------------------------------ RMSNorm
// h[t] = bf16(x[t] * rsqrt(mean(x[t]^2) + eps) * g); one CTA per token row.
__global__ void rmsnorm_kernel(const float* x, int d, const float* gain, float eps,
                               __nv_bfloat16* h) {
    __shared__ float red[8];
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    rmsnorm_row(x + static_cast<size_t>(t) * d, gain, d, eps, h + static_cast<size_t>(t) * d, red);
}

void launch_rmsnorm(int w, const float* x, int d, const float* gain, float eps, __nv_bfloat16* h,
                    cudaStream_t s) {
    launch_pdl(rmsnorm_kernel, dim3(w), dim3(256), 0, s, x, d, gain, eps, h);
}

// ------------------------------------------------------------ KV compaction
// One launch for a whole compaction: CTA = (layer, k|v, kv head), thread =
// head-dim element, moves applied in list order.  With strictly increasing
// dst <= src (host-checked), move i's source slot src[i] is never the
// destination of an earlier move j < i (dst[j] <= src[j] < src[i]), so each
// thread walking the moves in order is exact without any grid-wide barrier.
// Element type T: bf16 pool, or the fp32 pool of fp32-accumulate mode.
template <typename T>
__global__ void kv_compact_kernel(T* pool, const int32_t* page_table, int page_size, ModelDims m,
                                  const int32_t* src, const int32_t* dst, int n) {
    const int layer = blockIdx.x, kv = blockIdx.y, h = blockIdx.z;
    for (int i = threadIdx.x; i < m.head_dim; i += blockDim.x)
        for (int k = 0; k < n; ++k) {
            const int sp = src[k], dp = dst[k];
            if (sp == dp) continue;
            const T v = pool[kv_offset(m, page_size, page_table[sp / page_size], layer, kv, h, sp % page_size) + i];
            pool[kv_offset(m, page_size, page_table[dp / page_size], layer, kv, h, dp % page_size) + i] = v;
        }
}

void launch_kv_compact(__nv_bfloat16* kv_pool, float* kv_f32, const int32_t* page_table,
                       int page_size, const ModelDims& m, const int32_t* src_pos_d,
                       const int32_t* dst_pos_d, int n, cudaStream_t s) {
    const dim3 grid(m.n_layers, 2, m.n_kv_heads);
    if (kv_f32)
        kv_compact_kernel<float><<<grid, 128, 0, s>>>(kv_f32, page_table, page_size, m, src_pos_d, dst_pos_d, n);
    else
        kv_compact_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(kv_pool, page_table, page_size, m, src_pos_d,
                                                            dst_pos_d, n);
}

}  // namespace dd

namespace dd {
void preload_model_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, init_matrix_kernel);
    cudaFuncGetAttributes(&a, init_matrix_il_kernel);
    cudaFuncGetAttributes(&a, init_head_kernel);
    cudaFuncGetAttributes(&a, fill_f32_kernel);
    cudaFuncGetAttributes(&a, embed_norm_kernel);
    cudaFuncGetAttributes(&a, rmsnorm_kernel);
    cudaFuncGetAttributes(&a, kv_compact_kernel<float>);
    cudaFuncGetAttributes(&a, kv_compact_kernel<__nv_bfloat16>);
}
}  // namespace dd
