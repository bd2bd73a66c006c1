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

// ------------------------------------------------------------ weights
__global__ void init_matrix_kernel(__nv_bfloat16* dst, uint64_t n, uint64_t seed, float amp) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        dst[e] = __float2bfloat16_rn(__fmul_rn(weight_unit(seed, e), amp));
    }
}

void launch_init_matrix(__nv_bfloat16* dst, uint64_t rows, uint64_t cols, uint64_t seed,
                        float amp, cudaStream_t s) {
    init_matrix_kernel<<<kNumSMs * 8, 256, 0, s>>>(dst, rows * cols, seed, amp);
}

// LM head: random rows plus, for planted tokens t, row pi(t) += coef * E[t].
// plant_src[v] = t (or -1) with pi(t) = v.
__global__ void init_head_kernel(__nv_bfloat16* head, const __nv_bfloat16* emb,
                                 const int32_t* plant_src, uint64_t vocab, uint64_t d,
                                 uint64_t seed, float amp, float coef) {
    const uint64_t n = vocab * d;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        float w = __fmul_rn(weight_unit(seed, e), amp);
        const uint64_t v = e / d, i = e % d;
        const int32_t t = plant_src ? plant_src[v] : -1;
        if (t >= 0) w = __fmaf_rn(coef, __bfloat162float(emb[static_cast<uint64_t>(t) * d + i]), w);
        head[e] = __float2bfloat16_rn(w);
    }
}

void launch_init_head(__nv_bfloat16* head, const __nv_bfloat16* emb, const int32_t* plant_src,
                      uint64_t vocab, uint64_t d, uint64_t seed, float amp, float plant_coef,
                      cudaStream_t s) {
    init_head_kernel<<<kNumSMs * 8, 256, 0, s>>>(head, emb, plant_src, vocab, d, seed, amp,
                                                 plant_coef);
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
                                  __nv_bfloat16* h) {
    __shared__ float red[8];
    const int t = blockIdx.x;
    const int tok = ps->tokens[t];
    float* xr = x + static_cast<size_t>(t) * d;
    for (int i = threadIdx.x; i < d; i += 256)
        xr[i] = __bfloat162float(emb[static_cast<size_t>(tok) * d + i]);
    __syncthreads();
    rmsnorm_row(xr, gain, d, eps, h + static_cast<size_t>(t) * d, red);
}

void launch_embed_norm(const PassState* ps, int w, const __nv_bfloat16* emb, const float* gain,
                       int d, float eps, float* x, __nv_bfloat16* h, cudaStream_t s) {
    embed_norm_kernel<<<w, 256, 0, s>>>(ps, emb, gain, d, eps, x, h);
}

// ------------------------------------------------------------ QKV epilogue
// Reduce split-K partials of the fused QKV projection, apply RoPE (HF
// rotate_half convention) to q and k at absolute position n_cached + t, keep
// q in fp32, append bf16 k and v to the paged cache.
__global__ void qkv_epilogue_kernel(const PassState* ps, const float* ws, int splits,
                                    ModelDims m, const float* rope_cos, const float* rope_sin,
                                    float* q_out, __nv_bfloat16* kv_pool,
                                    const int32_t* page_table, int page_size, int layer) {
    const int t = blockIdx.x;
    const int w = ps->w;
    const int pos = ps->n_cached + t;
    const int hd = m.head_dim, half = hd / 2;
    const int rows = m.qkv_rows();
    const int n_q = m.q_dim(), n_kv = m.kv_dim();
    const size_t split_stride = static_cast<size_t>(w) * rows;
    const float* base = ws + static_cast<size_t>(t) * rows;
    const float* cs = rope_cos + static_cast<size_t>(pos) * half;
    const float* sn = rope_sin + static_cast<size_t>(pos) * half;
    const int page = page_table[pos / page_size], slot = pos % page_size;

    // rotary pairs over q heads and k heads
    const int n_pairs = (m.n_heads + m.n_kv_heads) * half;
    for (int p = threadIdx.x; p < n_pairs; p += blockDim.x) {
        const int head = p / half, i = p % half;
        const int r0 = head * hd + i;  // q heads first, then k heads (contiguous in qkv rows)
        float a = 0.0f, b = 0.0f;
        for (int s = 0; s < splits; ++s) {
            a = __fadd_rn(a, base[s * split_stride + r0]);
            b = __fadd_rn(b, base[s * split_stride + r0 + half]);
        }
        const float c = cs[i], sv = sn[i];
        const float lo = __fmaf_rn(a, c, -__fmul_rn(b, sv));
        const float hi = __fmaf_rn(b, c, __fmul_rn(a, sv));
        if (head < m.n_heads) {
            float* qd = q_out + static_cast<size_t>(t) * n_q + head * hd;
            qd[i] = lo;
            qd[i + half] = hi;
        } else {
            const int kh = head - m.n_heads;
            __nv_bfloat16* kd = kv_pool + kv_offset(m, page_size, page, layer, 0, kh, slot);
            kd[i] = __float2bfloat16_rn(lo);
            kd[i + half] = __float2bfloat16_rn(hi);
        }
    }
    for (int e = threadIdx.x; e < n_kv; e += blockDim.x) {
        const int r = n_q + n_kv + e;
        float v = 0.0f;
        for (int s = 0; s < splits; ++s) v = __fadd_rn(v, base[s * split_stride + r]);
        const int vh = e / hd, i = e % hd;
        kv_pool[kv_offset(m, page_size, page, layer, 1, vh, slot) + i] = __float2bfloat16_rn(v);
    }
}

void launch_qkv_epilogue(const PassState* ps, int w, const float* ws, int splits,
                         const ModelDims& m, const float* rope_cos, const float* rope_sin,
                         float* q_out, __nv_bfloat16* kv_pool, const int32_t* page_table,
                         int page_size, int layer, cudaStream_t s) {
    qkv_epilogue_kernel<<<w, 256, 0, s>>>(ps, ws, splits, m, rope_cos, rope_sin, q_out, kv_pool,
                                          page_table, page_size, layer);
}

// ------------------------------------------------------------ attention
// One CTA per (query head, new token). The query at absolute position
// pos = n_cached + t attends to keys 0..pos (cached prefix + the chain of new
// tokens up to itself).  Work per CTA depends only on (head, pos), so a
// token's output is independent of the pass width.
constexpr int kAttnThreads = 128;
__global__ void __launch_bounds__(kAttnThreads)
    attention_kernel(const PassState* ps, ModelDims m, const float* q,
                     const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                     int layer, float scale, __nv_bfloat16* o) {
    extern __shared__ float scores[];  // [n_keys]
    __shared__ float red[kAttnThreads / 32];
    const int head = blockIdx.x, t = blockIdx.y;
    const int pos = ps->n_cached + t;
    const int n_keys = pos + 1;
    const int hd = m.head_dim;
    const int kvh = head / (m.n_heads / m.n_kv_heads);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* qv = q + static_cast<size_t>(t) * m.q_dim() + head * hd;

    // scores: one warp per key, lanes split head_dim (hd <= 256, multiple of 32)
    const int per_lane = hd / 32;
    float qr[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) qr[j] = j < per_lane ? qv[lane * per_lane + j] : 0.0f;
    for (int key = warp; key < n_keys; key += kAttnThreads / 32) {
        const int page = page_table[key / page_size], slot = key % page_size;
        const __nv_bfloat16* kr = kv_pool + kv_offset(m, page_size, page, layer, 0, kvh, slot);
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < per_lane) acc = __fmaf_rn(qr[j], __bfloat162float(kr[lane * per_lane + j]), acc);
        acc = warp_sum(acc);
        if (lane == 0) scores[key] = __fmul_rn(acc, scale);
    }
    __syncthreads();
    // softmax (fp32)
    float mx = -INFINITY;
    for (int k = threadIdx.x; k < n_keys; k += kAttnThreads) mx = fmaxf(mx, scores[k]);
    mx = warp_max(mx);
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int i = 1; i < kAttnThreads / 32; ++i) mx = fmaxf(mx, red[i]);
    __syncthreads();
    float sum = 0.0f;
    for (int k = threadIdx.x; k < n_keys; k += kAttnThreads) {
        const float e = expf(scores[k] - mx);
        scores[k] = e;
        sum += e;
    }
    sum = warp_sum(sum);
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    sum = 0.0f;
#pragma unroll
    for (int i = 0; i < kAttnThreads / 32; ++i) sum += red[i];
    const float inv = 1.0f / sum;
    // o[d] = sum_k p_k v_k[d]; thread per dim (hd <= 128 here; loop otherwise)
    for (int d0 = threadIdx.x; d0 < hd; d0 += kAttnThreads) {
        float acc = 0.0f;
        for (int k = 0; k < n_keys; ++k) {
            const int page = page_table[k / page_size], slot = k % page_size;
            const __nv_bfloat16* vr =
                kv_pool + kv_offset(m, page_size, page, layer, 1, kvh, slot);
            acc = __fmaf_rn(scores[k], __bfloat162float(vr[d0]), acc);
        }
        o[static_cast<size_t>(t) * m.q_dim() + head * hd + d0] =
            __float2bfloat16_rn(__fmul_rn(acc, inv));
    }
}

static int g_attn_smem_bytes = 48 * 1024;

void attention_set_max_keys(int max_keys) {
    g_attn_smem_bytes = max_keys * static_cast<int>(sizeof(float));
    if (g_attn_smem_bytes > 48 * 1024)
        cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             g_attn_smem_bytes);
}

void launch_attention(const PassState* ps, int w, const ModelDims& m, const float* q,
                      const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                      int layer, __nv_bfloat16* o, cudaStream_t s) {
    dim3 grid(m.n_heads, w);
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(m.head_dim)));
    attention_kernel<<<grid, kAttnThreads, g_attn_smem_bytes, s>>>(ps, m, q, kv_pool, page_table,
                                                                   page_size, layer, scale, o);
}

// ------------------------------------------------------------ residual + norm
__global__ void residual_norm_kernel(const float* ws, int splits, int w, int d,
                                     const float* gain, float eps, float* x, __nv_bfloat16* h) {
    __shared__ float red[8];
    const int t = blockIdx.x;
    float* xr = x + static_cast<size_t>(t) * d;
    const size_t split_stride = static_cast<size_t>(w) * d;
    for (int i = threadIdx.x; i < d; i += 256) {
        float acc = 0.0f;
        for (int s = 0; s < splits; ++s)
            acc = __fadd_rn(acc, ws[s * split_stride + static_cast<size_t>(t) * d + i]);
        xr[i] = __fadd_rn(xr[i], acc);
    }
    __syncthreads();
    rmsnorm_row(xr, gain, d, eps, h + static_cast<size_t>(t) * d, red);
}

void launch_residual_norm(int w, const float* ws, int splits, int d, const float* gain, float eps,
                          float* x, __nv_bfloat16* h, cudaStream_t s) {
    residual_norm_kernel<<<w, 256, 0, s>>>(ws, splits, w, d, gain, eps, x, h);
}

// ------------------------------------------------------------ SwiGLU
__global__ void swiglu_kernel(const float* ws, int splits, int w, int ffn, __nv_bfloat16* a) {
    const int t = blockIdx.y;
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= ffn) return;
    const size_t row = static_cast<size_t>(t) * 2 * ffn;
    const size_t split_stride = static_cast<size_t>(w) * 2 * ffn;
    float g = 0.0f, u = 0.0f;
    for (int s = 0; s < splits; ++s) {
        g = __fadd_rn(g, ws[s * split_stride + row + f]);
        u = __fadd_rn(u, ws[s * split_stride + row + ffn + f]);
    }
    const float silu = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
    a[static_cast<size_t>(t) * ffn + f] = __float2bfloat16_rn(__fmul_rn(silu, u));
}

void launch_swiglu(int w, const float* ws, int splits, int ffn, __nv_bfloat16* a, cudaStream_t s) {
    dim3 grid((ffn + 255) / 256, w);
    swiglu_kernel<<<grid, 256, 0, s>>>(ws, splits, w, ffn, a);
}

// ------------------------------------------------------------ logits reduce
__global__ void reduce_rows_kernel(const float* ws, int splits, int w, int n, float* out) {
    const int t = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t split_stride = static_cast<size_t>(w) * n;
    float acc = 0.0f;
    for (int s = 0; s < splits; ++s)
        acc = __fadd_rn(acc, ws[s * split_stride + static_cast<size_t>(t) * n + i]);
    out[static_cast<size_t>(t) * n + i] = acc;
}

void launch_reduce_rows(int w, const float* ws, int splits, int n, float* out, cudaStream_t s) {
    dim3 grid((n + 255) / 256, w);
    reduce_rows_kernel<<<grid, 256, 0, s>>>(ws, splits, w, n, out);
}

// ------------------------------------------------------------ KV compaction
// Sequentially-ordered slot moves (src -> dst, dst <= src) for every layer,
// K and V, kv head: one CTA per (move, layer) with moves applied in order
// by a single launch per move index to respect overlapping chains.
__global__ void kv_move_kernel(__nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                               ModelDims m, int src, int dst) {
    const int layer = blockIdx.x;
    const int hd = m.head_dim;
    const int ps = page_table[src / page_size], ss = src % page_size;
    const int pd = page_table[dst / page_size], sd = dst % page_size;
    for (int e = threadIdx.x; e < 2 * m.n_kv_heads * hd; e += blockDim.x) {
        const int kv = e / (m.n_kv_heads * hd);
        const int rem = e % (m.n_kv_heads * hd);
        const int h = rem / hd, i = rem % hd;
        kv_pool[kv_offset(m, page_size, pd, layer, kv, h, sd) + i] =
            kv_pool[kv_offset(m, page_size, ps, layer, kv, h, ss) + i];
    }
}

void launch_kv_compact(__nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                       const ModelDims& m, const int32_t* src_pos, const int32_t* dst_pos, int n,
                       cudaStream_t s) {
    for (int i = 0; i < n; ++i) {
        if (src_pos[i] == dst_pos[i]) continue;
        kv_move_kernel<<<m.n_layers, 256, 0, s>>>(kv_pool, page_table, page_size, m, src_pos[i],
                                                  dst_pos[i]);
    }
}

}  // namespace dd
