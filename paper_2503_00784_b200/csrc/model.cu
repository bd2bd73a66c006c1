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
// Logical element e = r * cols + c of a generated tensor goes to physical row
// row0 + r (plain) of a pre-tiled matrix with `tcols` columns.
__global__ void init_matrix_kernel(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                   uint64_t seed, float amp, uint64_t row0, int tiled) {
    const uint64_t n = rows * cols;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const __nv_bfloat16 v = __float2bfloat16_rn(__fmul_rn(weight_unit(seed, e), amp));
        const uint64_t r = row0 + e / cols, c = e % cols;
        dst[tiled ? tiled_offset(r, c, cols) : r * cols + c] = v;
    }
}

void launch_init_matrix(__nv_bfloat16* dst, uint64_t rows, uint64_t cols, uint64_t seed,
                        float amp, cudaStream_t s, uint64_t row0, int tiled) {
    init_matrix_kernel<<<kNumSMs * 8, 256, 0, s>>>(dst, rows, cols, seed, amp, row0, tiled);
}

// Logical row r of a [rows, cols] tensor stored at physical row
// (r / 64) * 128 + offset + r % 64: the gate/up interleave that lets one
// 128-row GEMM tile hold matching gate and up features (SwiGLU epilogue).
__global__ void init_matrix_il_kernel(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                      uint64_t seed, float amp, int offset) {
    const uint64_t n = rows * cols;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t r = e / cols, c = e % cols;
        const uint64_t pr = (r / 64) * 128 + offset + r % 64;
        dst[tiled_offset(pr, c, cols)] = __float2bfloat16_rn(__fmul_rn(weight_unit(seed, e), amp));
    }
}

void launch_init_matrix_interleaved(__nv_bfloat16* dst, uint64_t rows, uint64_t cols,
                                    uint64_t seed, float amp, int offset, cudaStream_t s) {
    init_matrix_il_kernel<<<kNumSMs * 8, 256, 0, s>>>(dst, rows, cols, seed, amp, offset);
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
        head[tiled_offset(v, i, d)] = __float2bfloat16_rn(w);
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
                                  __nv_bfloat16* h, float* ss) {
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
        h[static_cast<size_t>(t) * d + i] = __float2bfloat16_rn(__fmul_rn(v, gain[i]));
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
                       int d, float eps, float* x, __nv_bfloat16* h, float* ss, cudaStream_t s) {
    launch_pdl(embed_norm_kernel, dim3(w), dim3(256), 0, s, ps, emb, gain, d, eps, x, h, ss);
}

// ------------------------------------------------------------ attention
// Split-KV decode attention over the paged bf16 cache (flash-decoding style).
// Grid (head, split, query group of 16).  Keys are cut into 64-key chunks by
// ABSOLUTE position; split s owns chunks s, s+S, ...  A CTA stages each chunk's
// K and V in shared memory once and uses them for all queries of its group
// (online softmax), writes (m, l, o) partials, and the last-arriving split of
// a (head, group) combines the S partials in split order.  The query at
// absolute position p = n_cached + t attends keys 0..p (chain causal mask).
// Every reduction order depends only on (head, position, chunk layout), so a
// token's output is independent of the pass width (greedy determinism).
constexpr int kAttnThreads = 128;
constexpr int kKeyChunk = 64;
constexpr int kQGroup = 16;
constexpr int kSplits = 8;

struct AttnScratch {
    float* part;      // [heads][groups][kSplits][kQGroup][hd + 2]
    int* counters;    // [heads][groups]
};

__global__ void __launch_bounds__(kAttnThreads)
    attention_kernel(const PassState* ps, ModelDims m, const float* q,
                     const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                     int layer, float scale, __nv_bfloat16* o, AttnScratch scr) {
    pdl_wait();
    pdl_launch();
    extern __shared__ __align__(16) uint8_t att_smem[];
    const int hd = m.head_dim;
    const int head = blockIdx.x, split = blockIdx.y, grp = blockIdx.z;
    const int w = ps->w, n0 = ps->n_cached;
    const int q0 = grp * kQGroup;
    const int nq = min(kQGroup, w - q0);
    if (nq <= 0) return;
    const int kvh = head / (m.n_heads / m.n_kv_heads);
    const int n_keys = n0 + q0 + nq;  // keys any query of this group may see
    const int n_chunks = (n_keys + kKeyChunk - 1) / kKeyChunk;
    const int tid = threadIdx.x;

    __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(att_smem);        // [64][hd]
    __nv_bfloat16* sv = sk + kKeyChunk * hd;                                // [64][hd]
    float* sq = reinterpret_cast<float*>(sv + kKeyChunk * hd);              // [16][hd]
    float* sp = sq + kQGroup * hd;                                          // [16][64]
    float* so = sp + kQGroup * kKeyChunk;                                   // [16][hd]
    float* sm = so + kQGroup * hd;                                          // [16] running max
    float* sl = sm + kQGroup;                                               // [16] running sum
    __shared__ int s_last;

    for (int i = tid; i < nq * hd; i += kAttnThreads) {
        const int t = i / hd, d = i % hd;
        sq[t * hd + d] = q[static_cast<size_t>(q0 + t) * m.q_dim() + head * hd + d];
    }
    for (int i = tid; i < kQGroup * hd; i += kAttnThreads) so[i] = 0.0f;
    if (tid < kQGroup) {
        sm[tid] = -INFINITY;
        sl[tid] = 0.0f;
    }
    __syncthreads();

    const int vec_per_row = hd / 8;  // 16-byte vectors per key row
    for (int c = split; c < n_chunks; c += kSplits) {
        const int k0 = c * kKeyChunk;
        const int nk = min(kKeyChunk, n_keys - k0);
        // stage K and V rows of this chunk (coalesced 16-byte loads)
        for (int i = tid; i < nk * vec_per_row; i += kAttnThreads) {
            const int j = i / vec_per_row, v = i % vec_per_row;
            const int key = k0 + j;
            const int page = page_table[key / page_size], slot = key % page_size;
            const uint4* kr = reinterpret_cast<const uint4*>(
                kv_pool + kv_offset(m, page_size, page, layer, 0, kvh, slot));
            const uint4* vr = reinterpret_cast<const uint4*>(
                kv_pool + kv_offset(m, page_size, page, layer, 1, kvh, slot));
            reinterpret_cast<uint4*>(sk + j * hd)[v] = __ldg(kr + v);
            reinterpret_cast<uint4*>(sv + j * hd)[v] = __ldg(vr + v);
        }
        __syncthreads();
        // scores for (query t, key j); masked keys -> -inf
        for (int i = tid; i < nq * kKeyChunk; i += kAttnThreads) {
            const int t = i / kKeyChunk, j = i % kKeyChunk;
            const int key = k0 + j;
            float sc = -INFINITY;
            if (j < nk && key <= n0 + q0 + t) {
                const float* qv = sq + t * hd;
                const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(sk + j * hd);
                float acc = 0.0f;
#pragma unroll 8
                for (int d2 = 0; d2 < hd / 2; ++d2) {
                    const float2 f = __bfloat1622float2(kr[d2]);
                    acc = __fmaf_rn(qv[2 * d2], f.x, acc);
                    acc = __fmaf_rn(qv[2 * d2 + 1], f.y, acc);
                }
                sc = __fmul_rn(acc, scale);
            }
            sp[t * kKeyChunk + j] = sc;
        }
        __syncthreads();
        // online softmax update per query (rescale the running output)
        if (tid < nq) {
            const int t = tid;
            float mx = sm[t];
            for (int j = 0; j < kKeyChunk; ++j) mx = fmaxf(mx, sp[t * kKeyChunk + j]);
            const float corr = mx == -INFINITY ? 1.0f : expf(sm[t] - mx);
            float sum = 0.0f;
            for (int j = 0; j < kKeyChunk; ++j) {
                const float s2 = sp[t * kKeyChunk + j];
                const float e = s2 == -INFINITY ? 0.0f : expf(s2 - mx);
                sp[t * kKeyChunk + j] = e;
                sum += e;
            }
            sl[t] = __fadd_rn(__fmul_rn(sl[t], corr), sum);
            sm[t] = mx;
            for (int d = 0; d < hd; ++d) so[t * hd + d] = __fmul_rn(so[t * hd + d], corr);
        }
        __syncthreads();
        // o[t][d] += sum_j p[t][j] * V[j][d]; thread per dim, all queries of the group
        for (int d = tid; d < hd; d += kAttnThreads) {
            float acc[kQGroup];
#pragma unroll
            for (int t = 0; t < kQGroup; ++t) acc[t] = 0.0f;
            for (int j = 0; j < nk; ++j) {
                const float v = __bfloat162float(sv[j * hd + d]);
#pragma unroll
                for (int t = 0; t < kQGroup; ++t)
                    if (t < nq) acc[t] = __fmaf_rn(sp[t * kKeyChunk + j], v, acc[t]);
            }
#pragma unroll
            for (int t = 0; t < kQGroup; ++t)
                if (t < nq) so[t * hd + d] = __fadd_rn(so[t * hd + d], acc[t]);
        }
        __syncthreads();
    }

    // partials -> workspace; last split combines in split order
    const int groups = gridDim.z;
    const size_t rec = static_cast<size_t>(hd) + 2;
    float* part = scr.part + ((static_cast<size_t>(head) * groups + grp) * kSplits + split) * kQGroup * rec;
    for (int i = tid; i < nq * hd; i += kAttnThreads) part[(i / hd) * rec + 2 + i % hd] = so[i];
    if (tid < nq) {
        part[tid * rec + 0] = sm[tid];
        part[tid * rec + 1] = sl[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int prev = atomicAdd(&scr.counters[head * groups + grp], 1);
        s_last = (prev == kSplits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* base = scr.part + (static_cast<size_t>(head) * groups + grp) * kSplits * kQGroup * rec;
    for (int i = tid; i < nq * hd; i += kAttnThreads) {
        const int t = i / hd, d = i % hd;
        float mx = -INFINITY;
        for (int s2 = 0; s2 < kSplits; ++s2) mx = fmaxf(mx, __ldcg(base + (s2 * kQGroup + t) * rec));
        float l = 0.0f, acc = 0.0f;
        for (int s2 = 0; s2 < kSplits; ++s2) {
            const float* r = base + (s2 * kQGroup + t) * rec;
            const float ms = __ldcg(r);
            if (ms == -INFINITY) continue;
            const float f = expf(ms - mx);
            l = __fmaf_rn(__ldcg(r + 1), f, l);
            acc = __fmaf_rn(__ldcg(r + 2 + d), f, acc);
        }
        o[static_cast<size_t>(q0 + t) * m.q_dim() + head * hd + d] =
            __float2bfloat16_rn(__fdiv_rn(acc, l));
    }
    if (tid == 0) scr.counters[head * groups + grp] = 0;
}

static AttnScratch g_attn_scratch{nullptr, nullptr};

void attention_set_max_keys(int max_keys) {
    (void)max_keys;
    const int hd = 256;  // upper bound for the smem carve-up
    const int bytes = 2 * kKeyChunk * hd * 2 + (2 * kQGroup * hd + kQGroup * kKeyChunk + 2 * kQGroup) * 4;
    cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (!g_attn_scratch.part) {
        const size_t groups = (kMaxPassTokens + kQGroup - 1) / kQGroup;
        cudaMalloc(&g_attn_scratch.part,
                   sizeof(float) * 64 * groups * kSplits * kQGroup * (256 + 2));  // <= 64 heads
        cudaMalloc(&g_attn_scratch.counters, sizeof(int) * 64 * groups);
        cudaMemset(g_attn_scratch.counters, 0, sizeof(int) * 64 * groups);
    }
}

void launch_attention(const PassState* ps, int w, const ModelDims& m, const float* q,
                      const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                      int layer, __nv_bfloat16* o, cudaStream_t s) {
    const int groups = (w + kQGroup - 1) / kQGroup;
    dim3 grid(m.n_heads, kSplits, groups);
    const int hd = m.head_dim;
    const int smem = 2 * kKeyChunk * hd * 2 + (2 * kQGroup * hd + kQGroup * kKeyChunk + 2 * kQGroup) * 4;
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(hd)));
    launch_pdl(attention_kernel, grid, dim3(kAttnThreads), smem, s, ps, m, q, kv_pool, page_table,
               page_size, layer, scale, o, g_attn_scratch);
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
