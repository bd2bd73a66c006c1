// Attention of the fp32-accumulate mode (DD_PREC_FP32ACC, north star: "fp32-
// accumulate mode within 1e-4 relative").  This mode is the precision
// reference of the forward contract (proj/include/duodec/model.hpp:57-65),
// not the throughput path: queries, the paged KV cache and the softmax stay in
// fp32 and run on CUDA cores, one CTA per (token, head); the output is written
// as bf16 hi + lo halves for the split-activation tcgen05 O-projection.
// Causal over keys 0 .. n_cached + t, like oracle/llama_ref.c attn_range.
#include "common.cuh"
#include "model.h"

namespace dd {
namespace {

constexpr int kF32Threads = 128;

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < kF32Threads / 32; ++i) r = fmaxf(r, red[i]);
    return r;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < kF32Threads / 32; ++i) r = __fadd_rn(r, red[i]);
    return r;
}

__global__ void __launch_bounds__(kF32Threads) attn_f32_kernel(
    const PassState* ps, ModelDims m, const float* __restrict__ q, const float* __restrict__ kv,
    const int32_t* __restrict__ page_table, int page_size, int layer, float scale,
    __nv_bfloat16* __restrict__ o, __nv_bfloat16* __restrict__ o_lo) {
    extern __shared__ float sc[];  // [n_keys] scores, then softmax weights
    __shared__ float qs[256];
    __shared__ float red[kF32Threads / 32];
    const int t = blockIdx.x, head = blockIdx.y, tid = threadIdx.x;
    const int hd = m.head_dim, qd = m.q_dim();
    const int pos = ps->n_cached + t, nk = pos + 1;
    const int kvh = head / (m.n_heads / m.n_kv_heads);
    for (int i = tid; i < hd; i += kF32Threads) qs[i] = q[static_cast<size_t>(t) * qd + head * hd + i];
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int j = warp; j < nk; j += kF32Threads / 32) {
        const float* kr = kv + kv_offset(m, page_size, page_table[j / page_size], layer, 0, kvh, j % page_size);
        float acc = 0.0f;
        for (int i = lane; i < hd; i += 32) acc = __fmaf_rn(qs[i], kr[i], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (lane == 0) sc[j] = __fmul_rn(acc, scale);
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int j = tid; j < nk; j += kF32Threads) mx = fmaxf(mx, sc[j]);
    mx = block_max(mx, red);
    float sum = 0.0f;
    for (int j = tid; j < nk; j += kF32Threads) {
        const float e = expf(__fsub_rn(sc[j], mx));
        sc[j] = e;
        sum = __fadd_rn(sum, e);
    }
    sum = block_sum(sum, red);  // ends with __syncthreads: every sc[j] written
    const float inv = 1.0f / sum;
    for (int i = tid; i < hd; i += kF32Threads) {
        float acc = 0.0f;
        for (int j = 0; j < nk; ++j) {
            const float* vr = kv + kv_offset(m, page_size, page_table[j / page_size], layer, 1, kvh, j % page_size);
            acc = __fmaf_rn(sc[j], vr[i], acc);
        }
        const float v = __fmul_rn(acc, inv);
        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
        const size_t oi = static_cast<size_t>(t) * qd + head * hd + i;
        o[oi] = hi;
        o_lo[oi] = __float2bfloat16_rn(__fsub_rn(v, __bfloat162float(hi)));
    }
}

}  // namespace

int launch_attention_f32(const PassState* ps, int w, const ModelDims& m, const float* q,
                         const float* kv_f32, const int32_t* page_table, int page_size, int layer,
                         int max_keys, __nv_bfloat16* o, __nv_bfloat16* o_lo, cudaStream_t s) {
    if (m.head_dim > 256) return 1;
    const size_t smem = sizeof(float) * static_cast<size_t>(max_keys);
    static bool attr[kMaxDevices] = {};
    const int dev = current_device_slot();
    if (!attr[dev]) {
        if (cudaFuncSetAttribute(attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kMaxF32AttnKeys * sizeof(float))) != cudaSuccess)
            return 2;
        attr[dev] = true;
    }
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(m.head_dim)));
    attn_f32_kernel<<<dim3(w, m.n_heads), kF32Threads, smem, s>>>(ps, m, q, kv_f32, page_table,
                                                                  page_size, layer, scale, o, o_lo);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

}  // namespace dd

namespace dd {
void preload_attention_f32_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, attn_f32_kernel);
}
}  // namespace dd
