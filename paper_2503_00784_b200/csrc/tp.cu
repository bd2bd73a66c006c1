// Tensor-parallel reductions over NVLink peer memory (tp.h).  Both kernels
// are latency-bound (a [W, d] fp32 partial per rank, W <= 128): one CTA per
// 128-column tile of the residual stream, loads of every rank's partial issued
// back to back, no shared-memory staging.
#include <algorithm>

#include "common.cuh"
#include "tp.h"

namespace dd {

TpLayout tp_layout(int d, int max_local_vocab) {
    TpLayout L{};
    L.flags_off = 0;
    L.part_off = 4096;
    L.part_stride = static_cast<size_t>(kMaxPassTokens) * d;
    L.lg_off = L.part_off + sizeof(float) * 2 * L.part_stride;
    L.pflag_off = L.lg_off + sizeof(float) * static_cast<size_t>(kMaxPassTokens) * max_local_vocab;
    L.pflag_off = (L.pflag_off + 4095) & ~static_cast<size_t>(4095);
    L.pxch_off = L.pflag_off + sizeof(int) * static_cast<size_t>(kMaxTp) * kTpPassTiles * kTpFlagStride;
    L.bytes = L.pxch_off + sizeof(float) * static_cast<size_t>(kTpPassSlots) * kTpPassTiles * 128 * 16;
    L.bytes = (L.bytes + 4095) & ~static_cast<size_t>(4095);
    return L;
}

namespace {

__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float ld_relaxed_sys(const float* p) {
    float v;
    asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Signal op `expected` to every rank (CTA 0), then wait for every rank's
// signal.  A peer that never arrives (dead process, mismatched pass
// sequence) traps after 10 s instead of hanging the GPU.
// Flag values are the op's sequence number mod 2^32 (epoch * ops + op + 1
// wraps after ~13M 70B passes), compared wrap-safely.
__device__ void tp_barrier(const TpPeers& P, unsigned expected) {
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && tid < P.size) {
        __threadfence_system();
        st_release_sys(P.flags[tid] + P.rank * kTpFlagStride, static_cast<int>(expected));
    }
    if (tid < P.size) {
        const int* f = P.flags[P.rank] + tid * kTpFlagStride;
        const unsigned long long t0 = now_ns();
        while (static_cast<int>(static_cast<unsigned>(ld_acquire_sys(f)) - expected) < 0) {
            __nanosleep(64);
            if (now_ns() - t0 > 10000000000ull) __trap();
        }
    }
    __syncthreads();
}

// x[t][c] += sum_r part_r[t][c]; u = bf16(x * g); ss_out[t][tile] = sum of
// squares of the tile's 128 columns (the kEpiResidual epilogue's tree).
__global__ void __launch_bounds__(128) tp_reduce_residual_kernel(
    TpPeers P, const PassState* ps, int op, int ops_per_pass, int d, float* x, __nv_bfloat16* u,
    const float* gain, float* ss_out) {
    const int w = ps->w;
    tp_barrier(P, static_cast<unsigned>(ps->epoch) * static_cast<unsigned>(ops_per_pass) +
                      static_cast<unsigned>(op) + 1u);
    __shared__ float part[4];
    const int tid = threadIdx.x;
    const int tiles = d / 128;
    const size_t off = static_cast<size_t>(op & 1) * kMaxPassTokens * d;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int col = tile * 128 + tid;
    const float g = gain[col];
    for (int t = 0; t < w; ++t) {
        const size_t i = static_cast<size_t>(t) * d + col;
        float v[kMaxTp];
#pragma unroll
        for (int r = 0; r < kMaxTp; ++r) v[r] = r < P.size ? ld_relaxed_sys(P.part[r] + off + i) : 0.0f;
        float y = v[0];
#pragma unroll
        for (int r = 1; r < kMaxTp; ++r)
            if (r < P.size) y = __fadd_rn(y, v[r]);
        const float xv = __fadd_rn(x[i], y);
        x[i] = xv;
        u[i] = __float2bfloat16_rn(__fmul_rn(xv, g));
        float sq = __fmul_rn(xv, xv);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
        if ((tid & 31) == 0) part[tid >> 5] = sq;
        __syncthreads();
        if (tid == 0)
            ss_out[static_cast<size_t>(t) * tiles + tile] =
                __fadd_rn(__fadd_rn(part[0], part[1]), __fadd_rn(part[2], part[3]));
        __syncthreads();
    }
    }
}

__global__ void __launch_bounds__(256) tp_gather_logits_kernel(TpPeers P, const PassState* ps,
                                                               int op, int ops_per_pass, int vocab,
                                                               float* logits) {
    const int w = ps->w;
    tp_barrier(P, static_cast<unsigned>(ps->epoch) * static_cast<unsigned>(ops_per_pass) +
                      static_cast<unsigned>(op) + 1u);
    const size_t n = static_cast<size_t>(w) * vocab;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < n;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int t = static_cast<int>(e / vocab), v = static_cast<int>(e % vocab);
        int r = 0;
        while (r + 1 < P.size && v >= P.v0[r + 1]) ++r;
        const int vl = P.v0[r + 1] - P.v0[r];
        logits[e] = ld_relaxed_sys(P.lg[r] + static_cast<size_t>(t) * vl + (v - P.v0[r]));
    }
}

}  // namespace

void launch_tp_reduce_residual(const TpPeers& P, const PassState* ps, int op, int ops_per_pass,
                               int d, float* x, __nv_bfloat16* u, const float* gain,
                               float* ss_out, cudaStream_t s) {
    // ranks sharing one device: few spinning CTAs, so a peer's GEMM (whose
    // stream-K reducers need all of its CTAs resident) always finds its SMs
    const int grid = P.shared ? std::min(d / 128, 4) : d / 128;
    tp_reduce_residual_kernel<<<grid, 128, 0, s>>>(P, ps, op, ops_per_pass, d, x, u, gain, ss_out);
}

void launch_tp_gather_logits(const TpPeers& P, const PassState* ps, int op, int ops_per_pass,
                             int vocab, float* logits, cudaStream_t s) {
    tp_gather_logits_kernel<<<P.shared ? 4 : kNumSMs, 256, 0, s>>>(P, ps, op, ops_per_pass, vocab, logits);
}

}  // namespace dd

namespace dd {
void preload_tp_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, tp_reduce_residual_kernel);
    cudaFuncGetAttributes(&a, tp_gather_logits_kernel);
}
}  // namespace dd
