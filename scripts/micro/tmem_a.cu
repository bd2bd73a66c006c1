// Micro-check (scripts/micro; not product): weights staged smem -> TMEM with
// tcgen05.cp and used as the A operand of tcgen05.mma (kind::f16, M=128, N=16),
// against the smem-A path and a host reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_00784_b200/csrc
//   scripts/micro/tmem_a.cu -o scripts/micro/tmem_a_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "common.cuh"
using namespace dd;

__device__ __forceinline__ void tcp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// mode 0: A from smem; mode 1: A via tcgen05.cp into TMEM
__global__ void k(const __nv_bfloat16* wt, const __nv_bfloat16* xt, float* out, int mode, int nblk) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x;
    if (tid < 32) tmem_alloc<512>(&slot);
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // stage nblk weight blocks (16 KiB each) and activation blocks (16 x 64 bf16, SW128 rows)
    for (int i = tid; i < nblk * 8192 / 8; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(wt)[i];
    uint8_t* sx = sm + nblk * 16384;
    for (int i = tid; i < nblk * 1024 / 8; i += blockDim.x)
        reinterpret_cast<uint4*>(sx)[i] = reinterpret_cast<const uint4*>(xt)[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, 16);
        const uint32_t acc = tmem;          // columns 0..15
        const uint32_t aslot = tmem + 64;   // A slots from column 64
        for (int b = 0; b < nblk; ++b) {
            const uint32_t sa = smem_u32(sm + b * 16384);
            const uint32_t sb = smem_u32(sx + b * 2048);
            if (mode == 1) {
                for (int kk = 0; kk < 4; ++kk)
                    tcp_128x256b(aslot + b * 32 + kk * 8, sw128_kmajor_desc(sa) + 2 * kk);
            }
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bdesc = sw128_kmajor_desc(sb) + 2 * kk;
                if (mode == 0)
                    umma_bf16(acc, sw128_kmajor_desc(sa) + 2 * kk, bdesc, idesc, (b | kk) ? 1u : 0u);
                else
                    umma_bf16_ts(acc, aslot + b * 32 + kk * 8, bdesc, idesc, (b | kk) ? 1u : 0u);
            }
        }
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < 4) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
        for (int t = 0; t < 16; ++t) out[t * 128 + warp * 32 + lane] = v[t];
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc<512>(tmem);
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); u += 0x7fff + ((u >> 16) & 1); return u >> 16; }
static float bf2f(uint16_t b) { uint32_t u = uint32_t(b) << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
    const int nblk = 4, K = 64 * nblk;
    std::vector<float> W(128 * K), X(16 * K);
    srand(1);
    for (auto& w : W) w = bf2f(f2bf((rand() / float(RAND_MAX)) * 2 - 1));
    for (auto& x : X) x = bf2f(f2bf((rand() / float(RAND_MAX)) * 2 - 1));
    // weights: pre-tiled SW128 blocks (tiled_offset); activations: per k-block a
    // 16-row x 128-byte SW128 box (chunk c of row r at c ^ (r % 8))
    std::vector<uint16_t> wt(128 * K), xt(16 * K);
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < K; ++c) wt[tiled_offset(r, c, K)] = f2bf(W[r * K + c]);
    for (int b = 0; b < nblk; ++b)
        for (int r = 0; r < 16; ++r)
            for (int kk = 0; kk < 64; ++kk)
                xt[b * 1024 + r * 64 + (((kk >> 3) ^ (r & 7)) << 3) + (kk & 7)] = f2bf(X[r * K + b * 64 + kk]);
    __nv_bfloat16 *dw, *dx;
    float* dout;
    cudaMalloc(&dw, wt.size() * 2);
    cudaMalloc(&dx, xt.size() * 2);
    cudaMalloc(&dout, 16 * 128 * 4);
    cudaMemcpy(dw, wt.data(), wt.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, xt.data(), xt.size() * 2, cudaMemcpyHostToDevice);
    const int smem = nblk * (16384 + 2048) + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dout, 0, 16 * 128 * 4);
        k<<<1, 128, smem>>>(dw, dx, dout, mode, nblk);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> o(16 * 128);
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        for (int t = 0; t < 16; ++t)
            for (int r = 0; r < 128; ++r) {
                double ref = 0;
                for (int c = 0; c < K; ++c) ref += double(W[r * K + c]) * X[t * K + c];
                maxerr = std::max(maxerr, std::fabs(ref - o[t * 128 + r]));
            }
        printf("mode %d (%s): %s, max abs err %.3g  (o[0]=%.4f)\n", mode, mode ? "A in TMEM via tcgen05.cp" : "A in smem",
               cudaGetErrorString(e), maxerr, o[0]);
    }
    return 0;
}
