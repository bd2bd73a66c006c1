// Micro-benchmark (scripts/micro; not product): stream pre-tiled weight blocks
// through 148 persistent CTAs into tcgen05.mma (M=128, N=16), weights as the A
// operand either straight from the shared-memory ring (mode 0) or staged into
// TMEM slots with tcgen05.cp (mode 1: one thread pumps copies while it waits,
// mode 2: copies in MMA order, no look-ahead).  Prints GB/s of weight bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2503_00784_b200/csrc
//   scripts/micro/tmem_stream.cu -o scripts/micro/tmem_stream_bench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace dd;

struct RP {
    int s = 0;
    uint32_t ph = 0, n = 0;
    __device__ void next(int S) { if (++s == S) { s = 0; ph ^= 1u; } ++n; }
};

__global__ void __launch_bounds__(128, 1)
stream_k(const __nv_bfloat16* w, long blocks_per_cta, float* out, int mode, int S, int NS) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* act = sm + S * 16384;  // 2 KiB static activation block
    uint64_t* wfull = reinterpret_cast<uint64_t*>(act + 2048);
    uint64_t* wempty = wfull + S;
    uint64_t* sfree = wempty + S;
    uint64_t* done = sfree + 16;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 1) tmem_alloc<512>(&slot);
    if (tid == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
        for (int j = 0; j < 16; ++j) mbar_init(&sfree[j], 1);
        mbar_init(done, 1);
        fence_barrier_init();
    }
    for (int i = tid; i < 2048 / 16; i += 128) reinterpret_cast<uint4*>(act)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const __nv_bfloat16* src = w + static_cast<size_t>(blockIdx.x) * blocks_per_cta * 8192;
    const uint32_t total = static_cast<uint32_t>(blocks_per_cta);
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        RP rp;
        for (uint32_t g = 0; g < total; ++g) {
            if (rp.n >= static_cast<uint32_t>(S)) mbar_wait(&wempty[rp.s], rp.ph ^ 1u);
            mbar_arrive_expect_tx(&wfull[rp.s], 16384);
            bulk_load(sm + rp.s * 16384, src + static_cast<size_t>(g) * 8192, 16384, &wfull[rp.s], pol);
            rp.next(S);
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t idesc = idesc_bf16_f32(128, 16);
        const uint64_t bdesc = sw128_kmajor_desc(smem_u32(act));
        const uint32_t acc = tmem, slot0 = tmem + 64;
        if (mode == 0) {
            RP rp;
            for (uint32_t g = 0; g < total; ++g) {
                mbar_wait(&wfull[rp.s], rp.ph);
                tc_fence_after();
                const uint64_t ad = sw128_kmajor_desc(smem_u32(sm + rp.s * 16384));
                for (int k = 0; k < 4; ++k) umma_bf16(acc, ad + 2 * k, bdesc + 2 * k, idesc, (g | k) ? 1u : 0u);
                umma_commit(&wempty[rp.s]);
                rp.next(S);
            }
        } else {
            RP cw, cs, ms;
            auto pump = [&]() {
                while (cw.n < total) {
                    if (cs.n >= static_cast<uint32_t>(NS) && !mbar_test_wait(&sfree[cs.s], cs.ph ^ 1u)) return;
                    if (!mbar_test_wait(&wfull[cw.s], cw.ph)) return;
                    tc_fence_after();
                    const uint64_t sd = sw128_kmajor_desc(smem_u32(sm + cw.s * 16384));
                    if (mode == 3) {  // 128x128b: 8 copies of 16 bytes per row
                        for (int k = 0; k < 8; ++k)
                            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(slot0 + cs.s * 32 + 4 * k), "l"(sd + k) : "memory");
                    } else {
                        for (int k = 0; k < 4; ++k) tmem_cp_128x256b(slot0 + cs.s * 32 + 8 * k, sd + 2 * k);
                    }
                    umma_commit(&wempty[cw.s]);
                    cw.next(S);
                    cs.next(NS);
                    if (mode == 2) return;
                }
            };
            for (uint32_t g = 0; g < total; ++g) {
                if (mode == 2) {
                    if (cs.n >= static_cast<uint32_t>(NS)) mbar_wait(&sfree[cs.s], cs.ph ^ 1u);
                    mbar_wait(&wfull[cw.s], cw.ph);
                    pump();
                } else {
                    while (cw.n <= ms.n) pump();
                }
                const uint32_t asl = slot0 + ms.s * 32;
                if (mode != 4)  // mode 4: copies only
                    for (int k = 0; k < 4; ++k) umma_bf16_ts(acc, asl + 8 * k, bdesc + 2 * k, idesc, (g | k) ? 1u : 0u);
                umma_commit(&sfree[ms.s]);
                ms.next(NS);
                if (mode != 2) pump();
            }
        }
        umma_commit(done);
    }
    __syncthreads();
    mbar_wait(done, 0);
    tc_fence_after();
    if (warp < 4) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
        if (blockIdx.x == 0) out[tid] = v[0];
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

int main() {
    const long per_cta = 4096;  // 64 MiB per CTA, 9.7 GB total
    const size_t n = static_cast<size_t>(per_cta) * 148 * 8192;
    __nv_bfloat16* w;
    if (cudaMalloc(&w, n * 2) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(w, 0, n * 2);
    float* out;
    cudaMalloc(&out, 4096);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Cfg { int mode, S, NS; } cfgs[] = {{0, 8, 0}, {0, 12, 0}, {1, 8, 14}, {1, 7, 14}, {2, 8, 14}, {1, 4, 14}, {1, 8, 4}, {3, 8, 14}, {4, 8, 14}};
    for (auto c : cfgs) {
        const int smem = c.S * 16384 + 2048 + 1024 + 64 * 8;
        cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            stream_k<<<148, 128, smem>>>(w, per_cta, out, c.mode, c.S, c.NS);
            cudaEventRecord(b);
            cudaError_t e = cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("mode %d S=%d NS=%d: %.3f ms  %.1f GB/s  (%s)\n", c.mode, c.S, c.NS, ms, n * 2 / ms / 1e6,
                       cudaGetErrorString(e));
        }
    }
    return 0;
}
