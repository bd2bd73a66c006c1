// Skinny weight-streaming GEMM for the target verification pass (sm_100a).
//
// The verification pass multiplies W <= 256 new-token activations by every
// weight matrix of the target once, so it is bound by streaming the weights
// from HBM.  Layout is swap-AB:
//
//   D[128 weight rows, NT tokens] (+)= Wtile[128, K] . X[NT, K]^T
//
// - A operand: a 128-row weight tile, K-major, fetched by TMA in 64-column
//   (128-byte) boxes with 128B swizzle and an evict-first L2 policy.
// - B operand: the NT (multiple of 16) activation rows, same layout, fetched
//   in 16-row boxes (evict-last: every CTA re-reads them from L2).
// - One elected thread issues tcgen05.mma (M=128, N=NT, K=16) into a TMEM
//   accumulator; tcgen05.commit releases each smem stage back to the TMA
//   producer through an mbarrier ring.
// - Split-K across blockIdx.y so that tiles x splits fills the 148 SMs; the
//   fp32 partials go to a workspace ws[split][token][row] and the consumer's
//   fused epilogue kernel reduces them in a fixed order (deterministic, and a
//   token's result does not depend on how many other tokens share the pass).
#include "common.cuh"
#include "gemm.h"

#include <algorithm>
#include <cstdio>

namespace dd {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;  // 16 KiB
constexpr int kTmemCols = 256;

__global__ void __launch_bounds__(128, 1)
    gemm_skinny_kernel(const __grid_constant__ CUtensorMap map_w,
                       const __grid_constant__ CUtensorMap map_x, GemmArgs a) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kBlockM;
    const int split = blockIdx.y;
    const int kb0 = split * a.kb_per_split;
    const int nkb = min(a.kb_per_split, a.k / kBlockK - kb0);
    const uint32_t b_bytes = static_cast<uint32_t>(a.nt) * 128u;
    const uint32_t stage_bytes = kABytes + b_bytes;
    const int stages = a.stages;

    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + stages;
    uint64_t* done = empty + stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map_w);
        tma_prefetch_desc(&map_x);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (threadIdx.x == 0) {
        // ---- TMA producer ----
        const uint64_t pol_w = policy_evict_first();
        const uint64_t pol_x = policy_evict_last();
        const int nbox = a.nt >> 4;
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % stages;
            const uint32_t use = static_cast<uint32_t>(kb / stages);
            mbar_wait(&empty[s], (use & 1u) ^ 1u);
            uint8_t* sa = smem + s * stage_bytes;
            uint8_t* sb = sa + kABytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            const int kc = (kb0 + kb) * kBlockK;
            tma_load_2d(sa, &map_w, &full[s], kc, m0, pol_w);
            for (int r = 0; r < nbox; ++r)
                tma_load_2d(sb + r * 2048, &map_x, &full[s], kc, r * 16, pol_x);
        }
    } else if (threadIdx.x == 32) {
        // ---- MMA issuer (single thread) ----
        const uint32_t idesc = idesc_bf16_f32(kBlockM, a.nt);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % stages;
            const uint32_t use = static_cast<uint32_t>(kb / stages);
            mbar_wait(&full[s], use & 1u);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * stage_bytes);
            const uint64_t adesc = sw128_kmajor_desc(sa);
            const uint64_t bdesc = sw128_kmajor_desc(sa + kABytes);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
                // +32 bytes along K inside the 128B swizzle atom = +2 in addr>>4
                umma_bf16(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            }
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }

    // ---- epilogue: TMEM -> registers -> fp32 partials (all 4 warps) ----
    __syncwarp();
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
    float* out = a.ws + static_cast<size_t>(split) * a.w * a.n_out;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int c0 = 0; c0 < a.nt; c0 += 16) {
        float v[16];
        tmem_ld16(t_lane + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (c0 + j < a.w) out[static_cast<size_t>(c0 + j) * a.n_out + row] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
#endif
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

}  // namespace

int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                   uint32_t box_rows) {
    auto fn = get_encode_fn();
    if (!fn) return -1;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBlockK), box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : -2;
}

GemmPlan plan_gemm(int n_out, int k, int nt) {
    GemmPlan p{};
    const int tiles = n_out / kBlockM;
    const int nkb = k / kBlockK;
    const uint32_t stage_bytes = kABytes + static_cast<uint32_t>(nt) * 128u;
    // two CTAs per SM when the ring fits in ~104 KiB, else one
    int stages = static_cast<int>(104u * 1024u / stage_bytes);
    int ctas_per_sm = 2;
    if (stages < 4) {
        stages = std::min(8, static_cast<int>(220u * 1024u / stage_bytes));
        ctas_per_sm = 1;
    }
    stages = std::min(stages, 8);
    // The split count depends only on the GEMM shape (never on nt), so a token's
    // fp32 reduction order is identical whatever the pass width: greedy outputs
    // do not depend on how tokens are batched into passes.
    const int slots = kNumSMs * 2;
    // choose split-K maximising wave efficiency, keeping >= 6 k-blocks per CTA
    int best_s = 1;
    double best_eff = -1.0;
    for (int s = 1; s <= 32; ++s) {
        const int kbps = (nkb + s - 1) / s;
        if (kbps < 6 && s > 1) break;
        const int real_s = (nkb + kbps - 1) / kbps;
        const int ctas = tiles * real_s;
        const int waves = (ctas + slots - 1) / slots;
        double eff = static_cast<double>(ctas) / (waves * slots);
        // mild preference for fewer waves (prologue/epilogue cost per CTA)
        eff -= 0.004 * waves;
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best_s = real_s;
        }
    }
    (void)ctas_per_sm;
    p.kb_per_split = (nkb + best_s - 1) / best_s;
    p.splits = (nkb + p.kb_per_split - 1) / p.kb_per_split;
    p.stages = stages;
    p.smem_bytes = static_cast<int>(stages * stage_bytes + (2 * stages + 1) * 8 + 16 + 1024);
    p.tiles = tiles;
    return p;
}

cudaError_t launch_gemm(const CUtensorMap* map_w, const CUtensorMap* map_x, int n_out, int k,
                        int w, int nt, const GemmPlan& plan, float* ws, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        attr_set = true;
    }
    GemmArgs a;
    a.n_out = n_out;
    a.k = k;
    a.w = w;
    a.nt = nt;
    a.kb_per_split = plan.kb_per_split;
    a.splits = plan.splits;
    a.stages = plan.stages;
    a.ws = ws;
    dim3 grid(plan.tiles, plan.splits);
    gemm_skinny_kernel<<<grid, 128, plan.smem_bytes, stream>>>(*map_w, *map_x, a);
    return cudaGetLastError();
}

}  // namespace dd
