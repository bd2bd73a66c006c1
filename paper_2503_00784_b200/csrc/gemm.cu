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
// - Split-K across blockIdx.y so that tiles x splits fills the 148 SMs.  The
//   S split CTAs of one tile form a thread-block cluster (1 x S): each stages
//   its fp32 accumulator in its own shared memory, and after a cluster barrier
//   CTA rank r reduces the tokens t = r (mod S) by reading all S partials over
//   DSMEM in rank order (deterministic, and a token's result does not depend
//   on the pass width).  The fused epilogue (RoPE + paged-KV append, residual
//   add, SwiGLU, logits store) is applied right there — no global workspace.
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
constexpr int kMaxSplits = 16;  // cluster size (non-portable above 8)

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

    // ---- epilogue: cluster (DSMEM) split-K reduction + fused epilogue ----
    __syncwarp();
    mbar_wait(done, 0);
    __syncwarp();
    tc_fence_after();
    const int tid = threadIdx.x;
    const uint32_t S = static_cast<uint32_t>(a.splits);
    const uint32_t rank = S > 1 ? cluster_ctarank() : 0u;
    float* red = reinterpret_cast<float*>(smem);  // [kChunk][128] staging, reuses the ring
    const uint32_t red_addr = smem_u32(red);
    constexpr int kChunk = 64;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const GemmEpiParams& e = a.epi;
    // sum over the cluster's partials of element (t, r) of the current chunk
    auto csum = [&](int t, int r) -> float {
        if (S == 1) return red[t * 128 + r];
        const uint32_t off = static_cast<uint32_t>((t * 128 + r) * 4);
        // issue all remote loads first (independent), then add in rank order
        float v[kMaxSplits];
#pragma unroll
        for (uint32_t s2 = 0; s2 < kMaxSplits; ++s2)
            if (s2 < S) v[s2] = ld_dsmem_f32(dsmem_addr(red_addr + off, s2));
        float acc = 0.0f;
#pragma unroll
        for (uint32_t s2 = 0; s2 < kMaxSplits; ++s2)
            if (s2 < S) acc = __fadd_rn(acc, v[s2]);
        return acc;
    };
    for (int t0 = 0; t0 < a.w; t0 += kChunk) {
        const int tn = min(kChunk, a.w - t0);
        for (int c0 = 0; c0 < tn; c0 += 16) {
            float v[16];
            tmem_ld16(t_lane + t0 + c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < tn) red[(c0 + j) * 128 + warp * 32 + lane] = v[j];
        }
        if (S > 1) cluster_sync(); else __syncthreads();
        for (int t = static_cast<int>(rank); t < tn; t += static_cast<int>(S)) {
            const int tg = t0 + t;  // token index in the pass
            if (e.kind == kEpiStore) {
                e.out[static_cast<size_t>(tg) * a.n_out + m0 + tid] = csum(t, tid);
            } else if (e.kind == kEpiResidual) {
                float* x = e.out + static_cast<size_t>(tg) * a.n_out + m0 + tid;
                *x = __fadd_rn(*x, csum(t, tid));
            } else if (e.kind == kEpiSwiGLU) {
                if (tid < 64) {
                    const float g = csum(t, tid), u = csum(t, 64 + tid);
                    const float silu = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
                    e.out_bf[static_cast<size_t>(tg) * (a.n_out / 2) + blockIdx.x * 64 + tid] =
                        __float2bfloat16_rn(__fmul_rn(silu, u));
                }
            } else {  // kEpiQkvRope
                const ModelDims& md = e.m;
                const int hd = md.head_dim, half = hd / 2;
                const int q_dim = md.q_dim(), kv_dim = md.kv_dim();
                const int pos = e.ps->n_cached + tg;
                const int page = e.page_table[pos / e.page_size], slot = pos % e.page_size;
                if (m0 < q_dim + kv_dim) {
                    if (tid < 64) {
                        const int hl = tid / half, i = tid % half;
                        const int r0 = hl * hd + i;
                        const float av = csum(t, r0), bv = csum(t, r0 + half);
                        const float c = e.rope_cos[static_cast<size_t>(pos) * half + i];
                        const float sn = e.rope_sin[static_cast<size_t>(pos) * half + i];
                        const float lo = __fmaf_rn(av, c, -__fmul_rn(bv, sn));
                        const float hi = __fmaf_rn(bv, c, __fmul_rn(av, sn));
                        const int grow = m0 + r0;
                        if (grow < q_dim) {
                            float* qd = e.q_out + static_cast<size_t>(tg) * q_dim + grow;
                            qd[0] = lo;
                            qd[half] = hi;
                        } else {
                            const int kh = (grow - q_dim) / hd;
                            __nv_bfloat16* kd =
                                e.kv_pool + kv_offset(md, e.page_size, page, e.layer, 0, kh, slot) + i;
                            kd[0] = __float2bfloat16_rn(lo);
                            kd[half] = __float2bfloat16_rn(hi);
                        }
                    }
                } else {
                    const int ve = m0 + tid - q_dim - kv_dim;
                    e.kv_pool[kv_offset(md, e.page_size, page, e.layer, 1, ve / hd, slot) +
                              ve % hd] = __float2bfloat16_rn(csum(t, tid));
                }
            }
        }
        if (S > 1) cluster_sync(); else __syncthreads();
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
    for (int s = 1; s <= kMaxSplits; ++s) {
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
                        int w, int nt, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                        cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gemm_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             220 * 1024);
        cudaFuncSetAttribute(gemm_skinny_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
    a.epi = epi;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.tiles, plan.splits, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = plan.smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = plan.splits;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_skinny_kernel, *map_w, *map_x, a);
}

}  // namespace dd
