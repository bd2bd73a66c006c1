// Skinny weight-streaming GEMM for the target verification pass (sm_100a).
//
// The verification pass multiplies W <= 256 new-token activations by every
// weight matrix of the target once, so it is bound by streaming the weights
// from HBM.  Layout is swap-AB:
//
//   D[128 weight rows, NT tokens] (+)= Wtile[128, K] . X[NT, K]^T
//
// Persistent, warp-specialised, stream-K:
// - One CTA per SM.  The (tile, k-block) space of the matrix is cut into P
//   equal contiguous ranges, one per CTA, so every SM streams the same number
//   of weight bytes with no waves and no tail.  A range crossing a tile
//   boundary yields one "segment" per tile it touches.
// - Weights are stored pre-tiled and pre-swizzled in HBM (common.cuh
//   tiled_offset): a CTA's range is ONE contiguous run of 16 KiB blocks, each
//   loaded by a single cp.async.bulk into the SW128 K-major image UMMA
//   expects, with an evict-first policy and an L2 prefetch running ahead of
//   the smem ring.  Activations (B) come through a TMA tensor map (L2-resident).
// - warp 0: producer; warp 1: single-thread tcgen05.mma issuer (M=128,
//   N=NT, K=16) into one of two TMEM accumulators; warps 2-5: epilogue
//   (tcgen05.ld -> registers), overlapping the next segment's streaming.
// - Segment reduction: a tile covered by one segment is finished from
//   shared memory directly; otherwise each segment writes fp32 partials and
//   the last-arriving segment sums them in segment order (deterministic; the
//   partition depends only on the matrix shape, never on W, so a token's
//   result is independent of the pass width) and applies the fused epilogue
//   (RoPE + paged-KV append, residual add, SwiGLU, logits store).
// - Programmatic dependent launch: the first ring stages of weights are
//   requested before griddepcontrol.wait, so a GEMM starts streaming while
//   the previous kernel of the pass drains.
#include "common.cuh"
#include "gemm.h"
#include "gemm_epi.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace dd {

namespace {

using namespace gemm_dev;

__global__ void __launch_bounds__(kThreads, 2)
    gemm_sk_kernel(const __nv_bfloat16* __restrict__ w_tiled,
                   const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_x_lo, GemmArgs a) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int P = gridDim.x, c = blockIdx.x;
    const long T = static_cast<long>(a.tiles) * a.nkb;
    const long g0 = sk_begin(c, T, P), g1 = sk_begin(c + 1, T, P);
    const int len = static_cast<int>(g1 - g0);
    const uint32_t b_bytes = static_cast<uint32_t>(a.nt) * 128u;
    const uint32_t stage_bytes = kABytes + b_bytes * (a.split ? 2u : 1u);
    const int stages = a.stages;

    float* red = reinterpret_cast<float*>(smem + stages * stage_bytes);  // [kChunk][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + kChunk * 128);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    __shared__ int s_last;
    __shared__ float s_part[4 * kChunk];
    __shared__ float s_rn[kMaxPassTokens];  // RMSNorm factor per token of the consumed h
    __shared__ int s_page[kMaxPassTokens], s_slot[kMaxPassTokens];

    unsigned long long* tr =
        a.trace ? a.trace + 8 * static_cast<size_t>(blockIdx.x) : nullptr;
    auto stamp = [&](int i) {
        if (tr) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tr[i] = t;
        }
    };

    if (threadIdx.x == 0) {
        stamp(0);
        if (tr) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            tr[7] = smid;
        }
        tma_prefetch_desc(&map_x);
        if (a.split) tma_prefetch_desc(&map_x_lo);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiThreads);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        const uint32_t cols = static_cast<uint32_t>(a.tmem_buf * 2);
        if (cols <= 32) tmem_alloc<32>(tmem_slot);
        else if (cols <= 64) tmem_alloc<64>(tmem_slot);
        else if (cols <= 128) tmem_alloc<128>(tmem_slot);
        else if (cols <= 256) tmem_alloc<256>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_launch();  // the next kernel may start prefetching its weights
    if (threadIdx.x == 0) stamp(1);

    // first / last tile touched by this CTA
    const int tile_lo = len > 0 ? static_cast<int>(g0 / a.nkb) : 0;
    const int tile_hi = len > 0 ? static_cast<int>((g1 - 1) / a.nkb) : -1;

    if (warp == 0) {
        if (lane == 0 && len > 0) {
            // ---------------- producer ----------------
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const int nbox = a.nt >> 4;
            const int pre = min(stages, len);
            const int kPrefetch = a.prefetch;
            // timing experiment only (DD_GEMM_INTERLEAVE): lockstep-sequential addresses
            auto blk = [&](int i) -> const __nv_bfloat16* {
                if (a.interleave) {
                    const long pidx = static_cast<long>(i) * P + c;
                    return w_tiled + (pidx < T ? pidx : (g0 + i)) * 8192;
                }
                return w_tiled + (g0 + i) * 8192;
            };
            for (int i = 0; i < pre; ++i) {  // weights do not depend on the previous kernel
                mbar_arrive_expect_tx(&full[i], stage_bytes);
                bulk_load(smem + i * stage_bytes, blk(i), kABytes, &full[i], pol_w);
            }
            for (int i = pre; i < min(len, pre + kPrefetch); ++i)
                prefetch_l2(w_tiled + (g0 + i) * 8192, kABytes);
            griddep_wait();  // activations are produced by the previous kernel
            stamp(2);
            for (int i = 0; i < len; ++i) {
                const int s = i % stages;
                const uint32_t use = static_cast<uint32_t>(i / stages);
                uint8_t* sa = smem + s * stage_bytes;
                if (i >= pre) {
                    mbar_wait(&empty[s], (use & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&full[s], stage_bytes);
                    bulk_load(sa, blk(i), kABytes, &full[s], pol_w);

                }
                const int kc = static_cast<int>((g0 + i) % a.nkb) * kBlockK;
                for (int r = 0; r < nbox; ++r)
                    tma_load_2d(sa + kABytes + r * 2048, &map_x, &full[s], kc, r * 16, pol_x);
                if (a.split)
                    for (int r = 0; r < nbox; ++r)
                        tma_load_2d(sa + kABytes + b_bytes + r * 2048, &map_x_lo, &full[s], kc,
                                    r * 16, pol_x);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && len > 0) {
            // ---------------- MMA issuer ----------------
            const uint32_t idesc = idesc_bf16_f32(kBlockM, a.nt);
            int i = 0;
            for (int tile = tile_lo, u = 0; tile <= tile_hi; ++tile, ++u) {
                const long lo = max(g0, static_cast<long>(tile) * a.nkb);
                const long hi = min(g1, static_cast<long>(tile + 1) * a.nkb);
                const int b = u & 1;
                if (u >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>(((u >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t acc = tmem + static_cast<uint32_t>(b * a.tmem_buf);
                for (long g = lo; g < hi; ++g, ++i) {
                    const int s = i % stages;
                    const uint32_t use = static_cast<uint32_t>(i / stages);
                    mbar_wait(&full[s], use & 1u);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * stage_bytes);
                    const uint64_t adesc = sw128_kmajor_desc(sa);
                    const uint64_t bdesc = sw128_kmajor_desc(sa + kABytes);
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k)
                        umma_bf16(acc, adesc + 2 * k, bdesc + 2 * k, idesc,
                                  (g != lo || k != 0) ? 1u : 0u);
                    if (a.split) {  // W.(x_hi + x_lo): the lo halves into the same accumulator
                        const uint64_t bdesc_lo = sw128_kmajor_desc(sa + kABytes + b_bytes);
#pragma unroll
                        for (int k = 0; k < kBlockK / 16; ++k)
                            umma_bf16(acc, adesc + 2 * k, bdesc_lo + 2 * k, idesc, 1u);
                    }
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[b]);
            }
            stamp(3);
        }
    } else {
        // ---------------- epilogue warps 2..5 ----------------
        // One output row per thread (row == tid == TMEM lane).  Per-token pass
        // constants (RMSNorm factor of the consumed h, KV page / slot) are built
        // once per launch, after the previous kernel of the pass completed.
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        const int tid = threadIdx.x - 64;  // 0..127
        const GemmEpiParams& ep = a.epi;
        griddep_wait();
        for (int t = tid; t < a.w; t += kEpiThreads) {
            if (ep.ss_in != nullptr) {
                const float* ssr = ep.ss_in + static_cast<size_t>(t) * ep.ss_tiles;
                float acc = 0.0f;
                for (int i0 = 0; i0 < ep.ss_tiles; i0 += 16) {
                    float v16[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) v16[j] = i0 + j < ep.ss_tiles ? __ldcg(ssr + i0 + j) : 0.0f;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (i0 + j < ep.ss_tiles) acc = __fadd_rn(acc, v16[j]);
                }
                s_rn[t] = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(acc, static_cast<float>(ep.norm_d)), ep.eps));
            }
            if (ep.kind == kEpiQkvRope) {
                const int pos = ep.ps->n_cached + t;
                s_page[t] = ep.page_table[pos / ep.page_size];
                s_slot[t] = pos % ep.page_size;
            }
        }
        epi_bar();
        const bool resid = ep.kind == kEpiResidual;
        for (int tile = tile_lo, u = 0; tile <= tile_hi; ++tile, ++u) {
            const int first = sk_owner(static_cast<long>(tile) * a.nkb, T, P);
            const int last = sk_owner(static_cast<long>(tile + 1) * a.nkb - 1, T, P);
            const int nseg = last - first + 1, seg = c - first;
            const int b = u & 1;
            const float gcol = (resid && ep.u_out != nullptr) ? ep.gain[tile * kBlockM + row] : 1.0f;
            // residual rows of this tile's chunk (issued before the data is needed)
            auto load_x = [&](int t0, int tn, float* xv) {
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    xv[j] = (resid && j < tn)
                                ? __ldcg(ep.out + static_cast<size_t>(t0 + j) * a.n_out + tile * kBlockM + row)
                                : 0.0f;
            };
            auto scale = [&](int t0, int tn, float* v) {
                if (ep.ss_in == nullptr) return;
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (j < tn) v[j] = __fmul_rn(v[j], s_rn[t0 + j]);
            };
            mbar_wait(&tfull[b], static_cast<uint32_t>((u >> 1) & 1));
            if (tid == 0 && tile == tile_hi) stamp(6);  // this CTA's last accumulator landed
            __syncwarp();
            tc_fence_after();
            const uint32_t t_lane =
                tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * a.tmem_buf);
            if (nseg == 1) {
                for (int t0 = 0; t0 < a.w; t0 += kChunk) {
                    const int tn = min(kChunk, a.w - t0);
                    float xv[kChunk];
                    load_x(t0, tn, xv);
                    float v[16];
                    tmem_ld16(t_lane + t0, v);
                    if (t0 + kChunk >= a.w) {  // accumulator fully read
                        tc_fence_before();
                        mbar_arrive(&tempty[b]);
                    }
                    scale(t0, tn, v);
                    chunk_epilogue_rows(a, tile, t0, tn, v, xv, gcol, s_page, s_slot, red, s_part, row, tid);
                    epi_bar();
                }
            } else {
                float* part = a.ws + (static_cast<size_t>(tile) * a.max_seg + seg) * a.w * 128;
                for (int t0 = 0; t0 < a.w; t0 += 16) {
                    float v[16];
                    tmem_ld16(t_lane + t0, v);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (t0 + j < a.w) part[static_cast<size_t>(t0 + j) * 128 + row] = v[j];
                }
                tc_fence_before();
                mbar_arrive(&tempty[b]);
                __threadfence();
                epi_bar();
                if (tid == 0) {
                    const int prev = atomicAdd(&a.epi.counters[tile], 1);
                    s_last = (prev == nseg - 1);
                }
                epi_bar();
                if (s_last) {
                    __threadfence();
                    // this thread's row of every segment, all loads of a chunk in flight,
                    // summed in segment order
                    const float* base = a.ws + static_cast<size_t>(tile) * a.max_seg * a.w * 128 + row;
                    const size_t seg_stride = static_cast<size_t>(a.w) * 128;
                    for (int t0 = 0; t0 < a.w; t0 += kChunk) {
                        const int tn = min(kChunk, a.w - t0);
                        float xv[kChunk];
                        load_x(t0, tn, xv);
                        float v[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = 0.0f;
                        for (int s0 = 0; s0 < nseg; s0 += 4) {
                            float pv[4][16];
#pragma unroll
                            for (int k = 0; k < 4; ++k)
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    pv[k][j] = (s0 + k < nseg && j < tn)
                                                   ? __ldcg(base + (s0 + k) * seg_stride + static_cast<size_t>(t0 + j) * 128)
                                                   : 0.0f;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (s0 + k < nseg)
#pragma unroll
                                    for (int j = 0; j < 16; ++j) v[j] = __fadd_rn(v[j], pv[k][j]);
                        }
                        scale(t0, tn, v);
                        chunk_epilogue_rows(a, tile, t0, tn, v, xv, gcol, s_page, s_slot, red, s_part, row, tid);
                        epi_bar();
                    }
                    if (tid == 0) a.epi.counters[tile] = 0;
                }
            }
        }
        if (tid == 0) stamp(4);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        const uint32_t cols = static_cast<uint32_t>(a.tmem_buf * 2);
        if (cols <= 32) tmem_dealloc<32>(tmem);
        else if (cols <= 64) tmem_dealloc<64>(tmem);
        else if (cols <= 128) tmem_dealloc<128>(tmem);
        else if (cols <= 256) tmem_dealloc<256>(tmem);
        else tmem_dealloc<512>(tmem);
    }
    if (threadIdx.x == 0) stamp(5);
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

GemmPlan plan_gemm(int n_out, int k, int nt, int split) {
    static const int env_stages = getenv("DD_GEMM_STAGES") ? atoi(getenv("DD_GEMM_STAGES")) : 0;
    static const int env_ctas = getenv("DD_GEMM_CTAS") ? atoi(getenv("DD_GEMM_CTAS")) : 0;
    GemmPlan p{};
    p.tiles = n_out / kBlockM;
    p.nkb = k / kBlockK;
    const long T = static_cast<long>(p.tiles) * p.nkb;
    const uint32_t stage_bytes = kABytes + static_cast<uint32_t>(nt) * 128u * (split ? 2u : 1u);
    const uint32_t fixed = kChunk * 128 * 4 + 64 * 8 + 1024 + 64;
    const uint32_t budget = 110u * 1024u;
    int stages = static_cast<int>((budget - fixed) / stage_bytes);
    int per_sm = 2;  // two persistent CTAs per SM when the ring fits in ~110 KiB
    if (stages < 3) {
        stages = static_cast<int>((220u * 1024u - fixed) / stage_bytes);
        per_sm = 1;
    }
    stages = std::max(2, std::min(stages, 5));
    if (env_stages > 0) stages = env_stages;
    p.stages = stages;
    p.smem_bytes = static_cast<int>(stages * stage_bytes + fixed);
    int buf = 32;
    while (buf < nt) buf <<= 1;
    p.tmem_cols = 2 * buf;
    auto segs = [&](int ctas) {
        int ms = 1;
        for (int t = 0; t < p.tiles; ++t) {
            const int f = sk_owner(static_cast<long>(t) * p.nkb, T, ctas);
            const int l = sk_owner(static_cast<long>(t + 1) * p.nkb - 1, T, ctas);
            ms = std::max(ms, l - f + 1);
        }
        return ms;
    };
    p.ctas = static_cast<int>(std::min<long>(env_ctas > 0 ? env_ctas : kNumSMs * per_sm, T));
    while (segs(p.ctas) > kMaxSeg) p.ctas = std::max(1, p.ctas * 3 / 4);
    p.max_seg = segs(p.ctas);
    return p;
}

size_t gemm_ws_floats(const GemmPlan& p, int w) {
    return static_cast<size_t>(p.tiles) * p.max_seg * static_cast<size_t>(w) * 128;
}

static unsigned long long* g_trace = nullptr;
void gemm_set_trace(unsigned long long* buf) { g_trace = buf; }

cudaError_t launch_gemm(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x, int n_out, int k,
                        int w, int nt, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                        cudaStream_t stream, const CUtensorMap* map_x_lo) {
    // per device (a process may drive several GPUs: tensor-parallel ranks)
    static bool attr_set[kMaxDevices] = {};
    const int dev = current_device_slot();
    if (!attr_set[dev]) {
        cudaFuncSetAttribute(gemm_sk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             220 * 1024);
        attr_set[dev] = true;
    }
    GemmArgs a{};
    a.n_out = n_out;
    a.k = k;
    a.w = w;
    a.nt = nt;
    a.tiles = plan.tiles;
    a.nkb = plan.nkb;
    a.stages = plan.stages;
    a.max_seg = plan.max_seg;
    a.tmem_buf = plan.tmem_cols / 2;
    a.ws = ws;
    a.epi = epi;
    a.trace = g_trace;
    static const int env_pf = getenv("DD_GEMM_PREFETCH") ? atoi(getenv("DD_GEMM_PREFETCH")) : 0;
    a.prefetch = env_pf;
    static const int env_il = getenv("DD_GEMM_INTERLEAVE") ? atoi(getenv("DD_GEMM_INTERLEAVE")) : 0;
    a.interleave = env_il;
    a.split = map_x_lo != nullptr ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.ctas, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = plan.smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, gemm_sk_kernel, w_tiled, *map_x, map_x_lo ? *map_x_lo : *map_x, a);
}

}  // namespace dd

namespace dd {
void preload_gemm_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, gemm_sk_kernel);
}
}  // namespace dd
