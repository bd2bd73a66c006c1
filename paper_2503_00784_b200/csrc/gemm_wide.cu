// Prefill GEMM (wide passes, 17..128 new tokens) for sm_100a.
//
// The decode GEMM puts 128 weight rows on M and the few tokens on N.  For a
// prefill chunk that leaves the tensor core reading 8 KiB of shared memory per
// 128x128x16 MMA, and it runs several times below its peak.  Here the tokens
// are M (128, one TMEM lane per token) and the weights N = 256 rows, so each
// 128x256x16 MMA reads 4 KiB of activations + 8 KiB of weights:
//
//   D[128 tokens, 256 weight rows] (+)= X[128, K] . Wtile[256, K]^T
//
// Same persistent stream-K skeleton as gemm.cu (one CTA per SM, equal
// contiguous ranges of (256-row tile, k-block), TMEM double buffer of 2 x 256
// columns, warp-specialised producer / MMA / epilogue).  A 256-row tile is two
// consecutive pre-tiled 128-row tiles: one stage = two 16 KiB bulk copies of
// weights + one 128-row TMA box of activations.
//
// Epilogue: TMEM lane = token, so each epilogue thread owns one token's 256
// outputs and every fused epilogue is thread-local: RoPE pairs (i, i + hd/2),
// SwiGLU gate/up halves and the residual sum of squares of a 128-row tile all
// sit in the same thread.  Stream-K partials are stored [segment][row][token]
// (coalesced over threads); the last segment reduces them in segment order.
#include "common.cuh"
#include "gemm.h"
#include "gemm_epi.cuh"

#include <algorithm>
#include <cstdlib>

namespace dd {

namespace {

using gemm_dev::kABytes;
using gemm_dev::kBlockK;
using gemm_dev::sk_begin;
using gemm_dev::sk_segments;

constexpr int kWideM = 128;        // tokens per tile (TMEM lanes)
constexpr int kWideThreads = 192;  // producer, MMA, 4 epilogue warps
constexpr uint32_t kXBytes = kWideM * kBlockK * 2;  // 16 KiB of activations
// NW = weight rows per tile (256, or 128 for the d_model-output GEMMs, whose
// 32 row tiles would otherwise be split over ~9 stream-K segments each)
template <int NW>
struct WideCfg {
    static constexpr int kHalves = NW / 128;
    static constexpr uint32_t kWBytes = kHalves * kABytes;
    static constexpr uint32_t kStageBytes = kWBytes + kXBytes;
};

__device__ __forceinline__ void wide_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// 16 consecutive weight-row columns [c0, c0 + 16) of this thread's token.
template <int NCH, int KS>
__device__ __forceinline__ void load_cols_n(uint32_t t_lane, int c0, const float* part_tok, int nseg,
                                            size_t seg_stride, float (*v)[16]) {
    // NCH consecutive 16-column chunks: this CTA's own segment (segment 0, the
    // designated reducer) from TMEM plus the other segments' partials
    // ([segment][col / 4][token][4]) in segment order.  Every partial load is
    // issued before the TMEM loads (whose wait is a compiler barrier), so one
    // round trip covers all NCH chunks of up to KS segments.
    for (int s0 = 1; s0 < nseg || s0 == 1; s0 += KS) {
        float4 pv[KS][NCH][4];
#pragma unroll
        for (int k = 0; k < KS; ++k)
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    pv[k][ch][q4] = s0 + k < nseg
                                        ? __ldcg(reinterpret_cast<const float4*>(
                                              part_tok + (s0 + k) * seg_stride +
                                              static_cast<size_t>(((c0 + 16 * ch) >> 2) + q4) * kWideM * 4))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        if (s0 == 1) {
            uint32_t r[NCH][16];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) tmem_ld16_async(t_lane + c0 + 16 * ch, r[ch]);
            tmem_wait_ld();
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int j = 0; j < 16; ++j) v[ch][j] = __uint_as_float(r[ch][j]);
        }
#pragma unroll
        for (int k = 0; k < KS; ++k)
            if (s0 + k < nseg)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4) {
                        v[ch][4 * q4] = __fadd_rn(v[ch][4 * q4], pv[k][ch][q4].x);
                        v[ch][4 * q4 + 1] = __fadd_rn(v[ch][4 * q4 + 1], pv[k][ch][q4].y);
                        v[ch][4 * q4 + 2] = __fadd_rn(v[ch][4 * q4 + 2], pv[k][ch][q4].z);
                        v[ch][4 * q4 + 3] = __fadd_rn(v[ch][4 * q4 + 3], pv[k][ch][q4].w);
                    }
        if (nseg <= 1) break;
    }
}
__device__ __forceinline__ void load_cols(uint32_t t_lane, int c0, const float* part_tok, int nseg,
                                          size_t seg_stride, float* v) {
    load_cols_n<1, 4>(t_lane, c0, part_tok, nseg, seg_stride, reinterpret_cast<float(*)[16]>(v));
}

__device__ __forceinline__ uint32_t bf2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// 16 bf16 (32 bytes, 16-byte aligned) from fp32
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* dst, const float* v) {
    uint4 a, b;
    a.x = bf2(v[0], v[1]);
    a.y = bf2(v[2], v[3]);
    a.z = bf2(v[4], v[5]);
    a.w = bf2(v[6], v[7]);
    b.x = bf2(v[8], v[9]);
    b.y = bf2(v[10], v[11]);
    b.z = bf2(v[12], v[13]);
    b.w = bf2(v[14], v[15]);
    reinterpret_cast<uint4*>(dst)[0] = a;
    reinterpret_cast<uint4*>(dst)[1] = b;
}

}  // namespace

// Fused epilogue of one NW-row weight tile for this thread's token (TMEM lane
// row; `tok` = the token's row in the pass, `valid` = tok < w): segment sums,
// RMSNorm scaling, and the store / residual + deferred-norm producer / SwiGLU /
// RoPE + paged-KV append of gemm_epi.cuh, written thread-locally.  Shared by the
// stream-K wide GEMM and the multi-tile prefill GEMM.
template <int NW>
__device__ __forceinline__ void wide_tile_epilogue(const GemmArgs& a, uint32_t t_lane, const float* pbase,
                                                   int nsum, size_t seg_stride, int tile, int tok, bool valid,
                                                   float rn, int page, int slot, int pos) {
    constexpr int kWideN = NW;
    constexpr int kHalves = WideCfg<NW>::kHalves;
    const GemmEpiParams& e = a.epi;
    const int tiles128 = a.n_out / 128;
    const int m0 = tile * kWideN;
    if (e.kind == kEpiStore || e.kind == kEpiResidual) {
        for (int h = 0; h < kHalves; ++h) {  // 128-row halves (ss tiles)
            float ss = 0.0f;
            for (int c1 = h * 128; c1 < h * 128 + 128; c1 += 32) {
                // residual rows requested first, then 2 chunks of partial sums
                // and accumulators in one round trip
                float4 xr[2][4];
                if (e.kind == kEpiResidual && valid)
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch)
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4)
                            xr[ch][q4] = __ldcg(reinterpret_cast<const float4*>(
                                                    e.out + static_cast<size_t>(tok) * a.n_out + m0 + c1 + 16 * ch) + q4);
                float v2[2][16];
                load_cols_n<2, 2>(t_lane, c1, pbase, nsum, seg_stride, v2);
                if (!valid) continue;
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const int c0 = c1 + 16 * ch;
                    float* v = v2[ch];
                    if (e.ss_in != nullptr)
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = __fmul_rn(v[j], rn);
                    float* dst = e.out + static_cast<size_t>(tok) * a.n_out + m0 + c0;
                    if (e.kind == kEpiResidual) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            v[4 * q4] = __fadd_rn(xr[ch][q4].x, v[4 * q4]);
                            v[4 * q4 + 1] = __fadd_rn(xr[ch][q4].y, v[4 * q4 + 1]);
                            v[4 * q4 + 2] = __fadd_rn(xr[ch][q4].z, v[4 * q4 + 2]);
                            v[4 * q4 + 3] = __fadd_rn(xr[ch][q4].w, v[4 * q4 + 3]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    if (e.kind == kEpiResidual && e.u_out != nullptr) {
                        float uv[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            uv[j] = __fmul_rn(v[j], e.gain[m0 + c0 + j]);
                            ss = __fmaf_rn(v[j], v[j], ss);
                        }
                        store_bf16x16(e.u_out + static_cast<size_t>(tok) * a.n_out + m0 + c0, uv);
                    }
                }
            }
            if (e.kind == kEpiResidual && e.u_out != nullptr && valid)
                e.ss_out[static_cast<size_t>(tok) * tiles128 + kHalves * tile + h] = ss;
        }
    } else if (e.kind == kEpiSwiGLU) {
        const int ffn = a.n_out / 2;
        for (int h = 0; h < kHalves; ++h)
            for (int k = 0; k < 4; ++k) {
                float g[16], up[16];
                load_cols(t_lane, h * 128 + 16 * k, pbase, nsum, seg_stride, g);
                load_cols(t_lane, h * 128 + 64 + 16 * k, pbase, nsum, seg_stride, up);
                if (!valid) continue;
                float av[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float gv = __fmul_rn(g[j], rn), uv = __fmul_rn(up[j], rn);
                    // fast exp / divide: prefill-only activations (the decode
                    // epilogue keeps the IEEE forms the oracle mirrors)
                    const float silu = __fdividef(gv, 1.0f + __expf(-gv));
                    av[j] = __fmul_rn(silu, uv);
                }
                store_bf16x16(e.out_bf + static_cast<size_t>(tok) * ffn + (kHalves * tile + h) * 64 + 16 * k, av);
            }
    } else {  // kEpiQkvRope
        const ModelDims& md = e.m;
        const int hd = md.head_dim, half = hd / 2;
        const int q_dim = md.q_dim(), kv_dim = md.kv_dim();
        for (int h = 0; h < kHalves; ++h) {
            const int r0 = m0 + h * 128;  // first weight row of this 128-row half
            if (r0 < q_dim + kv_dim) {
                // pairs (i, i + half) of every head in the half
                for (int hb = 0; hb < 128; hb += hd)
                    for (int i0 = 0; i0 < half; i0 += 16) {
                        float lo_v[16], hi_v[16];
                        load_cols(t_lane, h * 128 + hb + i0, pbase, nsum, seg_stride, lo_v);
                        load_cols(t_lane, h * 128 + hb + i0 + half, pbase, nsum, seg_stride, hi_v);
                        if (!valid) continue;
                        const int grow = r0 + hb;  // first row of the head
                        float lo16[16], hi16[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int i = i0 + j;
                            const float av = __fmul_rn(lo_v[j], rn), bv = __fmul_rn(hi_v[j], rn);
                            const float cs = e.rope_cos[static_cast<size_t>(pos) * half + i];
                            const float sn = e.rope_sin[static_cast<size_t>(pos) * half + i];
                            lo16[j] = __fmaf_rn(av, cs, -__fmul_rn(bv, sn));
                            hi16[j] = __fmaf_rn(bv, cs, __fmul_rn(av, sn));
                        }
                        if (grow < q_dim) {
                            float* qd = e.q_out + static_cast<size_t>(tok) * q_dim + grow + i0;
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4) {
                                reinterpret_cast<float4*>(qd)[q4] =
                                    make_float4(lo16[4 * q4], lo16[4 * q4 + 1], lo16[4 * q4 + 2], lo16[4 * q4 + 3]);
                                reinterpret_cast<float4*>(qd + half)[q4] =
                                    make_float4(hi16[4 * q4], hi16[4 * q4 + 1], hi16[4 * q4 + 2], hi16[4 * q4 + 3]);
                            }
                        } else {
                            __nv_bfloat16* kd = e.kv_pool +
                                kv_offset(md, e.page_size, page, e.layer, 0, (grow - q_dim) / hd, slot) + i0;
                            store_bf16x16(kd, lo16);
                            store_bf16x16(kd + half, hi16);
                        }
                    }
            } else {
                for (int c0 = 0; c0 < 128; c0 += 16) {
                    float v[16];
                    load_cols(t_lane, h * 128 + c0, pbase, nsum, seg_stride, v);
                    if (!valid) continue;
                    float vv[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) vv[j] = __fmul_rn(v[j], rn);
                    const int ve = r0 + c0 - q_dim - kv_dim;  // 16 dims of one kv head
                    store_bf16x16(e.kv_pool + kv_offset(md, e.page_size, page, e.layer, 1, ve / hd, slot) + ve % hd, vv);
                }
            }
        }
    }
}

template <int NW>
__global__ void __launch_bounds__(kWideThreads, 1)
    gemm_wide_kernel(const __nv_bfloat16* __restrict__ w_tiled, const __grid_constant__ CUtensorMap map_x,
                     GemmArgs a) {
    constexpr int kWideN = NW;
    constexpr int kHalves = WideCfg<NW>::kHalves;
    constexpr uint32_t kWBytes = WideCfg<NW>::kWBytes;
    constexpr uint32_t kStageBytes = WideCfg<NW>::kStageBytes;
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int P = gridDim.x, c = blockIdx.x;
    const int tiles = a.n_out / kWideN;  // NW-row tiles
    const long T = static_cast<long>(tiles) * a.nkb;
    const long g0 = sk_begin(c, T, P), g1 = sk_begin(c + 1, T, P);
    const int len = static_cast<int>(g1 - g0);
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    __shared__ int s_last;
    unsigned long long* tr = a.trace ? a.trace + 8 * static_cast<size_t>(blockIdx.x) : nullptr;
    auto stamp = [&](int i) {
        if (tr) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tr[i] = t;
        }
    };

    if (threadIdx.x == 0) {
        stamp(0);
        tma_prefetch_desc(&map_x);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<2 * NW>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    const int tile_lo = len > 0 ? static_cast<int>(g0 / a.nkb) : 0;
    const int tile_hi = len > 0 ? static_cast<int>((g1 - 1) / a.nkb) : -1;

    if (warp == 0) {
        if (lane == 0 && len > 0) {
            // ---------------- producer ----------------
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const int nkb = a.nkb;
            auto wsrc = [&](long g, int half) {
                const long tile = g / nkb, kb = g % nkb;
                return w_tiled + (static_cast<size_t>(kHalves * tile + half) * nkb + kb) * 8192;
            };
            // weights do not depend on the previous kernel: the first S stages are
            // requested before griddepcontrol.wait, the activations after it
            const int pre = min(S, len);
            for (int i = 0; i < pre; ++i) {
                uint8_t* st = smem + i * kStageBytes;
                mbar_arrive_expect_tx(&full[i], kStageBytes);
#pragma unroll
                for (int hh = 0; hh < kHalves; ++hh)
                    bulk_load(st + hh * kABytes, wsrc(g0 + i, hh), kABytes, &full[i], pol_w);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
            stamp(2);
            int s = 0;
            uint32_t ph = 0;
            int kb = static_cast<int>(g0 % nkb);
            for (int i = 0; i < len; ++i) {
                uint8_t* st = smem + s * kStageBytes;
                if (i >= pre) {
                    mbar_wait(&empty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
                    for (int hh = 0; hh < kHalves; ++hh)
                        bulk_load(st + hh * kABytes, wsrc(g0 + i, hh), kABytes, &full[s], pol_w);
                }
                tma_load_2d(st + kWBytes, &map_x, &full[s], kb * kBlockK, 0, pol_x);
                if (++kb == nkb) kb = 0;
                if (++s == S) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && len > 0) {
            // ---------------- MMA issuer ----------------
            const uint32_t idesc = idesc_bf16_f32(kWideM, kWideN);
            int s = 0;
            uint32_t ph = 0;
            for (int tile = tile_lo, u = 0; tile <= tile_hi; ++tile, ++u) {
                const long lo = max(g0, static_cast<long>(tile) * a.nkb);
                const long hi = min(g1, static_cast<long>(tile + 1) * a.nkb);
                const int b = u & 1;
                if (u >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>(((u >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t acc = tmem + static_cast<uint32_t>(b * kWideN);
                for (long g = lo; g < hi; ++g) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sw = smem_u32(smem + s * kStageBytes);
                    const uint64_t bdesc = sw128_kmajor_desc(sw);             // weights: N = 256
                    const uint64_t adesc = sw128_kmajor_desc(sw + kWBytes);   // tokens:  M = 128
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k)
                        umma_bf16(acc, adesc + 2 * k, bdesc + 2 * k, idesc, (g != lo || k != 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                umma_commit(&tfull[b]);
            }
            stamp(3);
        }
    } else {
        // ---------------- epilogue warps 2..5: thread = token ----------------
        const int q = warp & 3;
        const int tok = q * 32 + lane;  // TMEM lane
        const int tid = threadIdx.x - 64;
        const GemmEpiParams& e = a.epi;
        const bool valid = tok < a.w;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        // pass-level constants of this thread's token
        float rn = 1.0f;
        if (e.ss_in != nullptr && valid) {
            const float* ssr = e.ss_in + static_cast<size_t>(tok) * e.ss_tiles;
            float acc = 0.0f;
            for (int i0 = 0; i0 < e.ss_tiles; i0 += 16) {
                float v16[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) v16[j] = i0 + j < e.ss_tiles ? __ldcg(ssr + i0 + j) : 0.0f;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (i0 + j < e.ss_tiles) acc = __fadd_rn(acc, v16[j]);
            }
            rn = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(acc, static_cast<float>(e.norm_d)), e.eps));
        }
        int page = 0, slot = 0, pos = 0;
        if (e.kind == kEpiQkvRope) {
            pos = e.ps->n_cached + tok;
            page = e.page_table[pos / e.page_size];
            slot = pos % e.page_size;
        }
        const int tiles128 = a.n_out / 128;
        for (int tile = tile_lo, u = 0; tile <= tile_hi; ++tile, ++u) {
            int nseg, seg;
            sk_segments(tile, a.nkb, T, P, c, &nseg, &seg);
            const int b = u & 1;
            mbar_wait(&tfull[b], static_cast<uint32_t>((u >> 1) & 1));
            if (tid == 0 && tile == tile_hi) stamp(6);
            __syncwarp();
            tc_fence_after();
            const uint32_t t_lane = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * kWideN);
            const size_t seg_stride = static_cast<size_t>(kWideN) * kWideM;
            float* tile_part = a.ws + static_cast<size_t>(tile) * a.max_seg * seg_stride;
            int nsum = 1;  // segments summed into this tile (>1: this CTA is the reducer)
            if (nseg > 1) {
                if (seg != 0) {
                    // not the designated reducer: store this segment's partial
                    // ([segment][col / 4][token][4], coalesced) and release-add the counter
                    float* mine = tile_part + seg * seg_stride + static_cast<size_t>(tok) * 4;
                    for (int c0 = 0; c0 < kWideN; c0 += 64) {  // 4 TMEM loads in flight
                        uint32_t r[4][16];
#pragma unroll
                        for (int k = 0; k < 4; ++k) tmem_ld16_async(t_lane + c0 + 16 * k, r[k]);
                        tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < 4; ++k)
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4)
                                *reinterpret_cast<float4*>(mine + static_cast<size_t>(((c0 + 16 * k) >> 2) + q4) * kWideM * 4) =
                                    make_float4(__uint_as_float(r[k][4 * q4]), __uint_as_float(r[k][4 * q4 + 1]),
                                                __uint_as_float(r[k][4 * q4 + 2]), __uint_as_float(r[k][4 * q4 + 3]));
                    }
                    tc_fence_before();
                    mbar_arrive(&tempty[b]);
                    wide_bar();  // every partial store happens-before the release
                    if (tid == 0)
                        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&e.counters[tile]) : "memory");
                    continue;
                }
                // segment 0 finishes last (end of its CTA's range): wait for the others
                if (tid == 0) {
                    int v;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(&e.counters[tile]) : "memory");
                    } while (v < nseg - 1);
                    e.counters[tile] = 0;
                }
                wide_bar();
                nsum = nseg;
            }
            const float* pbase = tile_part + static_cast<size_t>(tok) * 4;
            wide_tile_epilogue<NW>(a, t_lane, pbase, nsum, seg_stride, tile, tok, valid, rn, page, slot, pos);
            tc_fence_before();
            mbar_arrive(&tempty[b]);
        }
    }
    if (threadIdx.x == 64) stamp(4);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<2 * NW>(tmem);
    if (threadIdx.x == 0) stamp(5);
#endif
}

GemmPlan plan_gemm_wide(int n_out, int k, int sm_avail) {
    GemmPlan p{};
    // 128-row tiles when 256-row tiles would leave fewer than 64 of them
    // 128-row weight tiles (measured: 256-row tiles, whose fewer and larger
    // stream-K partials lengthen the reducers' tails, make a 128-token pass 9%
    // slower; DD_WIDE_NW=256 restores them where n_out allows)
    static const int env_nw = getenv("DD_WIDE_NW") ? atoi(getenv("DD_WIDE_NW")) : 128;
    // CTAs for the d_model-output GEMMs (32 tiles): 96 = exactly 3 stream-K
    // segments per tile (64: 2 per tile but 57% of the SMs stream; 148: ragged)
    static const int env_small = getenv("DD_WIDE_SMALL_CTAS") ? atoi(getenv("DD_WIDE_SMALL_CTAS")) : 96;
    const int nw = (env_nw == 256 && n_out % 256 == 0) ? 256 : 128;
    p.tiles = n_out / nw;
    p.nkb = k / kBlockK;
    const long T = static_cast<long>(p.tiles) * p.nkb;
    const uint32_t stage = (nw == 256 ? WideCfg<256>::kStageBytes : WideCfg<128>::kStageBytes);
    p.stages = nw == 256 ? 4 : 6;
    p.smem_bytes = static_cast<int>(p.stages * stage + 1024 + 64 * 8);
    p.tmem_cols = 2 * nw;
    // the 4096-output GEMMs have only 32 row tiles: fewer CTAs keep their
    // stream-K segments per tile (and the last arriver's reduction) short
    static const int env_big = getenv("DD_WIDE_BIG_CTAS") ? atoi(getenv("DD_WIDE_BIG_CTAS")) : 0;
    int big = kNumSMs;
    if (env_big == -1) big = p.tiles / ((p.tiles + kNumSMs - 1) / kNumSMs);  // whole tiles per CTA
    else if (env_big > 0) big = env_big;
    p.ctas = static_cast<int>(std::min<long>(p.tiles >= 64 ? big : env_small, T));
    // the designated reducers wait for their segments: every CTA must be able to
    // be resident at once (sm_avail < 148 when other work may hold SMs)
    p.ctas = std::min(p.ctas, std::max(1, sm_avail));
    int ms = 1;
    for (int t = 0; t < p.tiles; ++t) {
        const int f = gemm_dev::sk_owner(static_cast<long>(t) * p.nkb, T, p.ctas);
        int nseg, seg;
        sk_segments(t, p.nkb, T, p.ctas, f, &nseg, &seg);
        ms = std::max(ms, nseg);
    }
    p.max_seg = ms;
    return p;
}

size_t gemm_wide_ws_floats(const GemmPlan& p) {
    return static_cast<size_t>(p.tiles) * p.max_seg * (p.tmem_cols / 2) * kWideM;
}

static unsigned long long* g_wide_trace = nullptr;
static size_t g_wide_trace_launch = 0;
void gemm_wide_set_trace(unsigned long long* buf) {
    g_wide_trace = buf;
    g_wide_trace_launch = 0;
}

cudaError_t launch_gemm_wide(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x128, int n_out, int k,
                             int w, const GemmPlan& plan, float* ws, const GemmEpiParams& epi,
                             cudaStream_t stream) {
    static bool attr_set[kMaxDevices] = {};  // per device: TP ranks of one process
    const int dev = current_device_slot();
    if (!attr_set[dev]) {
        cudaFuncSetAttribute(gemm_wide_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(gemm_wide_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr_set[dev] = true;
    }
    GemmArgs a{};
    a.n_out = n_out;
    a.k = k;
    a.w = w;
    a.nt = kWideM;
    a.tiles = plan.tiles;
    a.nkb = plan.nkb;
    a.stages = plan.stages;
    a.max_seg = plan.max_seg;
    a.tmem_buf = plan.tmem_cols / 2;
    a.ws = ws;
    a.epi = epi;
    a.trace = g_wide_trace ? g_wide_trace + (g_wide_trace_launch++) * 8 * kNumSMs : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(plan.ctas, 1, 1);
    cfg.blockDim = dim3(kWideThreads, 1, 1);
    cfg.dynamicSmemBytes = plan.smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (plan.tmem_cols == 512) return cudaLaunchKernelEx(&cfg, gemm_wide_kernel<256>, w_tiled, *map_x128, a);
    return cudaLaunchKernelEx(&cfg, gemm_wide_kernel<128>, w_tiled, *map_x128, a);
}

}  // namespace dd

// ---------------------------------------------------------------- prefill GEMM
// Long prompts: one pass over up to kMaxPrefillTokens
// tokens so every weight tile is streamed from HBM once for the whole prompt
// instead of once per 128-token chunk.  Work unit = (128-token tile m, NW-row
// weight tile n) over the full K; units are numbered n-major (m fastest), so
// the CTAs running at the same time share a few weight tiles (one HBM read,
// then L2 hits) while the prompt's activations (w x K bf16) stay L2-resident.
// No stream-K: with >= 148 units every SM has whole units.  Same warp roles,
// TMEM double buffer and thread-local epilogue (wide_tile_epilogue) as the
// stream-K wide GEMM above; TMEM lane = token row of the unit's m tile.
namespace dd {

template <int NW>
__global__ void __launch_bounds__(kWideThreads, 1)
    gemm_prefill_kernel(const __nv_bfloat16* __restrict__ w_tiled, const __grid_constant__ CUtensorMap map_x,
                        GemmArgs a) {
    constexpr int kHalves = WideCfg<NW>::kHalves;
    constexpr uint32_t kWBytes = WideCfg<NW>::kWBytes;
    constexpr uint32_t kStageBytes = WideCfg<NW>::kStageBytes;
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int P = gridDim.x, c = blockIdx.x;
    const int m_tiles = (a.w + kWideM - 1) / kWideM;
    const int units = m_tiles * (a.n_out / NW);
    const int nkb = a.nkb;
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&map_x);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<2 * NW>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer ----------------
            const uint64_t pol_w = policy_evict_normal();  // reused by the other m tiles
            const uint64_t pol_x = policy_evict_last();
            int s = 0;
            uint32_t ph = 0, n_issued = 0;
            bool waited = false;
            for (int u = c; u < units; u += P) {
                const int n = u / m_tiles, m = u % m_tiles;
                for (int kb = 0; kb < nkb; ++kb) {
                    uint8_t* st = smem + s * kStageBytes;
                    if (n_issued >= static_cast<uint32_t>(S)) mbar_wait(&empty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
                    for (int hh = 0; hh < kHalves; ++hh)
                        bulk_load(st + hh * kABytes,
                                  w_tiled + (static_cast<size_t>(kHalves * n + hh) * nkb + kb) * 8192, kABytes,
                                  &full[s], pol_w);
                    if (!waited) {  // weights never depend on the previous kernel; activations do
                        asm volatile("griddepcontrol.wait;" ::: "memory");
                        waited = true;
                    }
                    tma_load_2d(st + kWBytes, &map_x, &full[s], kb * kBlockK, m * kWideM, pol_x);
                    ++n_issued;
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            const uint32_t idesc = idesc_bf16_f32(kWideM, NW);
            int s = 0;
            uint32_t ph = 0;
            int j = 0;
            for (int u = c; u < units; u += P, ++j) {
                const int b = j & 1;
                if (j >= 2) mbar_wait(&tempty[b], static_cast<uint32_t>(((j >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t acc = tmem + static_cast<uint32_t>(b * NW);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sw = smem_u32(smem + s * kStageBytes);
                    const uint64_t bdesc = sw128_kmajor_desc(sw);
                    const uint64_t adesc = sw128_kmajor_desc(sw + kWBytes);
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k)
                        umma_bf16(acc, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != 0 || k != 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                umma_commit(&tfull[b]);
            }
        }
    } else {
        // ---------------- epilogue warps 2..5: thread = token row ----------------
        const int q = warp & 3;
        const int row = q * 32 + lane;  // TMEM lane
        const GemmEpiParams& e = a.epi;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        int j = 0;
        for (int u = c; u < units; u += P, ++j) {
            const int n = u / m_tiles, m = u % m_tiles;
            const int tok = m * kWideM + row;
            const bool valid = tok < a.w;
            float rn = 1.0f;
            if (e.ss_in != nullptr && valid) {
                const float* ssr = e.ss_in + static_cast<size_t>(tok) * e.ss_tiles;
                float acc = 0.0f;
                for (int i0 = 0; i0 < e.ss_tiles; i0 += 16) {
                    float v16[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) v16[jj] = i0 + jj < e.ss_tiles ? __ldcg(ssr + i0 + jj) : 0.0f;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        if (i0 + jj < e.ss_tiles) acc = __fadd_rn(acc, v16[jj]);
                }
                rn = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(acc, static_cast<float>(e.norm_d)), e.eps));
            }
            int page = 0, slot = 0, pos = 0;
            if (e.kind == kEpiQkvRope && valid) {
                pos = e.ps->n_cached + tok;
                page = e.page_table[pos / e.page_size];
                slot = pos % e.page_size;
            }
            const int b = j & 1;
            mbar_wait(&tfull[b], static_cast<uint32_t>((j >> 1) & 1));
            __syncwarp();
            tc_fence_after();
            const uint32_t t_lane = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * NW);
            wide_tile_epilogue<NW>(a, t_lane, nullptr, 1, 0, n, tok, valid, rn, page, slot, pos);
            tc_fence_before();
            mbar_arrive(&tempty[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<2 * NW>(tmem);
#endif
}

cudaError_t launch_gemm_prefill(const __nv_bfloat16* w_tiled, const CUtensorMap* map_x128, int n_out, int k,
                                int w, const GemmEpiParams& epi, cudaStream_t stream) {
    static bool attr_set[kMaxDevices] = {};  // per device: TP ranks of one process
    const int dev = current_device_slot();
    constexpr int kStages = 4;
    // 256-row weight tiles (a 128x256x16 MMA per 12 KiB of shared-memory operands
    // instead of 128x128x16 per 8 KiB) unless 128-row tiles fill the persistent
    // grid's waves much better (measured: 128-row tiles cost ~35% per flop)
    const int m_tiles = (w + kWideM - 1) / kWideM;
    auto wave_eff = [&](int nw) {
        const int u = m_tiles * (n_out / nw);
        return static_cast<double>(u) / (((u + kNumSMs - 1) / kNumSMs) * kNumSMs);
    };
    const bool nw256 = n_out % 256 == 0 && wave_eff(256) >= wave_eff(128) - 0.2;
    const uint32_t stage = nw256 ? WideCfg<256>::kStageBytes : WideCfg<128>::kStageBytes;
    const int smem = static_cast<int>(kStages * stage + 1024 + 64 * 8);
    if (!attr_set[dev]) {
        cudaFuncSetAttribute(gemm_prefill_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(gemm_prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr_set[dev] = true;
    }
    GemmArgs a{};
    a.n_out = n_out;
    a.k = k;
    a.w = w;
    a.nt = kWideM;
    a.nkb = k / kBlockK;
    a.tiles = n_out / (nw256 ? 256 : 128);
    a.stages = kStages;
    a.epi = epi;
    const int units = ((w + kWideM - 1) / kWideM) * a.tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::min(units, kNumSMs), 1, 1);
    cfg.blockDim = dim3(kWideThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (nw256) return cudaLaunchKernelEx(&cfg, gemm_prefill_kernel<256>, w_tiled, *map_x128, a);
    return cudaLaunchKernelEx(&cfg, gemm_prefill_kernel<128>, w_tiled, *map_x128, a);
}

}  // namespace dd

namespace dd {
void preload_gemm_wide_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, gemm_wide_kernel<128>);
    cudaFuncGetAttributes(&a, gemm_wide_kernel<256>);
    cudaFuncGetAttributes(&a, gemm_prefill_kernel<128>);
    cudaFuncGetAttributes(&a, gemm_prefill_kernel<256>);
}
}  // namespace dd
