// Device pieces shared by the standalone skinny GEMM (gemm.cu) and the
// persistent pass kernel (pass.cu): stream-K partition, fused epilogues
// (RoPE + paged-KV append, residual + deferred-RMSNorm producer, SwiGLU,
// logits store) and the deferred-RMSNorm consumer scaling.
#pragma once

#include "common.cuh"
#include "gemm.h"

namespace dd {
namespace gemm_dev {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;  // 16 KiB
constexpr int kThreads = 192;                         // 6 warps
constexpr int kEpiThreads = 128;                      // warps 2..5
constexpr int kChunk = 16;                            // tokens per staging chunk
constexpr int kMaxSeg = 16;                           // stream-K segments per tile (host-checked)


// (c * T fits 32 bits for every shape here: T <= 2^17 blocks, P <= 512; the
// 32-bit division keeps the single-thread issue loops cheap)
__host__ __device__ inline long sk_begin(int c, long T, int P) {
    return static_cast<long>(static_cast<uint32_t>(c) * static_cast<uint32_t>(T) / static_cast<uint32_t>(P));
}
// CTA whose range contains global k-block g
__host__ __device__ inline int sk_owner(long g, long T, int P) {
    int c = static_cast<int>(static_cast<uint32_t>(g) * static_cast<uint32_t>(P) / static_cast<uint32_t>(T));
    while (c + 1 < P && sk_begin(c + 1, T, P) <= g) ++c;
    while (c > 0 && sk_begin(c, T, P) > g) --c;
    return c;
}

// Stream-K segments of `tile`: the CTAs with a non-empty range covering its
// k-blocks (when T < P some CTAs own no block at all and take no part).
// nseg = their number, seg = the position of CTA c among them.
__host__ __device__ inline void sk_segments(int tile, int nkb, long T, int P, int c, int* nseg,
                                            int* seg) {
    const int first = sk_owner(static_cast<long>(tile) * nkb, T, P);
    const int last = sk_owner(static_cast<long>(tile + 1) * nkb - 1, T, P);
    if (T >= P) {  // every CTA owns at least one block
        *nseg = last - first + 1;
        *seg = c - first;
        return;
    }
    int n = 0, pos = 0;
    for (int k = first; k <= last; ++k) {
        if (sk_begin(k + 1, T, P) > sk_begin(k, T, P)) {
            if (k == c) pos = n;
            ++n;
        }
    }
    *nseg = n;
    *seg = pos;
}

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Apply the fused epilogue to tokens [t0, t0+tn) of tile `tile` whose reduced
// fp32 values are staged in red[t][128].
static __device__ void apply_epilogue(const GemmArgs& a, int tile, int t0, int tn, const float* red,
                               int tid, float* part /* [4][kChunk] scratch */) {
    const GemmEpiParams& e = a.epi;
    const int m0 = tile * kBlockM;
    if (e.kind == kEpiStore || e.kind == kEpiResidual) {
        // batch every load before any store (red is a generic pointer into
        // shared memory, so interleaving would serialise on aliasing)
        float v[kChunk], x[kChunk];
        float* dst = e.out + static_cast<size_t>(t0) * a.n_out + m0 + tid;
#pragma unroll
        for (int t = 0; t < kChunk; ++t) v[t] = t < tn ? red[t * 128 + tid] : 0.0f;
        if (e.kind == kEpiResidual) {
#pragma unroll
            for (int t = 0; t < kChunk; ++t)
                x[t] = t < tn ? __ldcg(dst + static_cast<size_t>(t) * a.n_out) : 0.0f;  // L2: written by other CTAs
#pragma unroll
            for (int t = 0; t < kChunk; ++t) v[t] = __fadd_rn(x[t], v[t]);
        }
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < tn) dst[static_cast<size_t>(t) * a.n_out] = v[t];
        if (e.kind == kEpiResidual && e.u_out != nullptr) {
            // deferred RMSNorm producer: u = bf16(x * g) and per-token sum of
            // squares of this tile's 128 rows (fixed shuffle / smem tree)
            const float g = e.gain[m0 + tid];
            __nv_bfloat16* u = e.u_out + static_cast<size_t>(t0) * a.n_out + m0 + tid;
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                if (t < tn) u[static_cast<size_t>(t) * a.n_out] = __float2bfloat16_rn(__fmul_rn(v[t], g));
                float sq = __fmul_rn(v[t], v[t]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
                if ((tid & 31) == 0) part[(tid >> 5) * kChunk + t] = sq;
            }
            epi_bar();
            if (tid < tn) {
                const float tot = __fadd_rn(__fadd_rn(part[tid], part[kChunk + tid]),
                                            __fadd_rn(part[2 * kChunk + tid], part[3 * kChunk + tid]));
                e.ss_out[static_cast<size_t>(t0 + tid) * a.tiles + tile] = tot;
            }
        }
    } else if (e.kind == kEpiSwiGLU) {
        const int ffn = a.n_out / 2;
        for (int idx = tid; idx < tn * 64; idx += kEpiThreads) {
            const int t = idx >> 6, f = idx & 63;
            const float g = red[t * 128 + f], u = red[t * 128 + 64 + f];
            const float silu = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
            e.out_bf[static_cast<size_t>(t0 + t) * ffn + tile * 64 + f] =
                __float2bfloat16_rn(__fmul_rn(silu, u));
        }
    } else {  // kEpiQkvRope
        const ModelDims& md = e.m;
        const int hd = md.head_dim, half = hd / 2;
        const int q_dim = md.q_dim(), kv_dim = md.kv_dim();
        const int n_cached = e.ps->n_cached;
        if (m0 < q_dim + kv_dim) {
            for (int idx = tid; idx < tn * 64; idx += kEpiThreads) {
                const int t = idx >> 6, pr = idx & 63;
                const int hl = pr / half, i = pr % half;
                const int r0 = hl * hd + i;
                const float av = red[t * 128 + r0], bv = red[t * 128 + r0 + half];
                const int pos = n_cached + t0 + t;
                const float c = e.rope_cos[static_cast<size_t>(pos) * half + i];
                const float sn = e.rope_sin[static_cast<size_t>(pos) * half + i];
                const float lo = __fmaf_rn(av, c, -__fmul_rn(bv, sn));
                const float hi = __fmaf_rn(bv, c, __fmul_rn(av, sn));
                const int grow = m0 + r0;
                if (grow < q_dim) {
                    float* qd = e.q_out + static_cast<size_t>(t0 + t) * q_dim + grow;
                    qd[0] = lo;
                    qd[half] = hi;
                } else {
                    const int kh = (grow - q_dim) / hd;
                    const int page = e.page_table[pos / e.page_size], slot = pos % e.page_size;
                    __nv_bfloat16* kd =
                        e.kv_pool + kv_offset(md, e.page_size, page, e.layer, 0, kh, slot) + i;
                    kd[0] = __float2bfloat16_rn(lo);
                    kd[half] = __float2bfloat16_rn(hi);
                }
            }
        } else {
            for (int idx = tid; idx < tn * 128; idx += kEpiThreads) {
                const int t = idx >> 7, r = idx & 127;
                const int pos = n_cached + t0 + t;
                const int ve = m0 + r - q_dim - kv_dim;
                const int page = e.page_table[pos / e.page_size], slot = pos % e.page_size;
                e.kv_pool[kv_offset(md, e.page_size, page, e.layer, 1, ve / hd, slot) + ve % hd] =
                    __float2bfloat16_rn(red[t * 128 + r]);
            }
        }
    }
}

// Deferred-RMSNorm consumer side: scale the staged accumulator rows of
// tokens [t0, t0+tn) by r[t] = 1/sqrt(sum_tiles(ss_in[t][:]) / d + eps).
static __device__ void scale_by_rnorm(const GemmArgs& a, int t0, int tn, float* red, int tid,
                               float* s_r) {
    const GemmEpiParams& e = a.epi;
    if (e.ss_in == nullptr) return;
    if (tid < tn) {
        const float* ss = e.ss_in + static_cast<size_t>(t0 + tid) * e.ss_tiles;
        float acc = 0.0f;
        for (int i0 = 0; i0 < e.ss_tiles; i0 += 16) {  // 16 loads in flight, summed in order
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = i0 + j < e.ss_tiles ? __ldcg(ss + i0 + j) : 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (i0 + j < e.ss_tiles) acc = __fadd_rn(acc, v[j]);
        }
        s_r[tid] = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(acc, static_cast<float>(e.norm_d)), e.eps));
    }
    epi_bar();
    for (int t = 0; t < tn; ++t) red[t * 128 + tid] = __fmul_rn(red[t * 128 + tid], s_r[t]);
    epi_bar();
}



// Wide-pass epilogue of tokens [t0, t0 + tn) of one 128-row tile with one output
// row per thread (row == epilogue thread id == TMEM lane): v[j] = D[row][t0 + j],
// already reduced over stream-K segments and scaled by the RMSNorm factor when
// the GEMM consumes h.  Store / residual write straight from registers; SwiGLU
// and RoPE pair rows of different warps and stage through `red` once.  Pass-level
// per-token constants (KV page and slot of position n_cached + t) come from
// shared memory.  Same arithmetic as apply_epilogue.
static __device__ void chunk_epilogue_rows(const GemmArgs& a, int tile, int t0, int tn, const float* v,
                                           const float* xv, float gcol, const int* s_page,
                                           const int* s_slot, float* red, float* part, int row, int tid) {
    const GemmEpiParams& e = a.epi;
    const int m0 = tile * kBlockM;
    if (e.kind == kEpiStore) {
        float* dst = e.out + static_cast<size_t>(t0) * a.n_out + m0 + row;
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < tn) dst[static_cast<size_t>(t) * a.n_out] = v[t];
    } else if (e.kind == kEpiResidual) {
        float y[kChunk];
        float* dst = e.out + static_cast<size_t>(t0) * a.n_out + m0 + row;
#pragma unroll
        for (int t = 0; t < kChunk; ++t) y[t] = t < tn ? __fadd_rn(xv[t], v[t]) : 0.0f;
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < tn) dst[static_cast<size_t>(t) * a.n_out] = y[t];
        if (e.u_out != nullptr) {
            __nv_bfloat16* u = e.u_out + static_cast<size_t>(t0) * a.n_out + m0 + row;
            __nv_bfloat16* ulo = e.lo_out ? e.lo_out + static_cast<size_t>(t0) * a.n_out + m0 + row : nullptr;
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                if (t < tn) {
                    const float uv = __fmul_rn(y[t], gcol);
                    const __nv_bfloat16 hi = __float2bfloat16_rn(uv);
                    u[static_cast<size_t>(t) * a.n_out] = hi;
                    if (ulo) ulo[static_cast<size_t>(t) * a.n_out] = __float2bfloat16_rn(__fsub_rn(uv, __bfloat162float(hi)));
                }
                float sq = __fmul_rn(y[t], y[t]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
                if ((row & 31) == 0) part[(row >> 5) * kChunk + t] = sq;
            }
            epi_bar();
            if (tid < tn) {
                const float tot = __fadd_rn(__fadd_rn(part[tid], part[kChunk + tid]),
                                            __fadd_rn(part[2 * kChunk + tid], part[3 * kChunk + tid]));
                e.ss_out[static_cast<size_t>(t0 + tid) * a.tiles + tile] = tot;
            }
        }
    } else {
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < tn) red[t * 128 + row] = v[t];
        epi_bar();
        if (e.kind == kEpiSwiGLU) {
            const int ffn = a.n_out / 2;
            for (int idx = tid; idx < tn * 64; idx += kEpiThreads) {
                const int t = idx >> 6, f = idx & 63;
                const float g = red[t * 128 + f], uu = red[t * 128 + 64 + f];
                const float silu = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
                const float av = __fmul_rn(silu, uu);
                const size_t ai = static_cast<size_t>(t0 + t) * ffn + tile * 64 + f;
                const __nv_bfloat16 hi = __float2bfloat16_rn(av);
                e.out_bf[ai] = hi;
                if (e.lo_out) e.lo_out[ai] = __float2bfloat16_rn(__fsub_rn(av, __bfloat162float(hi)));
            }
        } else {  // kEpiQkvRope
            const ModelDims& md = e.m;
            const int hd = md.head_dim, half = hd / 2;
            const int q_dim = md.q_dim(), kv_dim = md.kv_dim();
            const int n_cached = e.ps->n_cached;
            if (m0 < q_dim + kv_dim) {
                // the thread's (token, pair) items: cos / sin requested before use
                constexpr int kItems = kChunk * 64 / kEpiThreads;  // 8
                float cv[kItems], sv[kItems];
#pragma unroll
                for (int k = 0; k < kItems; ++k) {
                    const int idx = tid + k * kEpiThreads;
                    const int t = idx >> 6, pr = idx & 63, i = pr % half;
                    const size_t ro = static_cast<size_t>(n_cached + t0 + t) * half + i;
                    cv[k] = t < tn ? e.rope_cos[ro] : 0.0f;
                    sv[k] = t < tn ? e.rope_sin[ro] : 0.0f;
                }
#pragma unroll
                for (int k = 0; k < kItems; ++k) {
                    const int idx = tid + k * kEpiThreads;
                    const int t = idx >> 6, pr = idx & 63;
                    if (t >= tn) continue;
                    const int hl = pr / half, i = pr % half;
                    const int r0 = hl * hd + i;
                    const float av = red[t * 128 + r0], bv = red[t * 128 + r0 + half];
                    const float lo = __fmaf_rn(av, cv[k], -__fmul_rn(bv, sv[k]));
                    const float hi = __fmaf_rn(bv, cv[k], __fmul_rn(av, sv[k]));
                    const int grow = m0 + r0;
                    if (grow < q_dim) {
                        float* qd = e.q_out + static_cast<size_t>(t0 + t) * q_dim + grow;
                        qd[0] = lo;
                        qd[half] = hi;
                    } else {
                        const int kh = (grow - q_dim) / hd;
                        const size_t ko = kv_offset(md, e.page_size, s_page[t0 + t], e.layer, 0, kh, s_slot[t0 + t]) + i;
                        if (e.kv_f32) {
                            e.kv_f32[ko] = lo;
                            e.kv_f32[ko + half] = hi;
                        } else {
                            e.kv_pool[ko] = __float2bfloat16_rn(lo);
                            e.kv_pool[ko + half] = __float2bfloat16_rn(hi);
                        }
                    }
                }
            } else {
                for (int idx = tid; idx < tn * 128; idx += kEpiThreads) {
                    const int t = idx >> 7, r = idx & 127;
                    const int ve = m0 + r - q_dim - kv_dim;
                    const size_t vo =
                        kv_offset(md, e.page_size, s_page[t0 + t], e.layer, 1, ve / hd, s_slot[t0 + t]) + ve % hd;
                    if (e.kv_f32) e.kv_f32[vo] = red[t * 128 + r];
                    else e.kv_pool[vo] = __float2bfloat16_rn(red[t * 128 + r]);
                }
            }
        }
    }
}
}  // namespace gemm_dev
}  // namespace dd
