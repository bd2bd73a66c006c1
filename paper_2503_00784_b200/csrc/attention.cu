// Split-KV causal attention over the paged bf16 KV cache, on tensor cores
// (mma.sync m16n8k16 bf16 -> fp32), for every pass width (decode W <= 32 and
// prefill chunks up to 256 tokens).
//
// Grid = (kRanks, query tiles of 16 new tokens, query heads); the kRanks CTAs
// of one (head, tile) form a thread-block cluster.  Keys are cut into splits
// of 128 at absolute positions; rank r takes splits r, r + kRanks, ... .  Per
// split the CTA stages K and V (128 keys) in shared memory with cp.async
// (16-byte chunks, XOR-swizzled so the fragment reads are conflict-free),
// then every warp computes the full S = QK^T of the split (16 rows x 128
// keys) and the online softmax (fp32, exp2 domain) - identical in the four
// warps - and warp w accumulates O for its quarter of the head dims.  No
// merge across warps is needed.  Fragments use two permutations:
//  * QK^T: the head dims are permuted inside each 32-dim chunk so that lane
//    quad c reads K[key][32ch + 8c .. +8] as one 16-byte chunk (the Q
//    fragments use the same permutation, so the dot products are unchanged);
//  * PV: lane group g supplies column g of the warp's n-tiles, mapped to the
//    NTW contiguous dims w*HD/4 + g*NTW + e, so one 8-byte (4-byte) read per
//    key feeds every n-tile; pairs are packed with byte permutes.
// Ranks merge through distributed shared memory (rank order).  Work placement
// depends only on absolute key positions and query rows are independent, so a
// token's output does not depend on the pass width (tests/test_gpu_kernels).
#include "common.cuh"
#include "model.h"

namespace dd {

namespace {

constexpr int kSplitKeys = 128;
constexpr int kRanks = 8;  // CTAs per cluster (portable maximum)
constexpr int kAttnCtaThreads = 128;
constexpr int kQTile = 16;

__device__ __forceinline__ void pdl_wait_() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte global -> shared copy; src_bytes = 0 zero-fills without reading
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// K row `key`, 16-byte chunk `ch` (8 dims) -> swizzled chunk
__device__ __forceinline__ int k_chunk(int key, int ch) { return ch ^ (key & 7); }
// V: move key pairs across the 128-byte bank window
template <int HD>
__device__ __forceinline__ int v_chunk(int key, int ch) {
    return ch ^ (((key >> 1) & 3) << (HD == 128 ? 2 : 1));
}

template <int HD>
struct AttnSmem {
    __nv_bfloat16 k[kSplitKeys][HD];
    __nv_bfloat16 v[kSplitKeys][HD];
    float res_o[kQTile][HD];  // this CTA's unnormalised O, read by the cluster
    float res_m[kQTile];
    float res_l[kQTile];
};

}  // namespace

#ifdef DD_ATTN_TRACE  // timing harness only (scripts/micro/attn_bench.cu)
__device__ unsigned long long* g_attn_trace = nullptr;
#define ATT_STAMP(k)                                                                       \
    do {                                                                                   \
        if (g_attn_trace && threadIdx.x == 0) {                                            \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
            const int b_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);  \
            if (b_ < 4096) g_attn_trace[b_ * 16 + (k)] = t_;                               \
        }                                                                                  \
    } while (0)
void attention_set_trace(unsigned long long* p) { cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p)); }
#else
#define ATT_STAMP(k) \
    do {             \
    } while (0)
#endif

// RANKS = CTAs per (head, query tile): kRanks (a cluster, split-KV + DSMEM
// merge) for long contexts, 1 (every split in sequence, no merge) when the
// context fits in two splits.
template <int HD, int RANKS>
__global__ void __launch_bounds__(kAttnCtaThreads)
    attn_cluster_kernel(const PassState* ps, ModelDims md, const float* __restrict__ q,
                        const __nv_bfloat16* __restrict__ kv_pool,
                        const int32_t* __restrict__ page_table, int page_size, int layer,
                        float scale_log2, __nv_bfloat16* __restrict__ o) {
    constexpr int NCH = HD / 32;      // 32-dim chunks of QK^T (2 k-steps each)
    constexpr int CHK = HD / 8;       // 16-byte chunks per K/V row
    constexpr int DW = HD / 4;        // output dims per warp
    constexpr int NTW = DW / 8;       // output n-tiles per warp (4 or 2)
    constexpr int NJ = kSplitKeys / 8;  // S n-tiles per split (16)
    extern __shared__ __align__(128) uint8_t attn_smem_raw[];
    AttnSmem<HD>& sm = *reinterpret_cast<AttnSmem<HD>*>(attn_smem_raw);
    ATT_STAMP(0);
    pdl_wait_();
    pdl_launch_();
    const int rank = RANKS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
    const int qt = blockIdx.y, head = blockIdx.z;
    const int n0 = ps->n_cached, W = ps->w;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, c = lane & 3;
    const int kvh = head / (md.n_heads / md.n_kv_heads);
    const int qd = md.q_dim();
    const int tid = threadIdx.x;

    const bool tile_live = qt * kQTile < W;
    const int t_hi = min(W, (qt + 1) * kQTile);  // exclusive
    const int kmax = n0 + t_hi - 1;               // last key any row of the tile may see
    const int n_split = tile_live ? kmax / kSplitKeys + 1 : 0;
    const int pos_g = n0 + qt * kQTile + g, pos_g8 = pos_g + 8;  // this lane's two rows
    const bool v_g = qt * kQTile + g < W, v_g8 = qt * kQTile + g + 8 < W;

    float acc[NTW][4];
#pragma unroll
    for (int t = 0; t < NTW; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
    float m_g = -INFINITY, m_g8 = -INFINITY, l_g = 0.f, l_g8 = 0.f;

    ATT_STAMP(1);
    if (rank < n_split) {
        // Q fragments (bf16, permuted dims), rows g and g + 8
        uint32_t qa[NCH][4], qb[NCH][4];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int d0 = head * HD + ch * 32 + c * 8;
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
            if (v_g) {
                const float4* src = reinterpret_cast<const float4*>(
                    q + static_cast<size_t>(qt * kQTile + g) * qd + d0);
                a0 = src[0];
                a1 = src[1];
            }
            if (v_g8) {
                const float4* src = reinterpret_cast<const float4*>(
                    q + static_cast<size_t>(qt * kQTile + g + 8) * qd + d0);
                b0 = src[0];
                b1 = src[1];
            }
            qa[ch][0] = pack_bf16(a0.x, a0.y);
            qa[ch][1] = pack_bf16(a0.z, a0.w);
            qa[ch][2] = pack_bf16(a1.x, a1.y);
            qa[ch][3] = pack_bf16(a1.z, a1.w);
            qb[ch][0] = pack_bf16(b0.x, b0.y);
            qb[ch][1] = pack_bf16(b0.z, b0.w);
            qb[ch][2] = pack_bf16(b1.x, b1.y);
            qb[ch][3] = pack_bf16(b1.z, b1.w);
        }
#pragma unroll 1
        for (int split = rank; split < n_split; split += RANKS) {
            const int kb = split * kSplitKeys;
            // ---- stage the split's K and V (zero-filled past kmax)
#pragma unroll 4
            for (int idx = tid; idx < kSplitKeys * CHK; idx += kAttnCtaThreads) {
                const int kk = idx / CHK, ch = idx % CHK;
                const int key = kb + kk;
                const bool ok = key <= kmax;
                const int kc = ok ? key : 0;
                const size_t base =
                    kv_offset(md, page_size, page_table[kc / page_size], layer, 0, kvh, kc % page_size);
                const __nv_bfloat16* ksrc = kv_pool + base + ch * 8;
                const __nv_bfloat16* vsrc = kv_pool +
                    kv_offset(md, page_size, page_table[kc / page_size], layer, 1, kvh, kc % page_size) + ch * 8;
                cp_async16(&sm.k[kk][k_chunk(kk, ch) * 8], ksrc, ok ? 16u : 0u);
                cp_async16(&sm.v[kk][v_chunk<HD>(kk, ch) * 8], vsrc, ok ? 16u : 0u);
            }
            cp_async_wait_all();
            __syncthreads();
            ATT_STAMP(2);
            // ---- S = Q K^T for the 128 keys (16 n-tiles of 8)
            float s[NJ][4];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
                const int kk = 8 * j + g;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const uint4 kr = *reinterpret_cast<const uint4*>(&sm.k[kk][k_chunk(kk, 4 * ch + c) * 8]);
                    const uint32_t a0[4] = {qa[ch][0], qb[ch][0], qa[ch][1], qb[ch][1]};
                    mma_bf16(s[j], a0, kr.x, kr.y);
                    const uint32_t a1[4] = {qa[ch][2], qb[ch][2], qa[ch][3], qb[ch][3]};
                    mma_bf16(s[j], a1, kr.z, kr.w);
                }
            }
            // ---- online softmax (log2 domain), causal mask per row
            float mx_g = -INFINITY, mx_g8 = -INFINITY;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int key = kb + 8 * j + 2 * c + e;
                    s[j][e] = key <= pos_g ? s[j][e] * scale_log2 : -INFINITY;
                    s[j][2 + e] = key <= pos_g8 ? s[j][2 + e] * scale_log2 : -INFINITY;
                    mx_g = fmaxf(mx_g, s[j][e]);
                    mx_g8 = fmaxf(mx_g8, s[j][2 + e]);
                }
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                mx_g = fmaxf(mx_g, __shfl_xor_sync(0xffffffffu, mx_g, off));
                mx_g8 = fmaxf(mx_g8, __shfl_xor_sync(0xffffffffu, mx_g8, off));
            }
            const float mn_g = fmaxf(m_g, mx_g), mn_g8 = fmaxf(m_g8, mx_g8);
            const float base_g = mn_g == -INFINITY ? 0.f : mn_g;
            const float base_g8 = mn_g8 == -INFINITY ? 0.f : mn_g8;
            const float cr_g = fast_exp2(m_g - base_g), cr_g8 = fast_exp2(m_g8 - base_g8);
            m_g = mn_g;
            m_g8 = mn_g8;
            l_g *= cr_g;
            l_g8 *= cr_g8;
#pragma unroll
            for (int t = 0; t < NTW; ++t) {
                acc[t][0] *= cr_g;
                acc[t][1] *= cr_g;
                acc[t][2] *= cr_g8;
                acc[t][3] *= cr_g8;
            }
            uint32_t pa[NJ / 2][4];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const float p0 = fast_exp2(s[j][0] - base_g), p1 = fast_exp2(s[j][1] - base_g);
                const float p2 = fast_exp2(s[j][2] - base_g8), p3 = fast_exp2(s[j][3] - base_g8);
                l_g += p0 + p1;
                l_g8 += p2 + p3;
                pa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p0, p1);
                pa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p2, p3);
            }
            // ---- O[:, warp's dims] += P V
            const int dbyte = (warp * DW + g * NTW) * 2;  // within the row
#pragma unroll
            for (int ks = 0; ks < NJ / 2; ++ks) {
                uint32_t vw[4][NTW / 2];  // keys 2c, 2c+1, 2c+8, 2c+9: NTW dims each
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int kk = 16 * ks + 2 * c + (r & 1) + (r >> 1) * 8;
                    const int ch = v_chunk<HD>(kk, dbyte >> 4);
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(&sm.v[kk][0]) + ch * 16 + (dbyte & 15);
                    if (NTW == 4) {
                        const uint2 x = *reinterpret_cast<const uint2*>(src);
                        vw[r][0] = x.x;
                        vw[r][NTW / 2 - 1] = x.y;
                    } else {
                        vw[r][0] = *reinterpret_cast<const uint32_t*>(src);
                    }
                }
#pragma unroll
                for (int e = 0; e < NTW; ++e) {
                    const uint32_t sel = (e & 1) ? 0x7632 : 0x5410;
                    const uint32_t b0 = __byte_perm(vw[0][e >> 1], vw[1][e >> 1], sel);
                    const uint32_t b1 = __byte_perm(vw[2][e >> 1], vw[3][e >> 1], sel);
                    mma_bf16(acc[e], pa[ks], b0, b1);
                }
            }
            __syncthreads();  // the next split overwrites K / V
        }
    }
    ATT_STAMP(3);
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
        l_g += __shfl_xor_sync(0xffffffffu, l_g, off);
        l_g8 += __shfl_xor_sync(0xffffffffu, l_g8, off);
    }
    // C fragment column 2c (2c+1) of n-tile e -> dim warp*DW + (2c)*NTW + e
    const int dcol = warp * DW + 2 * c * NTW;
    if (RANKS == 1 || n_split <= 1) {  // uniform over the cluster: rank 0 alone finishes
        if (rank == 0 && n_split >= 1) {
            const float ig = 1.0f / l_g, ig8 = 1.0f / l_g8;
            const size_t og = static_cast<size_t>(qt * kQTile + g) * qd + head * HD;
            const size_t og8 = og + static_cast<size_t>(8) * qd;
#pragma unroll
            for (int e = 0; e < NTW; ++e) {
                if (v_g) {
                    o[og + dcol + e] = __float2bfloat16_rn(acc[e][0] * ig);
                    o[og + dcol + NTW + e] = __float2bfloat16_rn(acc[e][1] * ig);
                }
                if (v_g8) {
                    o[og8 + dcol + e] = __float2bfloat16_rn(acc[e][2] * ig8);
                    o[og8 + dcol + NTW + e] = __float2bfloat16_rn(acc[e][3] * ig8);
                }
            }
        }
        return;
    }
    if constexpr (RANKS > 1) {
    // ---- cluster merge (rank order) through DSMEM; rank r finishes rows r, r + 8
#pragma unroll
    for (int e = 0; e < NTW; ++e) {
        sm.res_o[g][dcol + e] = acc[e][0];
        sm.res_o[g][dcol + NTW + e] = acc[e][1];
        sm.res_o[g + 8][dcol + e] = acc[e][2];
        sm.res_o[g + 8][dcol + NTW + e] = acc[e][3];
    }
    if (warp == 0 && c == 0) {
        sm.res_m[g] = m_g;
        sm.res_m[g + 8] = m_g8;
        sm.res_l[g] = l_g;
        sm.res_l[g + 8] = l_g8;
    }
    ATT_STAMP(4);
    cluster_sync();
    ATT_STAMP(5);
    {
        constexpr int kRowsPerRank = kQTile / kRanks;  // 2
        constexpr int kThreadsPerRow = kAttnCtaThreads / kRowsPerRank;
        const int r = rank + kRanks * (tid / kThreadsPerRow);
        const int t = qt * kQTile + r;
        if (t < W) {
            const uint32_t a_m = smem_u32(&sm.res_m[r]), a_l = smem_u32(&sm.res_l[r]);
            float mj[kRanks], lj[kRanks];
            const int nr = min(n_split, kRanks);
#pragma unroll
            for (int j = 0; j < kRanks; ++j) {
                mj[j] = j < nr ? ld_dsmem_f32(dsmem_addr(a_m, j)) : -INFINITY;
                lj[j] = j < nr ? ld_dsmem_f32(dsmem_addr(a_l, j)) : 0.f;
            }
            float M = -INFINITY;
#pragma unroll
            for (int j = 0; j < kRanks; ++j) M = fmaxf(M, mj[j]);
            float L = 0.f, f[kRanks];
#pragma unroll
            for (int j = 0; j < kRanks; ++j) {
                f[j] = mj[j] == -INFINITY ? 0.f : fast_exp2(mj[j] - M);
                L += lj[j] * f[j];
            }
            const float inv = 1.0f / L;
            for (int d = tid % kThreadsPerRow; d < HD; d += kThreadsPerRow) {
                const uint32_t a_o = smem_u32(&sm.res_o[r][d]);
                float v[kRanks];
#pragma unroll
                for (int j = 0; j < kRanks; ++j) v[j] = j < nr ? ld_dsmem_f32(dsmem_addr(a_o, j)) : 0.f;
                float O = 0.f;
#pragma unroll
                for (int j = 0; j < kRanks; ++j) O += v[j] * f[j];
                o[static_cast<size_t>(t) * qd + head * HD + d] = __float2bfloat16_rn(O * inv);
            }
        }
    }
    ATT_STAMP(6);
    cluster_sync();  // keep this CTA's shared memory alive until every rank has read it
    ATT_STAMP(7);
    }
}

// Prefill attention (long prompts, enqueue_prefill_big): CTA = (head, 64-query
// tile), warp w owns queries [16 w, 16 w + 16) of the tile and computes its own
// S = Q K^T (16 x 64 keys per chunk), online softmax and O += P V over all head
// dims, so the K / V chunks staged in shared memory (cp.async, double-buffered,
// the same swizzles as above) are shared by 64 queries and no warp repeats
// another's work.  Causal: a chunk past a warp's last query is skipped, the
// CTA stops at its last query's key.  Heavier (later) query tiles of every head
// launch before any lighter one.
template <int HD>
__global__ void __launch_bounds__(kAttnCtaThreads, 3)
    attn_prefill_kernel(const PassState* ps, ModelDims md, const float* __restrict__ q,
                        const __nv_bfloat16* __restrict__ kv_pool, const int32_t* __restrict__ page_table,
                        int page_size, int layer, float scale_log2, __nv_bfloat16* __restrict__ o) {
    constexpr int kKeys = 64;      // keys per staged chunk
    constexpr int NCH = HD / 32;   // 32-dim chunks of QK^T (2 k-steps each)
    constexpr int CHK = HD / 8;    // 16-byte chunks per K/V row
    constexpr int NT = HD / 8;     // PV n-tiles: thread g owns dims [g NT, g NT + NT)
    constexpr int NW = NT / 2;     // 32-bit words of those dims per key row
    extern __shared__ __align__(128) uint8_t attn_smem_raw[];
    auto ks = [&](int b) { return reinterpret_cast<__nv_bfloat16(*)[HD]>(attn_smem_raw + b * 2 * kKeys * HD * 2); };
    auto vs = [&](int b) {
        return reinterpret_cast<__nv_bfloat16(*)[HD]>(attn_smem_raw + (b * 2 + 1) * kKeys * HD * 2);
    };
    pdl_wait_();
    pdl_launch_();
    const int n0 = ps->n_cached, W = ps->w;
    const int qtiles = (W + 63) / 64;
    // heads fastest, heaviest query tiles first: the launch order is globally
    // longest-first, so the last wave holds only the short early tiles
    const int qt = qtiles - 1 - static_cast<int>(blockIdx.y), head = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, c = lane & 3;
    const int kvh = head / (md.n_heads / md.n_kv_heads);
    const int qd = md.q_dim();
    const int kmax = n0 + min(W, 64 * (qt + 1)) - 1;  // last key of this CTA
    const int n_chunks = kmax / kKeys + 1;
    const int row_g = 64 * qt + 16 * warp + g, row_g8 = row_g + 8;  // query rows of this thread
    const int pos_g = n0 + row_g, pos_g8 = n0 + row_g8;
    const int warp_last = n0 + min(W - 1, 64 * qt + 16 * warp + 15);  // last key any row of the warp sees

    auto stage = [&](int chunk, int b) {
        __nv_bfloat16(*kd)[HD] = ks(b);
        __nv_bfloat16(*vd)[HD] = vs(b);
        const int kb = chunk * kKeys;
        // one page-table read and one row address per key (2 threads per key,
        // half of its 16-byte chunks each); V row = K row + one kv plane
        constexpr int kTpk = kAttnCtaThreads / kKeys;
        const int kk = tid / kTpk, ch0 = (tid % kTpk) * (CHK / kTpk);
        const int key = kb + kk;
        const bool ok = key <= kmax;
        const int kc = ok ? key : 0;
        const __nv_bfloat16* krow =
            kv_pool + kv_offset(md, page_size, page_table[kc / page_size], layer, 0, kvh, kc % page_size);
        const __nv_bfloat16* vrow = krow + static_cast<size_t>(md.n_kv_heads) * page_size * HD;
        const uint32_t nb = ok ? 16u : 0u;
#pragma unroll
        for (int i = 0; i < CHK / kTpk; ++i) {
            const int ch = ch0 + i;
            cp_async16(&kd[kk][k_chunk(kk, ch) * 8], krow + ch * 8, nb);
            cp_async16(&vd[kk][v_chunk<HD>(kk, ch) * 8], vrow + ch * 8, nb);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage(0, 0);

    uint32_t qa[NCH][4], qb[NCH][4];
    {
        const bool v_g = row_g < W, v_g8 = row_g8 < W;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int d0 = head * HD + ch * 32 + c * 8;
            float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
            if (v_g) {
                const float4* src = reinterpret_cast<const float4*>(q + static_cast<size_t>(row_g) * qd + d0);
                a0 = __ldg(src);
                a1 = __ldg(src + 1);
            }
            if (v_g8) {
                const float4* src = reinterpret_cast<const float4*>(q + static_cast<size_t>(row_g8) * qd + d0);
                b0 = __ldg(src);
                b1 = __ldg(src + 1);
            }
            qa[ch][0] = pack_bf16(a0.x, a0.y);
            qa[ch][1] = pack_bf16(a0.z, a0.w);
            qa[ch][2] = pack_bf16(a1.x, a1.y);
            qa[ch][3] = pack_bf16(a1.z, a1.w);
            qb[ch][0] = pack_bf16(b0.x, b0.y);
            qb[ch][1] = pack_bf16(b0.z, b0.w);
            qb[ch][2] = pack_bf16(b1.x, b1.y);
            qb[ch][3] = pack_bf16(b1.z, b1.w);
        }
    }
    float acc[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
    float m_g = -INFINITY, m_g8 = -INFINITY, l_g = 0.f, l_g8 = 0.f;

    for (int chunk = 0; chunk < n_chunks; ++chunk) {
        const int b = chunk & 1;
        if (chunk + 1 < n_chunks) {
            stage(chunk + 1, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const int kb = chunk * kKeys;
        if (kb <= warp_last) {
            __nv_bfloat16(*kd)[HD] = ks(b);
            __nv_bfloat16(*vd)[HD] = vs(b);
            float sc[kKeys / 8][4];
#pragma unroll
            for (int j = 0; j < kKeys / 8; ++j) {
                sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
                const int kk = 8 * j + g;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const uint4 kr = *reinterpret_cast<const uint4*>(&kd[kk][k_chunk(kk, 4 * ch + c) * 8]);
                    const uint32_t a0[4] = {qa[ch][0], qb[ch][0], qa[ch][1], qb[ch][1]};
                    mma_bf16(sc[j], a0, kr.x, kr.y);
                    const uint32_t a1[4] = {qa[ch][2], qb[ch][2], qa[ch][3], qb[ch][3]};
                    mma_bf16(sc[j], a1, kr.z, kr.w);
                }
            }
            float mx_g = -INFINITY, mx_g8 = -INFINITY;
#pragma unroll
            for (int j = 0; j < kKeys / 8; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int key = kb + 8 * j + 2 * c + e;
                    sc[j][e] = key <= pos_g ? sc[j][e] * scale_log2 : -INFINITY;
                    sc[j][2 + e] = key <= pos_g8 ? sc[j][2 + e] * scale_log2 : -INFINITY;
                    mx_g = fmaxf(mx_g, sc[j][e]);
                    mx_g8 = fmaxf(mx_g8, sc[j][2 + e]);
                }
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                mx_g = fmaxf(mx_g, __shfl_xor_sync(0xffffffffu, mx_g, off));
                mx_g8 = fmaxf(mx_g8, __shfl_xor_sync(0xffffffffu, mx_g8, off));
            }
            const float mn_g = fmaxf(m_g, mx_g), mn_g8 = fmaxf(m_g8, mx_g8);
            const float base_g = mn_g == -INFINITY ? 0.f : mn_g;
            const float base_g8 = mn_g8 == -INFINITY ? 0.f : mn_g8;
            const float cr_g = fast_exp2(m_g - base_g), cr_g8 = fast_exp2(m_g8 - base_g8);
            m_g = mn_g;
            m_g8 = mn_g8;
            l_g *= cr_g;
            l_g8 *= cr_g8;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                acc[t][0] *= cr_g;
                acc[t][1] *= cr_g;
                acc[t][2] *= cr_g8;
                acc[t][3] *= cr_g8;
            }
#pragma unroll
            for (int kst = 0; kst < kKeys / 16; ++kst) {
                uint32_t pa[4];
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const float* sj = sc[2 * kst + jj];
                    const float p0 = fast_exp2(sj[0] - base_g), p1 = fast_exp2(sj[1] - base_g);
                    const float p2 = fast_exp2(sj[2] - base_g8), p3 = fast_exp2(sj[3] - base_g8);
                    l_g += p0 + p1;
                    l_g8 += p2 + p3;
                    pa[jj * 2 + 0] = pack_bf16(p0, p1);
                    pa[jj * 2 + 1] = pack_bf16(p2, p3);
                }
                uint32_t vw[4][NW];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int kk = 16 * kst + 2 * c + (r & 1) + (r >> 1) * 8;
                    if constexpr (HD == 128) {
                        const uint4 x0 = *reinterpret_cast<const uint4*>(&vd[kk][v_chunk<HD>(kk, 2 * g) * 8]);
                        const uint4 x1 = *reinterpret_cast<const uint4*>(&vd[kk][v_chunk<HD>(kk, 2 * g + 1) * 8]);
                        vw[r][0] = x0.x; vw[r][1] = x0.y; vw[r][2] = x0.z; vw[r][3] = x0.w;
                        vw[r][4] = x1.x; vw[r][5] = x1.y; vw[r][6] = x1.z; vw[r][7] = x1.w;
                    } else {
                        const uint4 x0 = *reinterpret_cast<const uint4*>(&vd[kk][v_chunk<HD>(kk, g) * 8]);
                        vw[r][0] = x0.x; vw[r][1] = x0.y; vw[r][2] = x0.z; vw[r][3] = x0.w;
                    }
                }
#pragma unroll
                for (int e = 0; e < NT; ++e) {
                    const uint32_t sel = (e & 1) ? 0x7632 : 0x5410;
                    const uint32_t b0 = __byte_perm(vw[0][e >> 1], vw[1][e >> 1], sel);
                    const uint32_t b1 = __byte_perm(vw[2][e >> 1], vw[3][e >> 1], sel);
                    mma_bf16(acc[e], pa, b0, b1);
                }
            }
        }
        __syncthreads();  // buffer b is refilled by the next iteration's stage
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
        l_g += __shfl_xor_sync(0xffffffffu, l_g, off);
        l_g8 += __shfl_xor_sync(0xffffffffu, l_g8, off);
    }
    // C fragment (row g / g + 8, col 2c + h) of tile e is dim (2c + h) * NT + e
    const float ig = 1.0f / l_g, ig8 = 1.0f / l_g8;
    if (row_g < W) {
        __nv_bfloat16* og = o + static_cast<size_t>(row_g) * qd + head * HD;
#pragma unroll
        for (int e = 0; e < NT; ++e) {
            og[(2 * c) * NT + e] = __float2bfloat16_rn(acc[e][0] * ig);
            og[(2 * c + 1) * NT + e] = __float2bfloat16_rn(acc[e][1] * ig);
        }
    }
    if (row_g8 < W) {
        __nv_bfloat16* og = o + static_cast<size_t>(row_g8) * qd + head * HD;
#pragma unroll
        for (int e = 0; e < NT; ++e) {
            og[(2 * c) * NT + e] = __float2bfloat16_rn(acc[e][2] * ig8);
            og[(2 * c + 1) * NT + e] = __float2bfloat16_rn(acc[e][3] * ig8);
        }
    }
}

// Prefill attention on tcgen05 (head_dim 128, long prompts): CTA = (head,
// 128-query tile), two threads per query row (TMEM lane), one per 64-key half
// of S and 64-dim half of O (8 warps: one warp per scheduler is latency-bound).
// Per 128-key block:
//   S = Q K^T   one elected thread, 8 MMAs 128x128x16 (A = Q, B = K, both
//               K-major SW128 in shared memory), S in TMEM columns [0, 128);
//   softmax     each thread reads its S row (tcgen05.ld), masks keys past its
//               position, updates the running base / sum (fp32, exp2 domain)
//               and writes P = bf16(exp2(s - base))
//               as the K-major SW128 A operand of the PV product;
//   O += P V    8 MMAs 128x128x16 with V read MN-major (the [key][dim] rows the
//               KV cache holds), O accumulated in TMEM columns [128, 256); a
//               row's O is rescaled in TMEM only when its exp2 base moves.
// K/V blocks are staged with cp.async (one page-table read per key and
// thread), double-buffered so block j+1 loads under block j.  Same roundings
// as the mma.sync kernel (q, P and K/V bf16, fp32 accumulate); different
// fp32 summation order.
namespace {
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
constexpr int kTcKeys = 128;
constexpr int kTcThreads = 256;  // 2 threads per query row (key / dim halves)
constexpr uint32_t kTcHalf = 128 * 128;  // one 64-dim (or 64-key) SW128 half: 128 rows x 128 B
__host__ __device__ constexpr uint32_t idesc_bf16_mn(int M, int N, int b_mn) {
    return idesc_bf16_f32(M, N) | (static_cast<uint32_t>(b_mn) << 16);
}
__device__ __forceinline__ uint64_t sw128_desc_lbo(uint32_t addr, uint32_t lbo) {
    return (sw128_kmajor_desc(addr) & ~(static_cast<uint64_t>(0x3FFF) << 16)) |
           (static_cast<uint64_t>(lbo >> 4) << 16);
}
// byte offset of 16-byte chunk `ch` (0..15, 8 bf16 each) of row `r` in a
// [2 halves][128 rows][128 B] SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int r, int ch) {
    return static_cast<uint32_t>((ch >> 3) * kTcHalf + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}
}  // namespace

__global__ void __launch_bounds__(kTcThreads, 1)
    attn_prefill_tc_kernel(const PassState* ps, ModelDims md, const float* __restrict__ q,
                           const __grid_constant__ CUtensorMap map_kv, const int32_t* __restrict__ page_table,
                           int page_size, int layer, float scale_log2, __nv_bfloat16* __restrict__ o) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    constexpr int HD = 128;
    extern __shared__ __align__(128) uint8_t attn_smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the __shared__ array (an
    // integer round trip would turn the exchange accesses into generic LD/ST)
    uint8_t* sm = attn_smem_raw + ((1024u - (smem_u32(attn_smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = sm;                       // 32 KiB
    uint8_t* sKV = sQ + 2 * kTcHalf;        // [2 buffers][K 32 KiB | V 32 KiB]
    uint8_t* sP = sKV + 8 * kTcHalf;        // 32 KiB
    float* xch = reinterpret_cast<float*>(sP + 2 * kTcHalf);  // [2 halves][128 rows] max / sum exchange
    uint64_t* bar = reinterpret_cast<uint64_t*>(xch + 2 * 128);  // [0] S done, [1] PV done, [2 + b] K/V buffer b full
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // thread = (query row r, key / dim half h): warps 0-3 take columns [0, 64)
    // of S and O, warps 4-7 columns [64, 128) of the same TMEM lanes
    const int h = warp >> 2, r = (warp & 3) * 32 + lane;
    if (warp == 0) tmem_alloc<256>(tslot);
    // V rows past the last key are read by the PV product with P = 0, so the
    // buffers must never hold non-finite bytes: zero them before any TMA
    for (int i = tid; i < 2 * 4 * static_cast<int>(kTcHalf) / 16; i += kTcThreads) {
        const int buf = i / (4 * kTcHalf / 16), off = i % (4 * kTcHalf / 16);
        reinterpret_cast<uint4*>(sm + 2 * kTcHalf + buf * 4 * kTcHalf)[off] = make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        tma_prefetch_desc(&map_kv);
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_barrier_init();
    }
    pdl_wait_();
    pdl_launch_();
    const int n0 = ps->n_cached, W = ps->w;
    const int qt = static_cast<int>(gridDim.y) - 1 - static_cast<int>(blockIdx.y), head = blockIdx.x;
    const int kvh = head / (md.n_heads / md.n_kv_heads);
    const int qd = md.q_dim();
    const int row = 128 * qt + r;  // this thread's query row in the pass
    const int pos = n0 + row;
    const int kmax = n0 + min(W, 128 * (qt + 1)) - 1;  // last key of the CTA
    const int n_blk = kmax / kTcKeys + 1;

    // staging (warp 0, lane = (page, K / V, 64-dim half)): per page of the
    // block holding a key <= kmax one TMA box of page_size rows lands as SW128
    // rows of the K-major (K) or MN-major (V) operand tile; pages past kmax
    // keep the buffer's earlier (finite) rows, masked to P = 0.  Page-table
    // entries are read one block ahead, so issuing never waits on them.
    const uint64_t pol = policy_evict_normal();
    const int st_pg = lane >> 2, st_kv = (lane >> 1) & 1, st_h = lane & 1;
    auto page_of = [&](int blk) {
        const int key = min(blk * kTcKeys + st_pg * page_size, kmax);
        return __ldg(page_table + key / page_size);
    };
    auto stage = [&](int blk, int b, int page) {
        const int kb0 = blk * kTcKeys;
        const int n_pg = min(kTcKeys, kmax - kb0 + page_size) / page_size;  // pages with a live key
        if (lane == 0) mbar_arrive_expect_tx(&bar[2 + b], static_cast<uint32_t>(n_pg * page_size * 128 * 4));
        __syncwarp();
        if (st_pg < n_pg) {
            const int row = static_cast<int>(kv_offset(md, page_size, page, layer, st_kv, kvh, 0) / HD);
            tma_load_2d(sKV + b * 4 * kTcHalf + (2 * st_kv + st_h) * kTcHalf + st_pg * page_size * 128, &map_kv,
                        &bar[2 + b], 64 * st_h, row, pol);
        }
    };
    __syncthreads();  // barriers initialised, buffers zeroed
    int page_next = 0;
    if (warp == 0) {
        stage(0, 0, page_of(0));
        if (n_blk > 1) page_next = page_of(1);
    }
    {  // Q row (fp32 -> bf16) half, zero past the pass
        const float* src = q + static_cast<size_t>(row) * qd + head * HD;
#pragma unroll 4
        for (int i = 0; i < 8; ++i) {
            const int ch = 8 * h + i;
            uint4 u = make_uint4(0u, 0u, 0u, 0u);
            if (row < W) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(src + ch * 8));
                const float4 b = __ldg(reinterpret_cast<const float4*>(src + ch * 8 + 4));
                u = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w));
            }
            *reinterpret_cast<uint4*>(sQ + sw128_off(r, ch)) = u;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + 64 * h, tO = tmem + 128 + lane_off + 64 * h;
    constexpr uint32_t kIdS = idesc_bf16_mn(128, 128, 0), kIdO = idesc_bf16_mn(128, 128, 1);

    // O accumulates in TMEM across blocks.  The exp2 base of a row moves only
    // when its block max exceeds the base by more than 8 (P <= 2^8 in bf16 is
    // exact in range), and then the row's O and sum are rescaled in place.
    float m_base = -INFINITY, l_run = 0.f;

    for (int blk = 0; blk < n_blk; ++blk) {
        const int b = blk & 1;
        mbar_wait(&bar[2 + b], static_cast<uint32_t>((blk >> 1) & 1));  // K/V of blk landed
        tc_fence_before();
        __syncthreads();  // (and every thread is past block blk - 1)
        tc_fence_after();
        const uint8_t* sk = sKV + b * 4 * kTcHalf;
        const uint8_t* sv = sk + 2 * kTcHalf;
        if (tid == 0) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const uint32_t off = (ks >> 2) * kTcHalf;
                umma_bf16(tmem, sw128_kmajor_desc(smem_u32(sQ + off)) + 2 * (ks & 3),
                          sw128_kmajor_desc(smem_u32(sk + off)) + 2 * (ks & 3), kIdS, ks ? 1u : 0u);
            }
            umma_commit(&bar[0]);
        }
        if (warp == 0 && blk + 1 < n_blk) {  // next block's K/V under this block's MMAs and softmax
            stage(blk + 1, b ^ 1, page_next);
            if (blk + 2 < n_blk) page_next = page_of(blk + 2);
        }
        __syncwarp();
        mbar_wait(&bar[0], static_cast<uint32_t>(blk & 1));
        tc_fence_after();
        const int kb = blk * kTcKeys + 64 * h;  // first key of this thread's half
        // pass 1: max of the masked, scaled scores over the half, then the row's
        float mx = -INFINITY;
        uint32_t srow[4][16];  // this thread's 64 scores, kept for pass 2
        {
            uint32_t (&rr)[4][16] = srow;
#pragma unroll
            for (int i = 0; i < 4; ++i) tmem_ld16_async(tS + 16 * i, rr[i]);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (kb + 16 * i + j <= pos) mx = fmaxf(mx, __uint_as_float(rr[i][j]) * scale_log2);
        }
        xch[h * 128 + r] = mx;
        // only warps w and w + 4 share rows: a 64-thread named barrier per pair
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp & 3)) : "memory");
        mx = fmaxf(xch[r], xch[128 + r]);
        const bool move = mx > m_base + 8.0f;  // false while both are -inf
        float corr = 1.0f;
        if (move) {
            corr = fast_exp2(m_base - mx);  // 0 on the first live block
            m_base = mx;
            l_run *= corr;
        }
        if (blk > 0 && __any_sync(0xffffffffu, move)) {  // warp-collective rescale of this half of O
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t rr[2][16];
                tmem_ld16_async(tO + c0, rr[0]);
                tmem_ld16_async(tO + c0 + 16, rr[1]);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 16; ++j) rr[i][j] = __float_as_uint(__uint_as_float(rr[i][j]) * corr);
                tmem_st16(tO + c0, rr[0]);
                tmem_st16(tO + c0 + 16, rr[1]);
            }
            tmem_wait_st();
        }
        const float base = m_base == -INFINITY ? 0.f : m_base;
        // pass 2: P = exp2(s - base) as bf16 into the SW128 A tile, half sums in fp32
        {
            const uint32_t (&rr)[4][16] = srow;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t pk[8];
#pragma unroll
                for (int j = 0; j < 16; j += 2) {
                    const int key = kb + 16 * i + j;
                    const float p0 = key <= pos ? fast_exp2(__uint_as_float(rr[i][j]) * scale_log2 - base) : 0.f;
                    const float p1 =
                        key + 1 <= pos ? fast_exp2(__uint_as_float(rr[i][j + 1]) * scale_log2 - base) : 0.f;
                    l_run += p0 + p1;
                    pk[j >> 1] = pack_bf16(p0, p1);
                }
                const int ch = 8 * h + 2 * i;  // 16-byte chunk of the key row
                *reinterpret_cast<uint4*>(sP + sw128_off(r, ch)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                *reinterpret_cast<uint4*>(sP + sw128_off(r, ch + 1)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();  // P and the O rescale complete, S reads done
        tc_fence_after();
        if (tid == 0) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)  // 16 keys per step
                umma_bf16(tmem + 128, sw128_kmajor_desc(smem_u32(sP + (ks >> 2) * kTcHalf)) + 2 * (ks & 3),
                          sw128_desc_lbo(smem_u32(sv + ks * 16 * 128), kTcHalf), kIdO,
                          (blk > 0 || ks > 0) ? 1u : 0u);
            umma_commit(&bar[1]);
        }
        __syncwarp();
        mbar_wait(&bar[1], static_cast<uint32_t>(blk & 1));
        tc_fence_after();
    }
    xch[h * 128 + r] = l_run;  // the last exchange read happened before two barriers
    __syncthreads();
    {
        const float il = 1.0f / (xch[r] + xch[128 + r]);
        __nv_bfloat16* og = o + static_cast<size_t>(row) * qd + head * HD + 64 * h;
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 32) {
            uint32_t rr[2][16];
            tmem_ld16_async(tO + c0, rr[0]);
            tmem_ld16_async(tO + c0 + 16, rr[1]);
            tmem_wait_ld();
            if (row < W)
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 16; j += 8) {
                        const float* f = reinterpret_cast<const float*>(&rr[i][j]);
                        *reinterpret_cast<uint4*>(og + c0 + 16 * i + j) =
                            make_uint4(pack_bf16(f[0] * il, f[1] * il), pack_bf16(f[2] * il, f[3] * il),
                                       pack_bf16(f[4] * il, f[5] * il), pack_bf16(f[6] * il, f[7] * il));
                    }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tmem);
#endif
}

int launch_attention_prefill(const PassState* ps, int w, const ModelDims& m, const float* q,
                             const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                             int layer, __nv_bfloat16* o, cudaStream_t s, const CUtensorMap* map_kv) {
    const float scale_log2 =
        static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(m.head_dim)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(m.n_heads, (w + 63) / 64, 1);
    cfg.blockDim = dim3(kAttnCtaThreads, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int dev = current_device_slot();
    static bool a128[kMaxDevices] = {}, a64[kMaxDevices] = {};
    auto go = [&](auto kernel, int hd, bool* attr) {
        const size_t smem = static_cast<size_t>(4) * 64 * hd * 2;
        cfg.dynamicSmemBytes = smem;
        if (!attr[dev]) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            attr[dev] = true;
        }
        return cudaLaunchKernelEx(&cfg, kernel, ps, m, q, kv_pool, page_table, page_size, layer, scale_log2, o);
    };
    cudaError_t e;
    static const bool tc = !(getenv("DD_ATTN_PREFILL_TC") && atoi(getenv("DD_ATTN_PREFILL_TC")) == 0);
    static bool atc[kMaxDevices] = {};
    if (m.head_dim == 128 && tc && map_kv != nullptr && m.n_heads % m.n_kv_heads == 0) {
        cfg.gridDim = dim3(m.n_heads, (w + 127) / 128, 1);
        const int smem = static_cast<int>(12 * kTcHalf + 1024 + 2 * 128 * 4 + 64 + 32);
        cfg.blockDim = dim3(kTcThreads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        if (!atc[dev]) {
            cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            atc[dev] = true;
        }
        e = cudaLaunchKernelEx(&cfg, attn_prefill_tc_kernel, ps, m, q, *map_kv, page_table, page_size, layer,
                               scale_log2, o);
    } else if (m.head_dim == 128) e = go(attn_prefill_kernel<128>, 128, a128);
    else if (m.head_dim == 64) e = go(attn_prefill_kernel<64>, 64, a64);
    else return -1;
    return e == cudaSuccess ? 0 : -2;
}

int launch_attention(const PassState* ps, int w, const ModelDims& m, const float* q,
                     const __nv_bfloat16* kv_pool, const int32_t* page_table, int page_size,
                     int layer, __nv_bfloat16* o, cudaStream_t s, int ranks) {
    const int qtiles = (w + kQTile - 1) / kQTile;
    const float scale_log2 =
        static_cast<float>(1.4426950408889634 / sqrt(static_cast<double>(m.head_dim)));
    const bool cluster = ranks > 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster ? kRanks : 1, qtiles, m.n_heads);
    cfg.blockDim = dim3(kAttnCtaThreads, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kRanks;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cluster ? 1 : 0;
    const int dev = current_device_slot();
    auto go = [&](auto kernel, size_t smem, bool* attr) {  // attr: per device (TP ranks of one process)
        cfg.dynamicSmemBytes = smem;
        if (!attr[dev]) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            attr[dev] = true;
        }
        return cudaLaunchKernelEx(&cfg, kernel, ps, m, q, kv_pool, page_table, page_size, layer,
                                  scale_log2, o);
    };
    cudaError_t e;
    static bool a128c[kMaxDevices] = {}, a128s[kMaxDevices] = {}, a64c[kMaxDevices] = {},
                a64s[kMaxDevices] = {};
    if (m.head_dim == 128) {
        e = cluster ? go(attn_cluster_kernel<128, kRanks>, sizeof(AttnSmem<128>), a128c)
                    : go(attn_cluster_kernel<128, 1>, sizeof(AttnSmem<128>), a128s);
    } else if (m.head_dim == 64) {
        e = cluster ? go(attn_cluster_kernel<64, kRanks>, sizeof(AttnSmem<64>), a64c)
                    : go(attn_cluster_kernel<64, 1>, sizeof(AttnSmem<64>), a64s);
    } else {
        return -1;
    }
    return e == cudaSuccess ? 0 : -2;
}

}  // namespace dd

namespace dd {
void preload_attention_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, attn_cluster_kernel<128, kRanks>);
    cudaFuncGetAttributes(&a, attn_cluster_kernel<128, 1>);
    cudaFuncGetAttributes(&a, attn_cluster_kernel<64, kRanks>);
    cudaFuncGetAttributes(&a, attn_cluster_kernel<64, 1>);
    cudaFuncGetAttributes(&a, attn_prefill_kernel<128>);
    cudaFuncGetAttributes(&a, attn_prefill_kernel<64>);
    cudaFuncGetAttributes(&a, attn_prefill_tc_kernel);
}
}  // namespace dd
