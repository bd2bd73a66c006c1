// Persistent whole-pass kernel for the target verification pass (sm_100a).
//
// One cooperative launch of 148 CTAs (one per SM) runs the whole scored pass:
// embedding, then per layer QKV GEMM -> attention -> O GEMM -> gate/up GEMM ->
// down GEMM, then the LM head.  Kernel boundaries are replaced by tile-level
// dataflow flags in global memory (value = the pass epoch): an output tile's
// epilogue publishes its flag with release semantics, and the activation
// producer of the next phase acquires the flag of exactly the tile that feeds
// the k-block it is about to load.  Weights never depend on activations, so
// the weight producer streams the next phase's weights into the shared-memory
// ring while the previous phase drains - the HBM stream does not stop at
// phase boundaries.
//
// Warp roles (256 threads):
//   warp 0  weight producer: one 16 KiB cp.async.bulk per k-block (pre-tiled,
//           pre-swizzled weights, evict-first)
//   warp 1  MMA issuer: tcgen05.mma (M=128 weight rows, N=nt tokens, K=16)
//           into one of two TMEM accumulators
//   warp 2  activation producer: waits the producing tile's flag, then TMA
//           (128B swizzle) of the k-block's activation tile
//   warp 3  idle
//   warps 4-7 epilogue (tcgen05.ld; stream-K segment reduction; fused RoPE +
//           paged-KV append / residual + deferred-RMSNorm / SwiGLU / logits),
//           the embedding phase and the attention phase.
// The stream-K partition of each GEMM (gemm_epi.cuh) depends only on its shape,
// attention work placement only on absolute key positions, and every
// reduction has a fixed order: a token's logits are identical whatever the
// pass width.  Deadlock freedom needs all CTAs co-resident: the launch is
// cooperative with one CTA per SM.
#include "common.cuh"
#include "gemm_epi.cuh"
#include "pass.h"

#include <cstdlib>
#include <cstring>

namespace dd {

using namespace gemm_dev;

// debug seam: per-CTA progress words in mapped host memory (dd_debug_pass_progress)
__device__ volatile int* g_pass_dbg = nullptr;
#define PASS_DBG(slot, val)                                                      \
    do {                                                                         \
        if (g_pass_dbg) g_pass_dbg[blockIdx.x * 8 + (slot)] = (val);             \
    } while (0)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void pass_put(const PassParams& P, int p, int k, unsigned long long v) {
    if (P.trace) P.trace[(static_cast<size_t>(blockIdx.x) * P.n_phases + p) * 12 + k] = v;
}
__device__ __forceinline__ void pass_stamp(const PassParams& P, int p, int k) {
    if (P.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[(static_cast<size_t>(blockIdx.x) * P.n_phases + p) * 12 + k] = t;
    }
}

namespace {

constexpr int kEpiBase = 128;  // first epilogue thread (warp 4)
#ifndef DD_ACC_BUFS
#define DD_ACC_BUFS 4
#endif
#ifndef DD_PUB_OFFLOAD
#define DD_PUB_OFFLOAD 1
#endif
#ifndef DD_ATTN_AHEAD
#define DD_ATTN_AHEAD 0  // attention chunks staged ahead (0: every buffer before the loop, each refilled after use; else that many, one buffer kept free)
#endif
#ifndef DD_PASS_STAGE_CAP
#define DD_PASS_STAGE_CAP 9
#endif
#ifndef DD_ATTN_ONEBAR
#define DD_ATTN_ONEBAR 1  // attention chunk loop: one CTA barrier per chunk (refill after the next chunk's barrier)
#endif
#ifndef DD_SUM_BATCH
#define DD_SUM_BATCH 6  // measured: 4 / 5 / 6 / 7 / 8 -> W=9 2.969 / 2.980 / 2.940 / 2.980 / 2.994 ms
#endif
constexpr int kSumBatch = DD_SUM_BATCH;  // stream-K partials loaded per round by a reducer thread
#ifndef DD_SS_UNROLL
#define DD_SS_UNROLL 1  // residual epilogue: the tile's sum of squares with its 16 shared loads in flight
#endif
#ifndef DD_ACQ_POLL
#define DD_ACQ_POLL 1  // activation producer: per-flag acquire loads instead of a full fence after the polls (W=9 3.12 -> 3.02 ms); 0: fence
#endif
constexpr int kAccBufs = DD_ACC_BUFS;  // TMEM accumulators: the MMA runs up to kAccBufs tile segments ahead of the epilogue
// Publish ring: the epilogue hands every gpu-scope release (stream-K partial
// counters, tile flags) to warp 3, so its own threads never wait for the
// release's memory barrier before starting the next tile.
constexpr int kPubSlots = 8;
enum PubKind { kPubExit = 0, kPubCount = 1, kPubFlag = 2 };
struct PubAction {
    int kind, base, idx, phase;
    int* ptr;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// replica `rep` of flag (base + idx)
__device__ __forceinline__ int* flag_at(int* flags, int base, int idx, int rep) {
    return flags + (static_cast<size_t>(base + idx) * kFlagReplicas + rep) * kFlagStride;
}
// the replica this CTA polls
__device__ __forceinline__ int* flag_poll(int* flags, int base, int idx) {
    return flag_at(flags, base, idx, blockIdx.x % kFlagReplicas);
}
__device__ __forceinline__ void st_release_flag(int* flags, int base, int idx, int v);
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// One release fence, then relaxed stores to every replica: each replica's
// store is ordered after the data by the fence (a release store to replica 0
// alone would leave the pollers of replicas 1..7 formally unsynchronised).
__device__ __forceinline__ void st_release_flag(int* flags, int base, int idx, int v) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#pragma unroll
    for (int r = 0; r < kFlagReplicas; ++r)
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(flag_at(flags, base, idx, r)), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const int* p, int epoch) {
    while (ld_acquire(p) - epoch < 0) __nanosleep(32);
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Tensor parallelism inside the pass (tp.h): the reducer of row-parallel tile
// `tile` (O or down, residual phase k of the pass) publishes its reduced fp32
// values v[16] (thread = row, 16 tokens) in slot k % 4 of its exchange buffer,
// signals every peer's flag line (system-scope release), waits for every
// peer's signal of the same tile and phase, and replaces v by the sum over
// ranks in rank order 0..N-1 (bit-identical on every rank, so the replicated
// residual stays identical).  Slot reuse: a rank rewrites slot k % 4 at phase
// k + 4 only after it saw every peer's phase k + 2 signal, which a peer sends
// after its phase k + 1, i.e. after finishing its phase-k reads.  A peer that
// never signals traps after 10 s.
__device__ void tp_exchange(const PassParams& P, int k, int tile, float* v, int tid, int epoch) {
    const TpPeers& T = P.tp;
    const unsigned val = static_cast<unsigned>(epoch) * static_cast<unsigned>(2 * P.m.n_layers) +
                         static_cast<unsigned>(k) + 1u;
    const size_t off = (static_cast<size_t>((k & (kTpPassSlots - 1)) * kTpPassTiles + tile) * 128 + tid) * 16;
    float4* mine = reinterpret_cast<float4*>(T.pxch[T.rank] + off);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) mine[q4] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
    epi_bar();  // every row's store happens-before the release below
    if (tid == 0) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (int r = 0; r < T.size; ++r)
            if (r != T.rank)
                asm volatile("st.relaxed.sys.global.b32 [%0], %1;" ::"l"(T.pflags[r] + (T.rank * kTpPassTiles + tile) * kTpFlagStride),
                             "r"(val) : "memory");
    }
    if (tid < T.size && tid != T.rank) {
        const int* f = T.pflags[T.rank] + (tid * kTpPassTiles + tile) * kTpFlagStride;
        const unsigned long long t0 = gtimer();
        for (;;) {
            int got;
            asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(got) : "l"(f) : "memory");
            if (static_cast<int>(static_cast<unsigned>(got) - val) >= 0) break;
            __nanosleep(64);
            if (gtimer() - t0 > 10000000000ull) __trap();
        }
    }
    epi_bar();  // every peer's tile happens-before the loads below
    float tot[16];
    for (int r = 0; r < T.size; ++r) {
        float x[16];
        if (r == T.rank) {
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = v[i];
        } else {
            const float* src = T.pxch[r] + off;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(x[i]) : "l"(src + i) : "memory");
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) tot[i] = r == 0 ? x[i] : __fadd_rn(tot[i], x[i]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = tot[i];
}

// ---------------------------------------------------------------- attention
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
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ int k_chunk(int key, int ch) { return ch ^ (key & 7); }
template <int HD>
__device__ __forceinline__ int v_chunk(int key, int ch) {
    return ch ^ (((key >> 1) & 3) << (HD == 128 ? 2 : 1));
}

// One attention item: (head, 16-query tile, chunk group) over 64-key chunks
// grp, grp + kAttnGroups, ... (absolute positions), run by the 128 epilogue
// threads.  K and V of a chunk are staged in shared memory (swizzled); every
// warp computes S = QK^T for the chunk (16 x 64) and the online softmax, and
// warp w accumulates O for its quarter of the head dims (mma.sync m16n8k16).
// Groups merge through global partials; the last-arriving group combines them
// in group order and publishes the (head, tile) flag.
// Chunk groups of a (head, query tile) item: an item of at most `single`
// chunks runs as one group (each extra group costs a partial round trip and
// the last arriver's combine); longer ones split into groups of `cpg` chunks,
// at most kAttnGroups.
__device__ __forceinline__ int attn_groups(int n_chunks, int cpg, int single) {
    if (n_chunks <= single) return 1;
    return min(kAttnGroups, max(1, (n_chunks + cpg - 1) / cpg));
}

template <int HD>
__device__ void attn_item(const PassParams& P, const PassPhase& ph, uint8_t* kv_smem, int* s_bcast,
                          int head, int qt, int grp, int epoch, int tid, int pidx) {
    constexpr int kAttnBufs = attn_bufs(HD);
    constexpr int NCH = HD / 32;
    constexpr int CHK = HD / 8;
    constexpr int DW = HD / 4;
    constexpr int NTW = DW / 8;
    constexpr int NJ = kAttnChunk / 8;
    const ModelDims& md = P.m;
    const int n0 = P.ps->n_cached, W = P.ps->w;
    const int t_hi = min(W, (qt + 1) * 16);
    const int kmax = n0 + t_hi - 1;
    const int n_chunks = kmax / kAttnChunk + 1;
    const int active = attn_groups(n_chunks, P.attn_cpg, P.attn_single);
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, c = lane & 3;
    const int kvh = head / (md.n_heads / md.n_kv_heads);
    const int qd = md.q_dim();
    // kAttnBufs K/V chunk buffers: up to kAttnBufs - 1 chunks are in flight
    // while one is computed
    constexpr int kBufBytes = 2 * kAttnChunk * HD * 2;
    auto ks_of = [&](int b) {
        return reinterpret_cast<__nv_bfloat16(*)[HD]>(kv_smem + b * kBufBytes);
    };
    auto vs_of = [&](int b) {
        return reinterpret_cast<__nv_bfloat16(*)[HD]>(kv_smem + b * kBufBytes + kAttnChunk * HD * 2);
    };
    // staging addresses: thread = one 16-byte column chunk `sch` of keys
    // skk0 + 128 / CHK * i; a key's K (V) row is the page base + the
    // (layer, k|v, kv head, slot) offset, the page base one 64-bit multiply per
    // key (page table read once per key, L1-resident)
    const int sch = tid % CHK, skk0 = tid / CHK;
    const size_t page_elems = kv_offset(md, P.page_size, 1, 0, 0, 0, 0);
    const uint32_t k_off = static_cast<uint32_t>(kv_offset(md, P.page_size, 0, ph.layer, 0, kvh, 0)) + sch * 8;
    const uint32_t v_off = static_cast<uint32_t>(kv_offset(md, P.page_size, 0, ph.layer, 1, kvh, 0)) + sch * 8;
    auto stage = [&](int chunk, int b) {
        __nv_bfloat16(*ks)[HD] = ks_of(b);
        __nv_bfloat16(*vs)[HD] = vs_of(b);
        const int kb = chunk * kAttnChunk;
#pragma unroll
        for (int i = 0; i < kAttnChunk * CHK / 128; ++i) {
            const int kk = skk0 + (128 / CHK) * i;
            const int key = kb + kk;
            const bool ok = key <= kmax;
            const int kc = ok ? key : 0;
            const __nv_bfloat16* pg = P.kv_pool + static_cast<size_t>(__ldg(P.page_table + kc / P.page_size)) * page_elems;
            const uint32_t so = static_cast<uint32_t>(kc % P.page_size) * HD;
            cp_async16(&ks[kk][k_chunk(kk, sch) * 8], pg + k_off + so, ok ? 16u : 0u);
            cp_async16(&vs[kk][v_chunk<HD>(kk, sch) * 8], pg + v_off + so, ok ? 16u : 0u);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // chunks of this group: grp, grp + active, ... (cnt of them)
    const int n_mine = (n_chunks - grp + active - 1) / active;
    int issued = 0;
    auto issue = [&]() {
        stage(grp + issued * active, issued % kAttnBufs);
        ++issued;
    };
    // Keys cached before this pass do not depend on the QKV phase: their
    // chunks are in flight before the flags are polled, so only the chunk(s)
    // holding this pass's keys wait for the QKV epilogue.
    if (tid == 0) pass_stamp(P, pidx, 0);  // debug: item entered
    // The cached keys' later chunks (beyond the cp.async window) are pulled
    // into L2 now, one bulk prefetch per contiguous page run of K and of V:
    // the chunk loop then stages them at L2 rather than HBM latency.
    {
        const int run = min(P.page_size, kAttnChunk);  // keys per contiguous run
        const int runs_per_chunk = kAttnChunk / run;
        const int n_runs = max(0, n_mine - (kAttnBufs - 1)) * runs_per_chunk;
        for (int r = tid; r < n_runs; r += 128) {
            const int chunk = grp + (kAttnBufs - 1 + r / runs_per_chunk) * active;
            const int key = chunk * kAttnChunk + (r % runs_per_chunk) * run;
            if (key + run > n0) continue;  // this pass's keys: written by the QKV epilogue
            const int page = P.page_table[key / P.page_size], slot = key % P.page_size;
            prefetch_l2(P.kv_pool + kv_offset(md, P.page_size, page, ph.layer, 0, kvh, slot), run * HD * 2);
            prefetch_l2(P.kv_pool + kv_offset(md, P.page_size, page, ph.layer, 1, kvh, slot), run * HD * 2);
        }
    }
    constexpr int kAhead = DD_ATTN_AHEAD > 0 ? DD_ATTN_AHEAD : kAttnBufs;  // chunks staged before the loop
    while (issued < min(n_mine, kAhead) && (grp + issued * active + 1) * kAttnChunk <= n0) issue();
    // inputs: this head's q rows and its kv head's k and v rows of the QKV GEMM
    if (tid < 3) {  // q, k and v tiles polled in parallel
        const int row = tid == 0 ? head * HD : tid == 1 ? qd + kvh * HD : qd + md.kv_dim() + kvh * HD;
        if (!(P.nodep & 4)) wait_flag(flag_poll(P.flags, ph.qkv_flag, row / 128), epoch);
    }
    epi_bar();
    if (tid == 0) pass_stamp(P, pidx, 1);  // debug: QKV flags seen
    while (issued < min(n_mine, kAhead)) issue();  // in flight while Q is loaded

    const int pos_g = n0 + qt * 16 + g, pos_g8 = pos_g + 8;
    const bool v_g = qt * 16 + g < W, v_g8 = qt * 16 + g + 8 < W;
    uint32_t qa[NCH][4], qb[NCH][4];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int d0 = head * HD + ch * 32 + c * 8;
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
        if (v_g) {
            const float4* src = reinterpret_cast<const float4*>(P.q + static_cast<size_t>(qt * 16 + g) * qd + d0);
            a0 = __ldcg(src);
            a1 = __ldcg(src + 1);
        }
        if (v_g8) {
            const float4* src = reinterpret_cast<const float4*>(P.q + static_cast<size_t>(qt * 16 + g + 8) * qd + d0);
            b0 = __ldcg(src);
            b1 = __ldcg(src + 1);
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
    float acc[NTW][4];
#pragma unroll
    for (int t = 0; t < NTW; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
    float m_g = -INFINITY, m_g8 = -INFINITY, l_g = 0.f, l_g8 = 0.f;

    for (int i = 0, chunk = grp; chunk < n_chunks; ++i, chunk += active) {
        const int kb = chunk * kAttnChunk;
        const int b = i % kAttnBufs;
        if (kAhead < kAttnBufs && issued < n_mine) issue();  // into the buffer chunk i - 1 released
        // chunk i landed: at most (issued - 1 - i) younger groups pending
        switch (issued - 1 - i) {
            case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
            case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
            case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
            default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        }
        epi_bar();
#if DD_ATTN_ONEBAR
        // every warp is past iteration i - 1: its buffer takes the next chunk
        // (one CTA barrier per chunk instead of two)
        if (kAhead == kAttnBufs && i > 0 && issued < n_mine) issue();
#endif
        if (tid == 0 && i == 0) pass_stamp(P, pidx, 2);  // debug: first chunk staged
        __nv_bfloat16(*ks)[HD] = ks_of(b);
        __nv_bfloat16(*vs)[HD] = vs_of(b);
        float s[NJ][4];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
            const int kk = 8 * j + g;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const uint4 kr = *reinterpret_cast<const uint4*>(&ks[kk][k_chunk(kk, 4 * ch + c) * 8]);
                const uint32_t a0[4] = {qa[ch][0], qb[ch][0], qa[ch][1], qb[ch][1]};
                mma_bf16(s[j], a0, kr.x, kr.y);
                const uint32_t a1[4] = {qa[ch][2], qb[ch][2], qa[ch][3], qb[ch][3]};
                mma_bf16(s[j], a1, kr.z, kr.w);
            }
        }
        float mx_g = -INFINITY, mx_g8 = -INFINITY;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int key = kb + 8 * j + 2 * c + e;
                s[j][e] = key <= pos_g ? s[j][e] * P.scale_log2 : -INFINITY;
                s[j][2 + e] = key <= pos_g8 ? s[j][2 + e] * P.scale_log2 : -INFINITY;
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
        const int dbyte = (warp * DW + g * NTW) * 2;
#pragma unroll
        for (int kst = 0; kst < NJ / 2; ++kst) {
            uint32_t vw[4][2];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int kk = 16 * kst + 2 * c + (r & 1) + (r >> 1) * 8;
                const int chn = v_chunk<HD>(kk, dbyte >> 4);
                const uint8_t* src = reinterpret_cast<const uint8_t*>(&vs[kk][0]) + chn * 16 + (dbyte & 15);
                if constexpr (NTW == 4) {
                    const uint2 xv = *reinterpret_cast<const uint2*>(src);
                    vw[r][0] = xv.x;
                    vw[r][1] = xv.y;
                } else {
                    vw[r][0] = *reinterpret_cast<const uint32_t*>(src);
                    vw[r][1] = 0;
                }
            }
#pragma unroll
            for (int e = 0; e < NTW; ++e) {
                const uint32_t sel = (e & 1) ? 0x7632 : 0x5410;
                const uint32_t b0 = __byte_perm(vw[0][e >> 1], vw[1][e >> 1], sel);
                const uint32_t b1 = __byte_perm(vw[2][e >> 1], vw[3][e >> 1], sel);
                mma_bf16(acc[e], pa[kst], b0, b1);
            }
        }
#if !DD_ATTN_ONEBAR
        epi_bar();  // buffer b is refilled by the stage issued in the next iteration
        if (kAhead == kAttnBufs && issued < n_mine) issue();  // into buffer b, just consumed
#endif
    }
#if DD_ATTN_ONEBAR
    epi_bar();  // every warp done with the staging buffers (the next item restages them)
#endif
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
        l_g += __shfl_xor_sync(0xffffffffu, l_g, off);
        l_g8 += __shfl_xor_sync(0xffffffffu, l_g8, off);
    }
    if (tid == 0) pass_stamp(P, pidx, 4);  // debug: chunks done
    const int dcol = warp * DW + 2 * c * NTW;  // C columns 2c / 2c+1 -> dims dcol + e / + NTW + e
    const int flag_idx = head * 16 + qt;
    if (active == 1) {
        const float ig = 1.0f / l_g, ig8 = 1.0f / l_g8;
        const size_t og = static_cast<size_t>(qt * 16 + g) * qd + head * HD;
        const size_t og8 = og + static_cast<size_t>(8) * qd;
#pragma unroll
        for (int e = 0; e < NTW; ++e) {
            if (v_g) {
                P.o[og + dcol + e] = __float2bfloat16_rn(acc[e][0] * ig);
                P.o[og + dcol + NTW + e] = __float2bfloat16_rn(acc[e][1] * ig);
            }
            if (v_g8) {
                P.o[og8 + dcol + e] = __float2bfloat16_rn(acc[e][2] * ig8);
                P.o[og8 + dcol + NTW + e] = __float2bfloat16_rn(acc[e][3] * ig8);
            }
        }
        epi_bar();  // every thread's o stores happen-before thread 0's release
        if (tid == 0) {
            pass_stamp(P, pidx, 5);  // debug: o stored
            st_release_flag(P.flags, ph.out_flag, flag_idx, epoch);
            pass_stamp(P, pidx, 6);  // debug: published
        }
        return;
    }
    // partials: [head][qt][grp] x (16 rows x (HD + 2)), unnormalised O, m, l
    constexpr int RS = HD + 2;
    float* part = P.attn_part + ((static_cast<size_t>(head) * 16 + qt) * kAttnGroups) * 16 * RS;
    float* mine = part + static_cast<size_t>(grp) * 16 * RS;
#pragma unroll
    for (int e = 0; e < NTW; ++e) {
        mine[g * RS + dcol + e] = acc[e][0];
        mine[g * RS + dcol + NTW + e] = acc[e][1];
        mine[(g + 8) * RS + dcol + e] = acc[e][2];
        mine[(g + 8) * RS + dcol + NTW + e] = acc[e][3];
    }
    if (warp == 0 && c == 0) {
        mine[g * RS + HD] = m_g;
        mine[g * RS + HD + 1] = l_g;
        mine[(g + 8) * RS + HD] = m_g8;
        mine[(g + 8) * RS + HD + 1] = l_g8;
    }
    epi_bar();
    int* cnt = P.attn_cnt + head * 16 + qt;
    // release this group's partials, acquire the other groups'
    if (tid == 0) *s_bcast = atom_add_acq_rel(cnt, 1) == active - 1;
    epi_bar();
    if (!*s_bcast) return;
    // last group: combine the active groups in group order; thread = one dim of
    // 16 / (128 / HD) rows
    constexpr int kRows = 16 * HD / 128;
    const int d = tid % HD, r0 = tid / HD, rstep = 128 / HD;
    float M[kRows], L[kRows], O[kRows];
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
        M[i] = -INFINITY;
        L[i] = 0.f;
        O[i] = 0.f;
    }
    for (int j = 0; j < active; ++j)
#pragma unroll
        for (int i = 0; i < kRows; ++i)
            M[i] = fmaxf(M[i], __ldcg(part + (static_cast<size_t>(j) * 16 + r0 + i * rstep) * RS + HD));
    for (int j = 0; j < active; ++j) {
        float mj[kRows], lj[kRows], oj[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const float* row = part + (static_cast<size_t>(j) * 16 + r0 + i * rstep) * RS;
            mj[i] = __ldcg(row + HD);
            lj[i] = __ldcg(row + HD + 1);
            oj[i] = __ldcg(row + d);
        }
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const float f = mj[i] == -INFINITY ? 0.f : fast_exp2(mj[i] - M[i]);
            L[i] += lj[i] * f;
            O[i] += oj[i] * f;
        }
    }
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
        const int t = qt * 16 + r0 + i * rstep;
        if (t < W) P.o[static_cast<size_t>(t) * qd + head * HD + d] = __float2bfloat16_rn(O[i] / L[i]);
    }
    epi_bar();
    if (tid == 0) {
        *cnt = 0;
        st_release_flag(P.flags, ph.out_flag, flag_idx, epoch);
    }
}

// Embedding of column tile `tile` (128 columns) for every token: x = E[tok],
// h = bf16(x * g), ss[t][tile] = sum of squares (warp tree, then warps 0..3 in
// the order ((0+1)+(2+3)) - the residual epilogue's formulation).
__device__ void embed_tile(const PassParams& P, int tile, int W, float* part /* [4][32] */, int tid) {
    const int d = P.m.d, tiles = d / 128;
    const int col = tile * 128 + tid;
    const int warp = tid >> 5;
    const float gcol = P.gain[col];
    for (int t0 = 0; t0 < W; t0 += 32) {
        const int tn = min(32, W - t0);
        for (int t = 0; t < tn; ++t) {
            const int tok = P.ps->tokens[t0 + t];
            const float v = __bfloat162float(P.emb[static_cast<size_t>(tok) * d + col]);
            P.x[static_cast<size_t>(t0 + t) * d + col] = v;
            P.h[static_cast<size_t>(t0 + t) * d + col] = __float2bfloat16_rn(__fmul_rn(v, gcol));
            float sq = __fmul_rn(v, v);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
            if ((tid & 31) == 0) part[warp * 32 + t] = sq;
        }
        epi_bar();
        if (tid < tn)
            P.ss[static_cast<size_t>(t0 + tid) * tiles + tile] =
                __fadd_rn(__fadd_rn(part[tid], part[32 + tid]), __fadd_rn(part[64 + tid], part[96 + tid]));
        epi_bar();
    }
}

// One sub-phase of a GEMM phase (PassPhase.kg x PassPhase.tg grid, k-group major).
struct SubPhase {
    int tiles, nkb, T;  // tile count, k-blocks per tile, blocks
    int tile0, kb0;     // first global tile / k-block
    int ki;             // k-group index
    bool last_k;        // the k-group that completes its tiles
};
__device__ __forceinline__ SubPhase sub_of(const PassPhase& ph, int sp) {
    SubPhase s;
    const int i = sp / ph.tg, j = sp - i * ph.tg;
    s.tiles = ph.a.tiles / ph.tg;
    s.nkb = ph.a.nkb / ph.kg;
    s.T = s.tiles * s.nkb;
    s.tile0 = j * s.tiles;
    s.kb0 = i * s.nkb;
    s.ki = i;
    s.last_k = i == ph.kg - 1;
    return s;
}

// Inputs of one sub-phase's k-range [g0, g1): the k-blocks it covers form one
// run (or two, when the range wraps into the next tile) inside the k-group;
// each lane spins on its own subset of the producer flags of those k-blocks
// (weak L2 loads), then acq_rel fences and a warp sync order every TMA read
// that follows (plus the generic -> async proxy fence for the TMA engine).
__device__ void wait_sub_inputs(const PassParams& P, int x_src, int x_flag, const SubPhase& s, int g0, int g1,
                                int epoch, int qtiles, int lane) {
    const int hd_shift = P.m.head_dim == 128 ? 7 : 6;
    auto key_of = [&](int kb) {
        return x_src == kXNormed ? kb >> 1 : x_src == kXSwiglu ? kb : (kb * 64) >> hd_shift;
    };
    const int n = min(g1 - g0, s.nkb);
    int lo[2], hi[2], runs = 1;
    if (n == s.nkb) {
        lo[0] = s.kb0;
        hi[0] = s.kb0 + s.nkb - 1;
    } else {
        const int a = s.kb0 + g0 % s.nkb, e = a + n - 1, top = s.kb0 + s.nkb - 1;
        lo[0] = a;
        hi[0] = min(e, top);
        if (e > top) {
            lo[1] = s.kb0;
            hi[1] = e - s.nkb;
            runs = 2;
        }
    }
    const int per_key = x_src == kXAttn ? qtiles : 1;
    for (int r = 0; r < runs; ++r) {
        const int k_lo = key_of(lo[r]), count = key_of(hi[r]) - k_lo + 1;
        for (int i = lane; i < count * per_key; i += 32) {
            const int key = k_lo + i / per_key;
            const int idx = x_src == kXAttn ? key * 16 + i % per_key : key;
            const int* f = flag_poll(P.flags, x_flag, idx);
#if DD_ACQ_POLL
            // poll weakly, then one acquire load of the observed flag (instead of a
            // full fence after the polls)
            while (!(P.nodep & 1) && ld_relaxed(f) - epoch < 0) __nanosleep(64);
            (void)ld_acquire(f);
#else
            while (!(P.nodep & 1) && ld_relaxed(f) - epoch < 0) __nanosleep(64);
#endif
        }
    }
#if !DD_ACQ_POLL
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
    __syncwarp();
    fence_proxy_async();  // generic-proxy writes -> the TMA (async proxy) reads that follow
}

// ---------------------------------------------------------------- fast epilogue
// Decode-width (W <= 16) epilogue of one 128-row output tile, one output row
// per thread (row == epilogue thread id == TMEM lane), from registers:
// v[t] = D[row][t] (already reduced over stream-K segments).  Store and
// residual epilogues write straight from registers; SwiGLU and RoPE pair rows
// that live in different warps, so they stage through `red` once.  Phase-level
// constants (RMSNorm factors, RoPE cos/sin of the W positions, KV pages) come
// from shared memory, prefetched at phase start.
constexpr int kFastMaxW = 32;  // decode widths served by the register-resident epilogue
struct FastEpi {
    float rn[kFastMaxW];       // RMSNorm factor per token (consumers of h)
    float cs[kFastMaxW][64];   // RoPE cos / sin at positions n_cached + t
    float sn[kFastMaxW][64];
    int page[kFastMaxW], slot[kFastMaxW];
};
// FastEpi lives in the attention K/V staging area (the epilogue warps run GEMM
// epilogues and attention items one after the other, never both at once)
static_assert(sizeof(FastEpi) <= attn_bufs(64) * 2 * kAttnChunk * 64 * 2 &&
                  sizeof(FastEpi) <= attn_bufs(128) * 2 * kAttnChunk * 128 * 2, "FastEpi exceeds the K/V staging area");

// Tokens [t0, t0 + 16) of the pass (W <= 32 runs two chunks).
__device__ void fast_tile_epilogue(const GemmArgs& a, const FastEpi& fe, int tile, int t0, float* v,
                                   const float* xv, float gcol, float* red, int tid) {
    const GemmEpiParams& e = a.epi;
    const int W = min(kChunk, a.w - t0);  // tokens of this chunk
    const int m0 = tile * kBlockM;
    if (e.ss_in != nullptr) {
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < W) v[t] = __fmul_rn(v[t], fe.rn[t0 + t]);
    }
    if (e.kind == kEpiStore) {
        float* dst = e.out + static_cast<size_t>(t0) * a.n_out + m0 + tid;
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < W) dst[static_cast<size_t>(t) * a.n_out] = v[t];
    } else if (e.kind == kEpiResidual) {
        float* dst = e.out + static_cast<size_t>(t0) * a.n_out + m0 + tid;
#pragma unroll
        for (int t = 0; t < kChunk; ++t) v[t] = t < W ? __fadd_rn(xv[t], v[t]) : 0.0f;
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < W) dst[static_cast<size_t>(t) * a.n_out] = v[t];
        if (e.u_out != nullptr) {
            __nv_bfloat16* u = e.u_out + static_cast<size_t>(t0) * a.n_out + m0 + tid;
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                if (t < W) u[static_cast<size_t>(t) * a.n_out] = __float2bfloat16_rn(__fmul_rn(v[t], gcol));
                red[t * 128 + tid] = __fmul_rn(v[t], v[t]);
            }
            epi_bar();
            // sum of squares of the tile's 128 rows per token: 8 threads per token,
            // 16 consecutive rows each (rolled), then a 3-step shuffle tree (compact
            // code: this runs once per tile on the phase boundary's critical path)
            const int t = tid >> 3, j = tid & 7;
            float sq = 0.0f;
            if (t < W) {
                const float* rr = red + t * 128 + j * 16;
#if DD_SS_UNROLL
                // 16 independent shared loads in flight, then the adds in row order
                float rv[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) rv[k] = rr[k];
#pragma unroll
                for (int k = 0; k < 16; ++k) sq = __fadd_rn(sq, rv[k]);
#else
#pragma unroll 1
                for (int k = 0; k < 16; ++k) sq = __fadd_rn(sq, rr[k]);
#endif
            }
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
            if (t < W && j == 0) e.ss_out[static_cast<size_t>(t0 + t) * a.tiles + tile] = sq;
        }
    } else {
        // SwiGLU / RoPE pair rows of different warps: stage once
#pragma unroll
        for (int t = 0; t < kChunk; ++t)
            if (t < W) red[t * 128 + tid] = v[t];
        epi_bar();
        if (e.kind == kEpiSwiGLU) {
            const int ffn = a.n_out / 2;
            for (int idx = tid; idx < W * 64; idx += kEpiThreads) {
                const int t = idx >> 6, f = idx & 63;
                const float g = red[t * 128 + f], u = red[t * 128 + 64 + f];
                const float silu = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
                e.out_bf[static_cast<size_t>(t0 + t) * ffn + tile * 64 + f] = __float2bfloat16_rn(__fmul_rn(silu, u));
            }
        } else {  // kEpiQkvRope
            const ModelDims& md = e.m;
            const int hd = md.head_dim, half = hd / 2;
            const int q_dim = md.q_dim(), kv_dim = md.kv_dim();
            if (m0 < q_dim + kv_dim) {
                for (int idx = tid; idx < W * 64; idx += kEpiThreads) {
                    const int t = idx >> 6, pr = idx & 63;
                    const int hl = pr / half, i = pr % half;
                    const int r0 = hl * hd + i;
                    const float av = red[t * 128 + r0], bv = red[t * 128 + r0 + half];
                    const float c = fe.cs[t0 + t][i], sn = fe.sn[t0 + t][i];
                    const float lo = __fmaf_rn(av, c, -__fmul_rn(bv, sn));
                    const float hi = __fmaf_rn(bv, c, __fmul_rn(av, sn));
                    const int grow = m0 + r0;
                    if (grow < q_dim) {
                        float* qd = e.q_out + static_cast<size_t>(t0 + t) * q_dim + grow;
                        qd[0] = lo;
                        qd[half] = hi;
                    } else {
                        const int kh = (grow - q_dim) / hd;
                        __nv_bfloat16* kd =
                            e.kv_pool + kv_offset(md, e.page_size, fe.page[t0 + t], e.layer, 0, kh, fe.slot[t0 + t]) + i;
                        kd[0] = __float2bfloat16_rn(lo);
                        kd[half] = __float2bfloat16_rn(hi);
                    }
                }
            } else {
                for (int idx = tid; idx < W * 128; idx += kEpiThreads) {
                    const int t = idx >> 7, r = idx & 127;
                    const int ve = m0 + r - q_dim - kv_dim;
                    e.kv_pool[kv_offset(md, e.page_size, fe.page[t0 + t], e.layer, 1, ve / hd, fe.slot[t0 + t]) + ve % hd] =
                        __float2bfloat16_rn(red[t * 128 + r]);
                }
            }
        }
    }
}

// Shared-memory ring position without divisions (the single-thread producer
// and MMA loops are issue-bound: every instruction per stage counts).
struct RingPos {
    int s = 0;         // stage
    uint32_t ph = 0;   // parity of the current use of stage s
    uint32_t n = 0;    // stages consumed so far
    __device__ __forceinline__ void next(int S) {
        if (++s == S) {
            s = 0;
            ph ^= 1u;
        }
        ++n;
    }
};

// Stream-K partition of a phase over the CTAs, optionally weighted per SM:
// SMs do not stream HBM equally fast (a stable, per-SM property measured at
// context set-up), so rank r (the rank of the CTA's SM) owns
// blocks [prefix[r] * T / prefix[P], prefix[r+1] * T / prefix[P]).  With no
// calibration (prefix == nullptr) the partition is the uniform sk_begin.
struct Partition {
    const int* begins;  // [P + 1] block offsets of this phase's ranks, or nullptr (uniform)
    int P;
    __device__ __forceinline__ int begin(int r, int T) const {
        return begins != nullptr ? begins[r] : static_cast<int>(sk_begin(r, T, P));
    }
    __device__ int owner(int g, int T) const {  // rank whose range holds block g
        int lo = 0, hi = P - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (begin(mid, T) <= g) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    }
    // segments of `tile`: the non-empty ranks covering its k-blocks; position of r
    __device__ void segments(int tile, int nkb, int T, int r, int* nseg, int* seg) const {
        if (begins == nullptr) {
            sk_segments(tile, nkb, T, P, r, nseg, seg);
            return;
        }
        const int first = owner(tile * nkb, T), last = owner((tile + 1) * nkb - 1, T);
        int n = 0, pos = 0;
        for (int k = first; k <= last; ++k)
            if (begin(k + 1, T) > begin(k, T)) {
                if (k == r) pos = n;
                ++n;
            }
        *nseg = n;
        *seg = pos;
    }
};

}  // namespace

// NCHUNK = 16-token chunks of the register-resident epilogue: 1 (W <= 16, the
// decode widths of every budget up to 16) or 2 (17 <= W <= 32); separate
// instantiations keep the common one free of the second chunk's registers.
template <int NCHUNK, int HD>
__global__ void __launch_bounds__(kPassThreads, 1)
    pass_kernel(const __grid_constant__ CUtensorMap map_h, const __grid_constant__ CUtensorMap map_o,
                const __grid_constant__ CUtensorMap map_a, const __grid_constant__ PassParams P) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned by pointer arithmetic on the __shared__ array (not an
    // integer round trip), so the compiler keeps the shared address space and
    // emits LDS/STS for every access derived from it
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nctas = gridDim.x;
    int c;  // this CTA's rank in the stream-K partition
    {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        c = P.rank_of_smid != nullptr ? P.rank_of_smid[smid] : static_cast<int>(blockIdx.x);
    }

    const int S = P.stages, nt = P.nt;
    const uint32_t b_bytes = static_cast<uint32_t>(nt) * 128u;
    const uint32_t stage_bytes = kABytes + b_bytes;
    constexpr int hd = HD;  // one instantiation per head_dim: the kernel's code stays within the I-cache budget
    uint8_t* kv_smem = smem + S * stage_bytes;                          // attention K/V chunk
    float* red = reinterpret_cast<float*>(kv_smem + attn_bufs(hd) * 2 * kAttnChunk * hd * 2);  // [kChunk][128]
    uint64_t* full = reinterpret_cast<uint64_t*>(red + kChunk * 128);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + kAccBufs;
    uint64_t* pfull = tempty + kAccBufs;  // publish ring (epilogue -> warp 3)
    uint64_t* pempty = pfull + kPubSlots;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + kPubSlots);
    __shared__ PubAction s_pub[kPubSlots];
    __shared__ int s_last;
    __shared__ float s_part[4 * 32];
    __shared__ GemmArgs s_args;
    FastEpi& s_fe = *reinterpret_cast<FastEpi*>(kv_smem);  // aliases the attention staging area
    __shared__ unsigned long long s_issue[16];  // debug: weight-load issue time per stage

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 2);  // weight producer + activation producer
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiThreads);
        }
        for (int b = 0; b < kPubSlots; ++b) {
            mbar_init(&pfull[b], 1);
            mbar_init(&pempty[b], 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&map_h);
        tma_prefetch_desc(&map_o);
        tma_prefetch_desc(&map_a);
    }
    if (warp == 1) {
        const uint32_t cols = static_cast<uint32_t>(P.tmem_buf * kAccBufs);
        if (cols <= 64) tmem_alloc<64>(tmem_slot);
        else if (cols <= 128) tmem_alloc<128>(tmem_slot);
        else if (cols <= 256) tmem_alloc<256>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int epoch = P.ps->epoch;
    const int W = P.ps->w;
    if (threadIdx.x == 0 && P.trace) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        pass_put(P, 0, 10, smid);  // debug: SM of this CTA
    }
    const int qtiles = (W + 15) / 16;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- weight producer ----------------
            const uint64_t pol_w = policy_evict_first();
            // L2 prefetch cursor runs P.prefetch blocks ahead of the ring loads,
            // across (sub-)phase boundaries, so HBM keeps streaming while a phase
            // waits for its activations
            int pf_p = -1, pf_sp = 0, pf_nsp = 0, pf_g = 0, pf_g1 = 0, pf_lkb = 0, pf_nkb = 1;
            const __nv_bfloat16* pf_src = nullptr;
            size_t pf_skip = 0;
            uint32_t pf_it = 0;
            auto pf_advance = [&](uint32_t target) {
                while (pf_it < target) {
                    while (pf_g >= pf_g1) {  // next sub-phase with work
                        if (pf_sp >= pf_nsp) {
                            if (pf_p >= P.n_phases) return;
                            do {
                                ++pf_p;
                            } while (pf_p < P.n_phases && P.phases[pf_p].type != kPhGemm);
                            if (pf_p >= P.n_phases) return;
                            pf_sp = 0;
                            pf_nsp = P.phases[pf_p].kg * P.phases[pf_p].tg;
                        }
                        const PassPhase& q = P.phases[pf_p];
                        const SubPhase sq = sub_of(q, pf_sp++);
                        const Partition pq{q.begins, nctas};
                        pf_g = pq.begin(c, sq.T);
                        pf_g1 = pq.begin(c + 1, sq.T);
                        const int lt = pf_g / sq.nkb;
                        pf_lkb = pf_g - lt * sq.nkb;
                        pf_nkb = sq.nkb;
                        pf_src = q.w + (static_cast<size_t>(sq.tile0 + lt) * q.a.nkb + sq.kb0 + pf_lkb) * 8192;
                        pf_skip = static_cast<size_t>(q.a.nkb - sq.nkb) * 8192;
                    }
                    prefetch_l2(pf_src, kABytes);
                    pf_src += 8192;
                    if (++pf_lkb == pf_nkb) {
                        pf_lkb = 0;
                        pf_src += pf_skip;
                    }
                    ++pf_g;
                    ++pf_it;
                }
            };
            RingPos rp;
            for (int p = 0; p < P.n_phases; ++p) {
                const PassPhase& ph = P.phases[p];
                if (ph.type != kPhGemm) continue;
                const Partition part{ph.begins, nctas};
                const int nsp = ph.kg * ph.tg;
                pass_stamp(P, p, 0);
                for (int sp = 0; sp < nsp; ++sp) {
                    const SubPhase sb = sub_of(ph, sp);
                    const int g0 = part.begin(c, sb.T);
                    const int g1 = part.begin(c + 1, sb.T);
                    if (g1 <= g0) continue;
                    const int lt = g0 / sb.nkb;
                    int lkb = g0 - lt * sb.nkb;
                    const __nv_bfloat16* src =
                        ph.w + (static_cast<size_t>(sb.tile0 + lt) * ph.a.nkb + sb.kb0 + lkb) * 8192;
                    const size_t skip = static_cast<size_t>(ph.a.nkb - sb.nkb) * 8192;
                    for (int g = g0; g < g1; ++g) {
                        if (P.prefetch > 0) pf_advance(rp.n + static_cast<uint32_t>(S + P.prefetch));
                        if (rp.n >= static_cast<uint32_t>(S)) mbar_wait(&empty[rp.s], rp.ph ^ 1u);
                        mbar_arrive_expect_tx(&full[rp.s], kABytes);
                        bulk_load(smem + rp.s * stage_bytes, src, kABytes, &full[rp.s], pol_w);
                        rp.next(S);
                        src += 8192;
                        if (++lkb == sb.nkb) {
                            lkb = 0;
                            src += skip;
                        }
                    }
                }
                pass_stamp(P, p, 11);
            }
        }
    } else if (warp == 2) {
        // ---------------- activation producer ----------------
        // (the whole warp polls the input flags; lane 0 feeds the ring)
        const uint64_t pol_x = policy_evict_last();
        RingPos rp;
        const int nbox = nt >> 4;
        for (int p = 0; p < P.n_phases; ++p) {
            const PassPhase& ph = P.phases[p];
            if (ph.type != kPhGemm) continue;
            const Partition part{ph.begins, nctas};
            const CUtensorMap* mx = ph.x_map == 0 ? &map_h : ph.x_map == 1 ? &map_o : &map_a;
            const int nsp = ph.kg * ph.tg;
            if (lane == 0) pass_stamp(P, p, 7);
            for (int sp = 0; sp < nsp; ++sp) {
                const SubPhase sb = sub_of(ph, sp);
                const int g0 = part.begin(c, sb.T);
                const int g1 = part.begin(c + 1, sb.T);
                if (g1 <= g0) continue;
                wait_sub_inputs(P, ph.x_src, ph.x_flag, sb, g0, g1, epoch, qtiles, lane);
                if (lane == 0) {
                    if (sp == 0) pass_stamp(P, p, 1);
                    int kb = sb.kb0 + g0 % sb.nkb;
                    const int kb_end = sb.kb0 + sb.nkb;
                    for (int g = g0; g < g1; ++g) {
                        if (rp.n >= static_cast<uint32_t>(S)) mbar_wait(&empty[rp.s], rp.ph ^ 1u);
                        mbar_arrive_expect_tx(&full[rp.s], b_bytes);
                        uint8_t* sbuf = smem + rp.s * stage_bytes + kABytes;
                        for (int r = 0; r < nbox; ++r)
                            tma_load_2d(sbuf + r * 2048, mx, &full[rp.s], kb * kBlockK, r * 16, pol_x);
                        rp.next(S);
                        if (++kb == kb_end) kb = sb.kb0;
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            const uint32_t idesc = idesc_bf16_f32(kBlockM, nt);
            RingPos rp;
            uint32_t u = 0;
            for (int p = 0; p < P.n_phases; ++p) {
                const PassPhase& ph = P.phases[p];
                if (ph.type != kPhGemm) continue;
                const Partition part{ph.begins, nctas};
                const int nsp = ph.kg * ph.tg;
                for (int sp = 0; sp < nsp; ++sp) {
                    const SubPhase sb = sub_of(ph, sp);
                    const int g0 = part.begin(c, sb.T);
                    const int g1 = part.begin(c + 1, sb.T);
                    if (g1 <= g0) continue;
                    const int tile_lo = g0 / sb.nkb, tile_hi = (g1 - 1) / sb.nkb;
                    for (int tile = tile_lo; tile <= tile_hi; ++tile, ++u) {
                        const int lo = max(g0, tile * sb.nkb);
                        const int hi = min(g1, (tile + 1) * sb.nkb);
                        const int b = u & (kAccBufs - 1);
                        if (u >= kAccBufs) mbar_wait(&tempty[b], ((u / kAccBufs) - 1) & 1u);
                        tc_fence_after();
                        const uint32_t acc = tmem + static_cast<uint32_t>(b * P.tmem_buf);
                        for (int g = lo; g < hi; ++g) {
                            mbar_wait(&full[rp.s], rp.ph);
                            tc_fence_after();
                            const uint32_t sa = smem_u32(smem + rp.s * stage_bytes);
                            const uint64_t adesc = sw128_kmajor_desc(sa);
                            const uint64_t bdesc = sw128_kmajor_desc(sa + kABytes);
#pragma unroll
                            for (int k = 0; k < kBlockK / 16; ++k)
                                umma_bf16(acc, adesc + 2 * k, bdesc + 2 * k, idesc,
                                          (g != lo || k != 0) ? 1u : 0u);
                            umma_commit(&empty[rp.s]);
                            rp.next(S);
                        }
                        umma_commit(&tfull[b]);
                    }
                }
                pass_stamp(P, p, 2);
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue / embedding / attention ----------------
        const int tid = threadIdx.x - kEpiBase;  // 0..127
        const int q = warp & 3;                  // TMEM lane quarter
        const int row = q * 32 + lane;
        uint32_t u = 0;
        uint32_t pub_n = 0;  // (thread 0) publish-ring cursor
        auto post_pub = [&](int kind, int base, int idx, int* ptr, int ph_idx) {
            if (!DD_PUB_OFFLOAD) {
                if (kind == kPubCount) asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ptr) : "memory");
                else if (kind == kPubFlag) {
                    st_release_flag(P.flags, base, idx, epoch);
                    pass_stamp(P, ph_idx, 6);
                }
                return;
            }
            const int sl = static_cast<int>(pub_n % kPubSlots);
            if (pub_n >= static_cast<uint32_t>(kPubSlots)) mbar_wait(&pempty[sl], ((pub_n / kPubSlots) - 1) & 1u);
            s_pub[sl].kind = kind;
            s_pub[sl].base = base;
            s_pub[sl].idx = idx;
            s_pub[sl].phase = ph_idx;
            s_pub[sl].ptr = ptr;
            mbar_arrive(&pfull[sl]);  // release (CTA scope): the slot and every store before the epi_bar
            ++pub_n;
        };
        for (int p = 0; p < P.n_phases; ++p) {
            const PassPhase& ph = P.phases[p];
            if (tid == 0) PASS_DBG(4, p);
            if (ph.type == kPhEmbed) {
                const int tiles = P.m.d / 128;
                for (int tile = c; tile < tiles; tile += nctas) {
                    embed_tile(P, tile, W, s_part, tid);
                    epi_bar();
                    if (tid == 0) st_release_flag(P.flags, ph.out_flag, tile, epoch);
                }
                if (tid == 0) pass_stamp(P, p, 3);
                continue;
            }
            if (ph.type == kPhAttn) {
                // only the (head, query tile, group) items that have work, numbered
                // densely (per head: the query tiles' active group counts in
                // order), CTA c taking items c, c + nctas, ...
                const int n0 = P.ps->n_cached;
                auto active_of = [&](int qt) {
                    return attn_groups((n0 + min(W, (qt + 1) * 16) - 1) / kAttnChunk + 1, P.attn_cpg, P.attn_single);
                };
                int per_head = 0;
                for (int qt = 0; qt < qtiles; ++qt) per_head += active_of(qt);
                const int items = P.m.n_heads * per_head;
                for (int item = P.attn_rank ? P.attn_rank[c] : c; item < items; item += nctas) {
                    const int head = item / per_head;
                    int grp = item % per_head, qt = 0;
                    for (int act = active_of(0); grp >= act; act = active_of(++qt)) grp -= act;
                    if (tid == 0) PASS_DBG(6, p * 100000 + item);
                    attn_item<HD>(P, ph, kv_smem, &s_last, head, qt, grp, epoch, tid, p);
                }
                if (tid == 0) pass_stamp(P, p, 3);
                continue;
            }
            // GEMM epilogue
            const Partition part{ph.begins, nctas};
            const int nsp = ph.kg * ph.tg, kg = ph.kg;
            if (tid == 0) s_args = ph.a;
            epi_bar();
            const GemmArgs& a = s_args;
            // W <= NCHUNK * 16 always (the host routes wider passes to the
            // per-launch path): one output row per thread, tokens in registers
            constexpr bool fast = true;
            const bool resid = a.epi.kind == kEpiResidual;
            const int tp_k = 2 * ph.layer + (ph.x_src == kXSwiglu ? 1 : 0);  // residual phase index (TP)
            bool consts = false;  // phase-level constants loaded (at the CTA's first sub-phase of the last k-group, before its tiles land)
            for (int sp = 0; sp < nsp; ++sp) {
                const SubPhase sb = sub_of(ph, sp);
                const int g0 = part.begin(c, sb.T), g1 = part.begin(c + 1, sb.T);
                if (g1 <= g0) continue;
                if (sb.last_k && fast && !consts) {
                    // every producer tile of this phase's input is complete before
                    // the phase-level constants are read (lanes poll in parallel)
                    consts = true;
                    const int hd_shift = P.m.head_dim == 128 ? 7 : 6;
                    const int nkb = ph.a.nkb;
                    const int n_keys = ph.x_src == kXNormed ? nkb >> 1 : ph.x_src == kXSwiglu ? nkb
                                                                         : (nkb * 64) >> hd_shift;
                    const int per_key = ph.x_src == kXAttn ? qtiles : 1;
                    for (int i = tid; i < n_keys * per_key; i += kEpiThreads) {
                        const int key = i / per_key;
                        const int idx = ph.x_src == kXAttn ? key * 16 + i % per_key : key;
                        if (!(P.nodep & 2)) wait_flag(flag_poll(P.flags, ph.x_flag, idx), epoch);
                    }
                    epi_bar();
                    const GemmEpiParams& ep = a.epi;
                    if (ep.ss_in != nullptr && tid < W) {
                        const float* ssr = ep.ss_in + static_cast<size_t>(tid) * ep.ss_tiles;
                        float acc = 0.0f;
                        for (int i0 = 0; i0 < ep.ss_tiles; i0 += 16) {
                            float v16[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j) v16[j] = i0 + j < ep.ss_tiles ? __ldcg(ssr + i0 + j) : 0.0f;
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (i0 + j < ep.ss_tiles) acc = __fadd_rn(acc, v16[j]);
                        }
                        s_fe.rn[tid] = 1.0f / sqrtf(__fadd_rn(__fdiv_rn(acc, static_cast<float>(ep.norm_d)), ep.eps));
                    }
                    if (ep.kind == kEpiQkvRope) {
                        const int half = P.m.head_dim / 2;
                        const int n0 = P.ps->n_cached;
                        for (int idx = tid; idx < W * half; idx += kEpiThreads) {
                            const int t = idx / half, i = idx % half;
                            s_fe.cs[t][i] = ep.rope_cos[static_cast<size_t>(n0 + t) * half + i];
                            s_fe.sn[t][i] = ep.rope_sin[static_cast<size_t>(n0 + t) * half + i];
                        }
                        if (tid < W) {
                            const int pos = n0 + tid;
                            s_fe.page[tid] = ep.page_table[pos / ep.page_size];
                            s_fe.slot[tid] = pos % ep.page_size;
                        }
                    }
                    epi_bar();
                }
                const int tile_lo = g0 / sb.nkb, tile_hi = (g1 - 1) / sb.nkb;
                for (int tile = tile_lo; tile <= tile_hi; ++tile, ++u) {
                    int nseg, seg;
                    part.segments(tile, sb.nkb, sb.T, c, &nseg, &seg);
                    const int gtile = sb.tile0 + tile;  // global output tile
                    // the tile's reducer: segment 0 of its last k-group (every other
                    // (k-group, segment) stores a partial); a lone segment of a
                    // single k-group runs the epilogue directly
                    const bool reducer = sb.last_k && seg == 0;
                    const int n_part = kg * nseg;  // partials + the reducer's own accumulator
                    const int b = u & (kAccBufs - 1);
                    float xv[kChunk];
                    float gcol = 1.0f;
                    if (fast && resid && reducer) {  // residual rows of this tile, before the accumulator lands
#pragma unroll
                        for (int t = 0; t < kChunk; ++t)
                            xv[t] = t < W ? __ldcg(a.epi.out + static_cast<size_t>(t) * a.n_out + gtile * kBlockM + tid) : 0.0f;
                        if (a.epi.u_out != nullptr) gcol = a.epi.gain[gtile * kBlockM + tid];
                    }
                    mbar_wait(&tfull[b], (u / kAccBufs) & 1u);
                    if (tid == 0) pass_stamp(P, p, 4);  // debug: accumulator of the CTA's latest tile ready
                    __syncwarp();
                    tc_fence_after();
                    const uint32_t t_lane =
                        tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * P.tmem_buf);
                    bool publish = false;
                    if (fast) {
                        // tokens in chunks of 16 (W <= 32: two chunks), one TMEM load each
                        const int nch = NCHUNK == 1 ? 1 : (W + kChunk - 1) / kChunk;
                        // partial layout [tile][k-group][segment][row][Wp] (Wp = W rounded
                        // up to 4): one 16-byte store / load per 4 tokens
                        const int Wp = (W + 3) & ~3;
                        const size_t slot_floats = static_cast<size_t>(Wp) * 128;
                        float* tile_ws = a.ws + static_cast<size_t>(gtile) * kg * a.max_seg * slot_floats +
                                         static_cast<size_t>(row) * Wp;
                        auto next_xv = [&](int t0) {  // residual rows of a later chunk
                            if (!resid) return;
#pragma unroll
                            for (int t = 0; t < kChunk; ++t)
                                xv[t] = t0 + t < W
                                            ? __ldcg(a.epi.out + static_cast<size_t>(t0 + t) * a.n_out + gtile * kBlockM + tid)
                                            : 0.0f;
                        };
                        if (n_part == 1) {
#pragma unroll 1
                            for (int ch = 0; ch < nch; ++ch) {
                                float v[16];
                                tmem_ld16(t_lane + ch * kChunk, v);
                                if (ch == nch - 1) {
                                    tc_fence_before();
                                    mbar_arrive(&tempty[b]);
                                }
                                if (ch > 0) {
                                    epi_bar();  // `red` of the previous chunk consumed
                                    next_xv(ch * kChunk);
                                }
                                if (NCHUNK == 1 && resid && P.tp.size > 1) tp_exchange(P, tp_k, gtile, v, tid, epoch);
                                fast_tile_epilogue(a, s_fe, gtile, ch * kChunk, v, xv, gcol, red, tid);
                            }
                            publish = true;
                        } else if (!reducer) {
                            // The reducer (segment 0 of the last k-group: the tile's first
                            // k-blocks of that group sit at the END of its CTA's range, so it
                            // finishes last) waits for the others: they store their partial
                            // and bump the tile counter with a fire-and-forget release; it
                            // adds them in (k-group, segment) order to its own registers.
                            float* part = tile_ws + static_cast<size_t>(sb.ki * a.max_seg + seg) * slot_floats;
#pragma unroll 1
                            for (int ch = 0; ch < nch; ++ch) {
                                float v[16];
                                tmem_ld16(t_lane + ch * kChunk, v);
#pragma unroll
                                for (int q4 = 0; q4 < 4; ++q4)
                                    if (ch * kChunk + 4 * q4 < W)
                                        reinterpret_cast<float4*>(part)[ch * 4 + q4] =
                                            make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
                            }
                            tc_fence_before();
                            mbar_arrive(&tempty[b]);
                            epi_bar();  // every partial store happens-before the release
                            if (tid == 0) post_pub(kPubCount, 0, 0, &a.epi.counters[gtile * kCounterStride], p);
                        } else {
                            if (tid == 0) {
                                while (!(P.nodep & 8) && ld_acquire(&a.epi.counters[gtile * kCounterStride]) < n_part - 1)
                                    __nanosleep(32);
                                a.epi.counters[gtile * kCounterStride] = 0;
                                pass_stamp(P, p, 5);  // debug: reducer saw every partial
                            }
                            epi_bar();
                            const int own = (kg - 1) * nseg;  // flat index of the reducer's own slot
#pragma unroll 1
                            for (int ch = 0; ch < nch; ++ch) {
                                float acc[16];
                                tmem_ld16(t_lane + ch * kChunk, acc);
                                if (ch == nch - 1) {
                                    tc_fence_before();
                                    mbar_arrive(&tempty[b]);
                                }
                                // partials in batches of kSumBatch loads in flight per thread
                                for (int o0 = 0; o0 < n_part - 1; o0 += kSumBatch) {
                                    float4 pv[kSumBatch][4];
#pragma unroll
                                    for (int k = 0; k < kSumBatch; ++k) {
                                        const int f = o0 + k < own ? o0 + k : o0 + k + 1;  // flat (k-group, segment)
                                        const int ki = f / nseg, si = f - ki * nseg;
                                        const float4* src = reinterpret_cast<const float4*>(
                                            tile_ws + static_cast<size_t>(ki * a.max_seg + si) * slot_floats);
#pragma unroll
                                        for (int q4 = 0; q4 < 4; ++q4)
                                            pv[k][q4] = (o0 + k < n_part - 1 && ch * kChunk + 4 * q4 < W)
                                                            ? __ldcg(src + ch * 4 + q4)
                                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                                    }
#pragma unroll
                                    for (int k = 0; k < kSumBatch; ++k)
                                        if (o0 + k < n_part - 1)
#pragma unroll
                                            for (int q4 = 0; q4 < 4; ++q4) {
                                                acc[4 * q4] = __fadd_rn(acc[4 * q4], pv[k][q4].x);
                                                acc[4 * q4 + 1] = __fadd_rn(acc[4 * q4 + 1], pv[k][q4].y);
                                                acc[4 * q4 + 2] = __fadd_rn(acc[4 * q4 + 2], pv[k][q4].z);
                                                acc[4 * q4 + 3] = __fadd_rn(acc[4 * q4 + 3], pv[k][q4].w);
                                            }
                                }
                                if (tid == 0) pass_stamp(P, p, 8);  // debug: partials summed
                                if (ch > 0) {
                                    epi_bar();
                                    next_xv(ch * kChunk);
                                }
                                if (NCHUNK == 1 && resid && P.tp.size > 1) tp_exchange(P, tp_k, gtile, acc, tid, epoch);
                                fast_tile_epilogue(a, s_fe, gtile, ch * kChunk, acc, xv, gcol, red, tid);
                            }
                            if (tid == 0) pass_stamp(P, p, 9);
                            publish = true;
                        }
                    }
                    if (publish) {
                        epi_bar();  // every epilogue store happens-before the release
                        if (tid == 0) post_pub(kPubFlag, ph.out_flag, gtile, nullptr, p);
                    }
                }
            }
            epi_bar();  // s_args reuse by the next phase
            if (tid == 0) pass_stamp(P, p, 3);
        }
        if (tid == 0) post_pub(kPubExit, 0, 0, nullptr, 0);
    } else if (warp == 3 && DD_PUB_OFFLOAD) {
        // ---------------- publisher ----------------
        // gpu-scope releases on behalf of the epilogue, in its order: one
        // acq_rel fence (cumulative over the epilogue's stores, which
        // happen-before the slot's mbarrier arrive) and the relaxed update
        if (lane == 0) {
            for (uint32_t n = 0;; ++n) {
                const int sl = static_cast<int>(n % kPubSlots);
                mbar_wait(&pfull[sl], (n / kPubSlots) & 1u);
                const PubAction act = s_pub[sl];
                mbar_arrive(&pempty[sl]);
                if (act.kind == kPubExit) break;
                if (act.kind == kPubCount) {
                    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(act.ptr) : "memory");
                } else {
                    st_release_flag(P.flags, act.base, act.idx, epoch);
                    pass_stamp(P, act.phase, 6);
                }
            }
        }
    }
    if (threadIdx.x == 0) PASS_DBG(7, -1);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        const uint32_t cols = static_cast<uint32_t>(P.tmem_buf * kAccBufs);
        if (cols <= 64) tmem_dealloc<64>(tmem);
        else if (cols <= 128) tmem_dealloc<128>(tmem);
        else if (cols <= 256) tmem_dealloc<256>(tmem);
        else tmem_dealloc<512>(tmem);
    }
#endif
}

void* pass_debug_enable(int on) {
    static int* host = nullptr;
    if (on && !host) {
        cudaHostAlloc(&host, sizeof(int) * kNumSMs * 8, cudaHostAllocMapped);
        memset(host, 0, sizeof(int) * kNumSMs * 8);
        int* dev = nullptr;
        cudaHostGetDevicePointer(&dev, host, 0);
        cudaMemcpyToSymbol(g_pass_dbg, &dev, sizeof(dev));
    }
    return host;
}

size_t pass_attn_part_floats(const ModelDims& m) {
    return static_cast<size_t>(m.n_heads) * 16 * kAttnGroups * 16 * (m.head_dim + 2);
}
size_t pass_attn_cnt_ints(const ModelDims& m) { return static_cast<size_t>(m.n_heads) * 16; }

int pass_smem_bytes(const ModelDims& m, int nt, int* stages) {
    const int stage_bytes = static_cast<int>(kABytes) + nt * 128;
    const int fixed = 1024 /* align */ + attn_bufs(m.head_dim) * 2 * kAttnChunk * m.head_dim * 2 + kChunk * 128 * 4 + 64 * 8 + 64;
    const int budget = 225 * 1024 - 2048 /* static shared */;
    static const int cap = getenv("DD_PASS_STAGES") ? atoi(getenv("DD_PASS_STAGES")) : DD_PASS_STAGE_CAP;
    int s = (budget - fixed) / stage_bytes;
    s = s > cap ? cap : s;
    if (s < 2) return -1;
    *stages = s;
    return fixed + s * stage_bytes;
}

cudaError_t launch_pass_kernel(const CUtensorMap& map_h, const CUtensorMap& map_o,
                               const CUtensorMap& map_a, const PassParams& p, int smem_bytes,
                               int nctas, cudaStream_t s) {
    static int attr_set[kMaxDevices][4] = {};  // per device: TP ranks of one process
    const int dev = current_device_slot();
    const int two = p.nt > kChunk ? 1 : 0;
    const int v = two * 2 + (p.m.head_dim == 128 ? 1 : 0);
    void (*const fns[4])(CUtensorMap, CUtensorMap, CUtensorMap, PassParams) = {
        pass_kernel<1, 64>, pass_kernel<1, 128>, pass_kernel<2, 64>, pass_kernel<2, 128>};
    if (p.nt > 2 * kChunk || (p.m.head_dim != 64 && p.m.head_dim != 128)) return cudaErrorInvalidValue;
    if (attr_set[dev][v] < smem_bytes) {
        cudaError_t e = cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        if (e != cudaSuccess) return e;
        attr_set[dev][v] = smem_bytes;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nctas, 1, 1);
    cfg.blockDim = dim3(kPassThreads, 1, 1);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fns[v], map_h, map_o, map_a, p);
}

}  // namespace dd

namespace dd {
void preload_pass_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, pass_kernel<1, 64>);
    cudaFuncGetAttributes(&a, pass_kernel<1, 128>);
    cudaFuncGetAttributes(&a, pass_kernel<2, 64>);
    cudaFuncGetAttributes(&a, pass_kernel<2, 128>);
}
}  // namespace dd
