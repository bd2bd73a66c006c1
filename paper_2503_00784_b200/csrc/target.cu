// Target-side context of the C ABI (include/duodec_b200.h): device weights,
// paged bf16 KV cache, the scored verification pass (one CUDA graph per pass
// width) and the acceptance kernel launch.
//
// A dd_ctx replaces the reference's ModelSpec on the target role
// (proj/include/duodec/model.hpp:57-65) but is stateful: it owns the KV cache
// and n_cached, so dd_score must be given exactly the tokens that are not yet
// cached ([last committed token] ++ tail).
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "accept.h"
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "gemm_epi.cuh"
#include "model.h"
#include "pass.h"

using namespace dd;

namespace dd {
// every kernel of each translation unit, loaded at context creation
void preload_accept_kernels();
void preload_attention_kernels();
void preload_attention_f32_kernels();
void preload_gemm_kernels();
void preload_gemm_wide_kernels();
void preload_model_kernels();
void preload_tp_kernels();
void preload_pass_kernels();
}  // namespace dd

thread_local std::string g_last_error;

extern "C" int dd_debug_pass_timeline(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_phases);
extern "C" int dd_pass_balance(dd_ctx* ctx);

#define CK(expr)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            return ctx_fail(ctx, DD_E_CUDA, std::string(#expr) + ": " +               \
                                                cudaGetErrorString(e_));              \
        }                                                                             \
    } while (0)

int ctx_fail(dd_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    g_last_error = msg;
    return code;
}

namespace {

enum GemmId { kGQkv = 0, kGO = 1, kGGu = 2, kGDown = 3, kGHead = 4, kNumGemm = 5 };

int round_nt(int w) { return std::max(16, (w + 15) / 16 * 16); }

void gemm_shape(const dd_ctx* c, int id, int* n_out, int* k) {
    const ModelDims& m = c->m;
    switch (id) {
        case kGQkv: *n_out = m.qkv_rows(); *k = m.d; break;
        case kGO: *n_out = m.d; *k = m.q_dim(); break;
        case kGGu: *n_out = 2 * m.ffn; *k = m.d; break;
        case kGDown: *n_out = m.d; *k = m.ffn; break;
        default: *n_out = m.vocab; *k = m.d; break;
    }
}

// CTAs per (head, query tile) of the per-launch attention kernel: one CTA
// walking the 128-key splits in sequence (no cluster merge, 1/8 of the CTAs)
// when the (head, query tile) pairs alone fill the GPU or the context spans at
// most DD_ATTN_SINGLE_MAX splits; else a cluster of 8 with a DSMEM merge
// (measured: 2K-token prefill 124 -> 101 ms, 128-token pass 5.33 -> 4.87 ms).
int attn_ranks(const dd_ctx* c, int w) {
    static const int single_max = getenv("DD_ATTN_SINGLE_MAX") ? atoi(getenv("DD_ATTN_SINGLE_MAX")) : 2;
    const int splits = (c->n_cached + w - 1) / 128 + 1;
    const int items = (w + 15) / 16 * c->m.n_heads;
    return (splits <= single_max || items >= 128) ? 1 : 8;
}

const GemmPlan& plan_for(dd_ctx* c, int id, int nt) {
    auto key = id * 1000 + nt;
    auto it = c->plans.find(key);
    if (it != c->plans.end()) return it->second;
    int n_out, k;
    gemm_shape(c, id, &n_out, &k);
    return c->plans[key] = plan_gemm(n_out, k, nt, c->fp32acc ? 1 : 0);
}

}  // namespace

// Enqueue one scored pass of width w on ctx->stream (all state via d_ps).
// `mark(cls)` (optional) records a CUDA event after each kernel for profiling:
// cls 0 = GEMM (+fused epilogue), 1 = attention, 2 = norms/embedding.
template <typename Mark>
int enqueue_pass_impl(dd_ctx* ctx, int w, bool want_logits, Mark mark) {
    const ModelDims& m = ctx->m;
    const int nt = round_nt(w);
    cudaStream_t s = ctx->stream;
    GemmEpiParams e{};
    e.counters = ctx->counters;
    e.ps = ctx->d_ps;
    e.rope_cos = ctx->rope_cos;
    e.rope_sin = ctx->rope_sin;
    e.q_out = ctx->q;
    e.kv_pool = ctx->kv_pool;
    e.page_table = ctx->page_table;
    e.page_size = ctx->page_size;
    e.m = m;
    // passes of 17..128 tokens run the tokens-on-M GEMM (gemm_wide.cu), ahead of
    // the skinny stream-K GEMM at every width above 16 with 128-row tiles
    // (scripts/wide_crossover.py: 4.29 vs 4.65 ms at 17, 4.69 vs 5.99 at 40)
    static const int wide_min = getenv("DD_WIDE_MIN") ? atoi(getenv("DD_WIDE_MIN")) : 17;
    const bool wide = w >= wide_min && w <= 128 && ctx->ws_wide != nullptr;
    auto gemm = [&](int id, const __nv_bfloat16* mw, const CUtensorMap* mx,
                    const GemmEpiParams& ep) -> cudaError_t {
        int n_out, k;
        gemm_shape(ctx, id, &n_out, &k);
        cudaError_t r;
        if (ctx->fp32acc) {  // split activations: hi + lo MMAs into one accumulator
            const CUtensorMap* lo = mx == &ctx->map_h ? &ctx->map_h_lo
                                    : mx == &ctx->map_o ? &ctx->map_o_lo : &ctx->map_a_lo;
            r = launch_gemm(mw, mx, n_out, k, w, nt, plan_for(ctx, id, nt), ctx->ws, ep, s, lo);
        } else if (wide) {
            const CUtensorMap* m128 = mx == &ctx->map_h ? &ctx->map_h128
                                      : mx == &ctx->map_o ? &ctx->map_o128 : &ctx->map_a128;
            r = launch_gemm_wide(mw, m128, n_out, k, w, ctx->wide_plans[id], ctx->ws_wide, ep, s);
        } else {
            const GemmPlan& p = plan_for(ctx, id, nt);
            r = launch_gemm(mw, mx, n_out, k, w, nt, p, ctx->ws, ep, s);
        }
        mark(0);
        return r;
    };
    // Row-parallel GEMM (O, down): unsharded, the residual epilogue is fused;
    // under tensor parallelism the GEMM stores its fp32 partial and
    // tp_reduce_residual sums the ranks' partials and applies the same epilogue.
    const bool tp = ctx->tp_size > 1;
    const int tp_ops = 2 * m.n_layers + 1;
    int tp_op = 0;
    auto row_parallel = [&](int id, const __nv_bfloat16* mw, const CUtensorMap* mx,
                            const GemmEpiParams& er) -> cudaError_t {
        if (!tp) return gemm(id, mw, mx, er);
        GemmEpiParams ep = er;
        ep.kind = kEpiStore;
        ep.out = ctx->tp_peers.part[ctx->tp_rank] + static_cast<size_t>(tp_op & 1) * ctx->tp_lay.part_stride;
        ep.u_out = nullptr;
        cudaError_t r = gemm(id, mw, mx, ep);
        if (r != cudaSuccess) return r;
        launch_tp_reduce_residual(ctx->tp_peers, ctx->d_ps, tp_op, tp_ops, m.d, er.out, er.u_out,
                                  er.gain, er.ss_out, s);
        mark(2);
        ++tp_op;
        return cudaGetLastError();
    };
    const int d_tiles = m.d / 128;
    // deferred RMSNorm: consumers of h scale by r computed from ss partials
    e.ss_in = ctx->ss;
    e.ss_tiles = d_tiles;
    e.eps = m.eps;
    e.norm_d = m.d;
    launch_embed_norm(ctx->d_ps, w, ctx->emb, ctx->gain_ones, m.d, m.eps, ctx->x, ctx->h, ctx->ss,
                      s, ctx->h_lo);
    mark(2);
    if (ctx->fp32acc) e.kv_f32 = ctx->kv_f32;
    for (int l = 0; l < m.n_layers; ++l) {
        const LayerW& L = ctx->layers[l];
        GemmEpiParams eq = e;
        eq.kind = kEpiQkvRope;
        eq.layer = l;
        CK(gemm(kGQkv, L.qkv, &ctx->map_h, eq));
        if (ctx->fp32acc) {
            if (launch_attention_f32(ctx->d_ps, w, m, ctx->q, ctx->kv_f32, ctx->page_table,
                                     ctx->page_size, l, ctx->max_seq, ctx->o, ctx->o_lo, s))
                return ctx_fail(ctx, DD_E_CUDA, "fp32 attention launch failed");
        } else if (launch_attention(ctx->d_ps, w, m, ctx->q, ctx->kv_pool, ctx->page_table,
                                    ctx->page_size, l, ctx->o, s, attn_ranks(ctx, w))) {
            return ctx_fail(ctx, DD_E_CUDA, "attention launch failed");
        }
        mark(1);
        GemmEpiParams er = e;  // residual add; writes u = bf16(x*g) + ss partials
        er.kind = kEpiResidual;
        er.out = ctx->x;
        er.ss_in = nullptr;
        er.u_out = ctx->h;
        er.lo_out = ctx->h_lo;
        er.gain = ctx->gain_ones;
        er.ss_out = ctx->ss;
        CK(row_parallel(kGO, L.o, &ctx->map_o, er));
        GemmEpiParams eg = e;
        eg.kind = kEpiSwiGLU;
        eg.out_bf = ctx->a;
        eg.lo_out = ctx->a_lo;
        CK(gemm(kGGu, L.gu, &ctx->map_h, eg));
        CK(row_parallel(kGDown, L.dn, &ctx->map_a, er));
    }
    if (want_logits) {
        GemmEpiParams el = e;
        el.kind = kEpiStore;
        el.out = tp ? ctx->tp_peers.lg[ctx->tp_rank] : ctx->logits;
        CK(gemm(kGHead, ctx->head, &ctx->map_h, el));
        if (tp) {
            launch_tp_gather_logits(ctx->tp_peers, ctx->d_ps, tp_op, tp_ops, ctx->vocab, ctx->logits, s);
            mark(2);
        }
    }
    CK(cudaGetLastError());
    return DD_OK;
}


// ------------------------------------------------------------ persistent pass
namespace {

// max stream-K segments of one tile when T blocks are cut over kNumSMs CTAs
// host mirror of pass.cu's Partition (weighted when calibrated)
struct HostPartition {
    const std::vector<int>* prefix;  // [P + 1] or empty
    int P;
    int begin(int r, int T) const {
        if (prefix == nullptr || prefix->empty()) return static_cast<int>(gemm_dev::sk_begin(r, T, P));
        return static_cast<int>(static_cast<unsigned long long>((*prefix)[r]) * static_cast<unsigned>(T) /
                                static_cast<unsigned>((*prefix)[P]));
    }
    int owner(int g, int T) const {
        int lo = 0, hi = P - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (begin(mid, T) <= g) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    }
    int nseg(int tile, int nkb, int T) const {
        const int first = owner(tile * nkb, T), last = owner((tile + 1) * nkb - 1, T);
        int n = 0;
        for (int k = first; k <= last; ++k)
            if (begin(k + 1, T) > begin(k, T)) ++n;
        return n;
    }
};

int pass_max_seg(const dd_ctx* ctx, int tiles, int nkb) {
    const HostPartition hp{&ctx->sk_prefix_h, ctx->pass_ctas};
    const int T = tiles * nkb;
    int ms = 1;
    for (int t = 0; t < tiles; ++t) ms = std::max(ms, hp.nseg(t, nkb, T));
    return ms;
}

// Sub-phase grid (k-groups x tile groups) of each GEMM of the persistent pass
// (PassPhase.kg / tg): DD_PASS_SPLIT="KGxTG,..." in the order qkv, o, gate/up,
// down, head overrides the default.  A split must divide the tiles and
// k-blocks and keep every tile within the partial-slot limit; otherwise, and
// for passes wider than 32 tokens (the per-thread epilogue), 1x1.
void pass_split(const dd_ctx* ctx, int id, int w, int* kg, int* tg) {
    static int cfg[kNumGemm][2] = {{-1, -1}};
    if (cfg[0][0] < 0) {
        // gate/up publishes two tile groups and down consumes them as two
        // k-groups, so most of down starts on the first half of the SwiGLU
        // output (W=9: 3.157 -> 3.113 ms); every other split measured slower
        // (more segments and polls per phase than it saves)
        static const int def[kNumGemm][2] = {{1, 1}, {1, 1}, {1, 2}, {2, 1}, {1, 1}};
        for (int i = 0; i < kNumGemm; ++i) {
            cfg[i][0] = def[i][0];
            cfg[i][1] = def[i][1];
        }
        if (const char* e = getenv("DD_PASS_SPLIT")) {
            for (int i = 0; i < kNumGemm && *e; ++i) {
                int a = 1, b = 1, nc = 0;
                if (sscanf(e, "%dx%d%n", &a, &b, &nc) == 2) {
                    cfg[i][0] = a;
                    cfg[i][1] = b;
                    e += nc;
                }
                if (*e == ',') ++e;
            }
        }
    }
    *kg = 1;
    *tg = 1;
    if (w > 32) return;
    int n_out, k;
    gemm_shape(ctx, id, &n_out, &k);
    const int tiles = n_out / 128, nkb = k / 64, a = cfg[id][0], b = cfg[id][1];
    if (a < 1 || b < 1 || tiles % b || nkb % a) return;
    if (a * pass_max_seg(ctx, tiles / b, nkb / a) > 64) return;  // partial slots per tile
    *kg = a;
    *tg = b;
}

// partial-buffer floats of one GEMM's phase (every split it may run with)
size_t pass_ws_floats(const dd_ctx* ctx, int id) {
    int n_out, k;
    gemm_shape(ctx, id, &n_out, &k);
    size_t best = static_cast<size_t>(n_out / 128) * pass_max_seg(ctx, n_out / 128, k / 64);
    int kg, tg;
    pass_split(ctx, id, 1, &kg, &tg);
    best = std::max(best, static_cast<size_t>(n_out / 128) * kg * pass_max_seg(ctx, n_out / 128 / tg, k / 64 / kg));
    return best * kMaxPassTokens * 128;
}

int tmem_buf_for(int nt) {
    int buf = 32;
    while (buf < nt) buf <<= 1;
    return buf;
}

// Phase table of a pass of width w: embed, per layer QKV / attention / O /
// gate-up / down, then the LM head (when logits are wanted).
int build_pass_phases(dd_ctx* ctx, int w, bool want_logits, const PassPhase** out, int* n_out) {
    const int key = w * 2 + (want_logits ? 1 : 0);
    auto it = ctx->pass_phases.find(key);
    if (it != ctx->pass_phases.end()) {
        *out = it->second;
        *n_out = ctx->pass_nphases[key];
        return DD_OK;
    }
    const ModelDims& m = ctx->m;
    const int nt = round_nt(w);
    std::vector<PassPhase> ph;
    GemmEpiParams e{};
    e.ps = ctx->d_ps;
    e.rope_cos = ctx->rope_cos;
    e.rope_sin = ctx->rope_sin;
    e.q_out = ctx->q;
    e.kv_pool = ctx->kv_pool;
    e.page_table = ctx->page_table;
    e.page_size = ctx->page_size;
    e.m = m;
    e.ss_in = ctx->ss;
    e.ss_tiles = m.d / 128;
    e.eps = m.eps;
    e.norm_d = m.d;
    int gidx = 0;
    int next_flag = 0;  // flags are packed: each phase reserves exactly its count
    auto reserve = [&](int n) {
        const int b = next_flag;
        next_flag += n;
        return b;
    };
    auto gemm = [&](int id, const __nv_bfloat16* W, int x_map, int x_src, int x_flag,
                    GemmEpiParams ep, int layer) {
        PassPhase p{};
        p.type = kPhGemm;
        p.x_map = x_map;
        p.x_src = x_src;
        p.x_flag = x_flag;
        p.layer = layer;
        p.w = W;
        int n_outr, k;
        gemm_shape(ctx, id, &n_outr, &k);
        GemmArgs& a = p.a;
        a.n_out = n_outr;
        a.k = k;
        a.w = w;
        a.nt = nt;
        a.tiles = n_outr / 128;
        a.nkb = k / 64;
        pass_split(ctx, id, w, &p.kg, &p.tg);
        a.max_seg = pass_max_seg(ctx, a.tiles / p.tg, a.nkb / p.kg);
        a.tmem_buf = tmem_buf_for(nt);
        a.ws = ctx->pass_ws + (gidx & 1) * ctx->pass_ws_half;
        ep.counters = ctx->pass_counters + (gidx & 1) * 512 * kCounterStride;
        a.epi = ep;
        p.out_flag = reserve(a.tiles);
        ++gidx;
        ph.push_back(p);
        return p.out_flag;
    };
    PassPhase pe{};
    pe.type = kPhEmbed;
    pe.out_flag = reserve(m.d / 128);
    ph.push_back(pe);
    int h_flag = pe.out_flag;  // producer of h (tile = 128 columns)
    for (int l = 0; l < m.n_layers; ++l) {
        const LayerW& L = ctx->layers[l];
        GemmEpiParams eq = e;
        eq.kind = kEpiQkvRope;
        eq.layer = l;
        const int qkv_flag = gemm(kGQkv, L.qkv, 0, kXNormed, h_flag, eq, l);
        PassPhase pa{};
        pa.type = kPhAttn;
        pa.layer = l;
        pa.qkv_flag = qkv_flag;
        pa.out_flag = reserve(m.n_heads * 16);
        ph.push_back(pa);
        GemmEpiParams er = e;
        er.kind = kEpiResidual;
        er.out = ctx->x;
        er.ss_in = nullptr;
        er.u_out = ctx->h;
        er.gain = ctx->gain_ones;
        er.ss_out = ctx->ss;
        h_flag = gemm(kGO, L.o, 1, kXAttn, pa.out_flag, er, l);
        GemmEpiParams eg = e;
        eg.kind = kEpiSwiGLU;
        eg.out_bf = ctx->a;
        const int gu_flag = gemm(kGGu, L.gu, 0, kXNormed, h_flag, eg, l);
        h_flag = gemm(kGDown, L.dn, 2, kXSwiglu, gu_flag, er, l);
    }
    if (want_logits) {
        GemmEpiParams el = e;
        el.kind = kEpiStore;
        el.out = ctx->tp_size > 1 ? ctx->tp_peers.lg[ctx->tp_rank] : ctx->logits;
        gemm(kGHead, ctx->head, 0, kXNormed, h_flag, el, m.n_layers);
    }
    if (static_cast<size_t>(next_flag) > ctx->pass_flag_count)
        return ctx_fail(ctx, DD_E_CAPACITY, "pass flag table too small");
    if (!ctx->sk_prefix_h.empty()) {
        // weighted partition: per GEMM phase, the block offset of every rank
        const std::vector<int>& pre = ctx->sk_prefix_h;
        std::vector<int> hb;
        std::vector<size_t> off(ph.size(), 0);
        for (size_t i = 0; i < ph.size(); ++i) {
            if (ph[i].type != kPhGemm) continue;
            // every sub-phase of a GEMM has the same shape: one partition
            const unsigned T = static_cast<unsigned>((ph[i].a.tiles / ph[i].tg) * (ph[i].a.nkb / ph[i].kg));
            off[i] = hb.size();
            for (int r = 0; r <= kNumSMs; ++r)
                hb.push_back(static_cast<int>(static_cast<unsigned long long>(pre[r]) * T / pre[kNumSMs]));
        }
        int* db = nullptr;
        CK(cudaMalloc(&db, sizeof(int) * hb.size()));
        CK(cudaMemcpy(db, hb.data(), sizeof(int) * hb.size(), cudaMemcpyHostToDevice));
        ctx->pass_begins.push_back(db);
        for (size_t i = 0; i < ph.size(); ++i)
            if (ph[i].type == kPhGemm) ph[i].begins = db + off[i];
    }
    {
        // Attention items go first to the CTAs with no QKV reducer duty (their
        // QKV range holds no tile start, so their epilogue only stores a partial
        // and is free first); the reducers follow.  Same order on every pass.
        static const bool order = !(getenv("DD_ATTN_ORDER") && getenv("DD_ATTN_ORDER")[0] == '0');
        const int P = ctx->pass_ctas;
        int kg = 1, tg = 1;
        pass_split(ctx, kGQkv, w, &kg, &tg);
        if (order && kg == 1 && tg == 1 && ctx->attn_rank_ctas != P) {
            int n_out, k;
            gemm_shape(ctx, kGQkv, &n_out, &k);
            const int nkb = k / 64, T = (n_out / 128) * nkb;
            const HostPartition hp{&ctx->sk_prefix_h, P};
            std::vector<int> red(P), rank(P);
            int n_free = 0;
            for (int r = 0; r < P; ++r) {
                const int g0 = hp.begin(r, T), g1 = hp.begin(r + 1, T);
                red[r] = (g0 + nkb - 1) / nkb * nkb < g1 ? 1 : 0;
                n_free += 1 - red[r];
            }
            for (int r = 0, f = 0, b = 0; r < P; ++r) rank[r] = red[r] ? n_free + b++ : f++;
            if (!ctx->attn_rank_d) CK(cudaMalloc(&ctx->attn_rank_d, sizeof(int) * kNumSMs));
            CK(cudaMemcpy(ctx->attn_rank_d, rank.data(), sizeof(int) * P, cudaMemcpyHostToDevice));
            ctx->attn_rank_ctas = P;
        }
    }
    PassPhase* d = nullptr;
    CK(cudaMalloc(&d, sizeof(PassPhase) * ph.size()));
    CK(cudaMemcpy(d, ph.data(), sizeof(PassPhase) * ph.size(), cudaMemcpyHostToDevice));
    ctx->pass_phases[key] = d;
    ctx->pass_nphases[key] = static_cast<int>(ph.size());
    *out = d;
    *n_out = static_cast<int>(ph.size());
    return DD_OK;
}

int enqueue_pass_kernel(dd_ctx* ctx, int w, bool want_logits, unsigned long long* trace = nullptr) {
    const PassPhase* phases = nullptr;
    int n = 0;
    int rc = build_pass_phases(ctx, w, want_logits, &phases, &n);
    if (rc) return rc;
    const ModelDims& m = ctx->m;
    PassParams p{};
    p.phases = phases;
    p.n_phases = n;
    p.nt = round_nt(w);
    p.tmem_buf = tmem_buf_for(p.nt);
    static const int env_pf = getenv("DD_PASS_PREFETCH") ? atoi(getenv("DD_PASS_PREFETCH")) : 4;
    p.prefetch = env_pf;
    // attention items of up to 10 chunks (320 keys) run unsplit (the groups'
    // partial round trip and combine cost more than running them in sequence);
    // longer ones split into groups of 4 chunks, at most 4 groups (W=9: 512
    // keys 3.28 -> 3.23 ms, 1024 keys 3.42 -> 3.37 ms)
    static const int env_cpg = getenv("DD_ATTN_CPG") ? atoi(getenv("DD_ATTN_CPG")) : 4;
    static const int env_single = getenv("DD_ATTN_SINGLE") ? atoi(getenv("DD_ATTN_SINGLE")) : 10;
    p.attn_cpg = env_cpg;
    p.attn_single = env_single;
    static const int env_nodep = getenv("DD_PASS_NODEP") ? atoi(getenv("DD_PASS_NODEP")) : 0;
    p.nodep = env_nodep;
    const int smem = pass_smem_bytes(m, p.nt, &p.stages);
    if (smem < 0) return ctx_fail(ctx, DD_E_ARG, "pass kernel shared memory plan failed");
    p.ps = ctx->d_ps;
    p.flags = ctx->pass_flags;
    p.emb = ctx->emb;
    p.gain = ctx->gain_ones;
    p.x = ctx->x;
    p.h = ctx->h;
    p.ss = ctx->ss;
    p.m = m;
    p.q = ctx->q;
    p.kv_pool = ctx->kv_pool;
    p.page_table = ctx->page_table;
    p.page_size = ctx->page_size;
    p.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(m.head_dim)));
    p.o = ctx->o;
    p.attn_part = ctx->attn_part;
    p.attn_cnt = ctx->attn_cnt;
    p.trace = trace;
    p.rank_of_smid = ctx->rank_of_smid_d;
    {
        int kg = 1, tg = 1;
        pass_split(ctx, kGQkv, w, &kg, &tg);
        p.attn_rank = kg == 1 && tg == 1 && ctx->attn_rank_ctas == ctx->pass_ctas ? ctx->attn_rank_d : nullptr;
    }
    p.tp = ctx->tp_peers;
    p.tp.size = ctx->tp_size;
    p.tp.rank = ctx->tp_rank;
    CK(launch_pass_kernel(ctx->map_h, ctx->map_o, ctx->map_a, p, smem, ctx->pass_ctas, ctx->stream));
    if (ctx->tp_size > 1 && want_logits) {  // vocabulary-parallel head: assemble full rows (op 2L of the pass)
        const int tp_ops = 2 * m.n_layers + 1;
        launch_tp_gather_logits(ctx->tp_peers, ctx->d_ps, tp_ops - 1, tp_ops, ctx->vocab, ctx->logits, ctx->stream);
        CK(cudaGetLastError());
    }
    return DD_OK;
}

}  // namespace

// The persistent pass kernel serves decode widths; wide (prefill) passes are
// compute-heavier and run as one launch per GEMM / attention, whose
// 2-CTA-per-SM GEMM keeps more tiles in flight for the epilogue-heavy wide case.
bool use_pass_kernel(const dd_ctx* ctx, int w) {
    // DD_PASS_MAXW (A/B knob, <= 32): the register-resident epilogue serves up to
    // 32 tokens (two 16-token chunks); wider passes take the per-launch path
    static const int max_w =
        getenv("DD_PASS_MAXW") ? std::min(32, atoi(getenv("DD_PASS_MAXW"))) : 32;
    if (ctx->tp_size > 1) {
        // tensor parallel: the O / down reducers exchange their tiles in the
        // epilogue (pass.cu tp_exchange), 16-token register chunks only
        static const bool tp_pass = !(getenv("DD_TP_PASS") && getenv("DD_TP_PASS")[0] == '0');
        return tp_pass && ctx->use_pass_kernel && ctx->tp_connected && w <= 16 && ctx->m.d / 128 <= kTpPassTiles;
    }
    return ctx->use_pass_kernel && w <= max_w;
}

int enqueue_pass(dd_ctx* ctx, int w, bool want_logits, int* kernels) {
    if (use_pass_kernel(ctx, w)) {
        if (kernels) *kernels = 1 + (ctx->tp_size > 1 && want_logits ? 1 : 0);  // + TP logits gather
        return enqueue_pass_kernel(ctx, w, want_logits);
    }
    int n = 0;
    int rc = enqueue_pass_impl(ctx, w, want_logits, [&n](int) { ++n; });
    if (kernels) *kernels = n;
    return rc;
}

int ctx_mark(dd_ctx* ctx, int which) {
    cudaEvent_t* e = which == 0 ? &ctx->t_start : which == 1 ? &ctx->t_end : &ctx->t_first;
    if (!*e) CK(cudaEventCreate(e));
    CK(cudaEventRecord(*e, ctx->stream));
    return DD_OK;
}

double ctx_elapsed_ms(dd_ctx* ctx, int which) {
    cudaEvent_t e = which == 2 ? ctx->t_first : ctx->t_end;
    if (!ctx->t_start || !e) return 0.0;
    cudaEventSynchronize(e);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ctx->t_start, e);
    return ms;
}

// One-launch-per-op prefill of a long prompt chunk (w <= kMaxPrefillTokens):
// embedding, per layer the multi-tile prefill GEMMs (fused RoPE + KV append,
// residual + deferred-RMSNorm producer, SwiGLU) and the causal attention over
// the paged cache; no LM head (prefill keeps no logits).
int enqueue_prefill_big(dd_ctx* ctx, int w) {
    const ModelDims& m = ctx->m;
    cudaStream_t s = ctx->stream;
    GemmEpiParams e{};
    e.counters = ctx->counters;
    e.ps = ctx->d_ps;
    e.rope_cos = ctx->rope_cos;
    e.rope_sin = ctx->rope_sin;
    e.q_out = ctx->q;
    e.kv_pool = ctx->kv_pool;
    e.page_table = ctx->page_table;
    e.page_size = ctx->page_size;
    e.m = m;
    e.ss_in = ctx->ss;
    e.ss_tiles = m.d / 128;
    e.eps = m.eps;
    e.norm_d = m.d;
    auto gemm = [&](int id, const __nv_bfloat16* mw, const CUtensorMap* mx, const GemmEpiParams& ep) {
        int n_out, k;
        gemm_shape(ctx, id, &n_out, &k);
        return launch_gemm_prefill(mw, mx, n_out, k, w, ep, s);
    };
    launch_embed_norm(ctx->d_ps, w, ctx->emb, ctx->gain_ones, m.d, m.eps, ctx->x, ctx->h, ctx->ss, s);
    for (int l = 0; l < m.n_layers; ++l) {
        const LayerW& L = ctx->layers[l];
        GemmEpiParams eq = e;
        eq.kind = kEpiQkvRope;
        eq.layer = l;
        CK(gemm(kGQkv, L.qkv, &ctx->map_h128, eq));
        if (launch_attention_prefill(ctx->d_ps, w, m, ctx->q, ctx->kv_pool, ctx->page_table, ctx->page_size,
                                     l, ctx->o, s, ctx->has_map_kv ? &ctx->map_kv : nullptr))
            return ctx_fail(ctx, DD_E_CUDA, "attention launch failed");
        GemmEpiParams er = e;
        er.kind = kEpiResidual;
        er.out = ctx->x;
        er.ss_in = nullptr;
        er.u_out = ctx->h;
        er.gain = ctx->gain_ones;
        er.ss_out = ctx->ss;
        CK(gemm(kGO, L.o, &ctx->map_o128, er));
        GemmEpiParams eg = e;
        eg.kind = kEpiSwiGLU;
        eg.out_bf = ctx->a;
        CK(gemm(kGGu, L.gu, &ctx->map_h128, eg));
        CK(gemm(kGDown, L.dn, &ctx->map_a128, er));
    }
    CK(cudaGetLastError());
    return DD_OK;
}

// The multi-tile prefill GEMM serves unsharded bf16 contexts; below
// DD_BIG_PREFILL_MIN tokens the 128-token chunked path is faster (too few
// (token tile, weight tile) units to fill the GPU).
bool use_big_prefill(const dd_ctx* ctx, int n) {
    static const int min_n = getenv("DD_BIG_PREFILL_MIN") ? atoi(getenv("DD_BIG_PREFILL_MIN")) : 512;
    return ctx->tp_size == 1 && !ctx->fp32acc && n >= min_n;
}

int run_prefill_big(dd_ctx* ctx, const int32_t* tokens, int w) {
    if (w < 1 || w > kMaxPrefillTokens) return ctx_fail(ctx, DD_E_CAPACITY, "prefill width out of range");
    if (ctx->n_cached + w > ctx->max_seq) return ctx_fail(ctx, DD_E_CAPACITY, "KV cache capacity exceeded");
    for (int i = 0; i < w; ++i)
        if (tokens[i] < 0 || tokens[i] >= ctx->vocab) return ctx_fail(ctx, DD_E_ARG, "token outside vocabulary");
    const int slot = ctx->ps_slot;
    ctx->ps_slot = (slot + 1) % kPsRing;
    CK(cudaEventSynchronize(ctx->ps_done[slot]));
    PassState* hp = ctx->h_ps + slot;
    hp->n_cached = ctx->n_cached;
    hp->w = w;
    hp->epoch = ++ctx->epoch;
    std::memcpy(hp->tokens, tokens, sizeof(int32_t) * w);
    const size_t bytes = offsetof(PassState, tokens) + sizeof(int32_t) * w;
    CK(cudaMemcpyAsync(ctx->d_ps, hp, bytes, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += bytes;
    CK(cudaEventRecord(ctx->ps_done[slot], ctx->stream));
    int rc = enqueue_prefill_big(ctx, w);
    if (rc != DD_OK) return rc;
    ctx->launches += 1 + 5 * static_cast<uint64_t>(ctx->m.n_layers);
    ctx->n_cached += w;
    ctx->last_w = 0;
    return DD_OK;
}

// Upload pass state, then replay (or capture) the graph for width w.
int run_pass(dd_ctx* ctx, const int32_t* tokens, int w, bool want_logits) {
    if (w < 1 || w > kMaxPassTokens) return ctx_fail(ctx, DD_E_CAPACITY, "pass width out of range");
    if (ctx->n_cached + w > ctx->max_seq)
        return ctx_fail(ctx, DD_E_CAPACITY, "KV cache capacity exceeded");
    for (int i = 0; i < w; ++i)
        if (tokens[i] < 0 || tokens[i] >= ctx->vocab)
            return ctx_fail(ctx, DD_E_ARG, "token outside vocabulary");
    if (ctx->tp_size > 1 && !ctx->tp_connected)
        return ctx_fail(ctx, DD_E_STATE, "tensor-parallel ranks not connected (dd_tp_connect)");
    const int slot = ctx->ps_slot;
    ctx->ps_slot = (slot + 1) % kPsRing;
    CK(cudaEventSynchronize(ctx->ps_done[slot]));
    PassState* hp = ctx->h_ps + slot;
    hp->n_cached = ctx->n_cached;
    hp->w = w;
    hp->epoch = ++ctx->epoch;
    std::memcpy(hp->tokens, tokens, sizeof(int32_t) * w);
    CK(cudaMemcpyAsync(ctx->d_ps, hp, offsetof(PassState, tokens) + sizeof(int32_t) * w,
                       cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += offsetof(PassState, tokens) + sizeof(int32_t) * w;
    CK(cudaEventRecord(ctx->ps_done[slot], ctx->stream));
    if (ctx->use_graphs) {
        // per-launch passes bake the attention CTA layout (context-dependent) into the graph
        const int key = (w * 2 + (want_logits ? 1 : 0)) * 2 +
                        (!use_pass_kernel(ctx, w) && attn_ranks(ctx, w) == 1 ? 1 : 0);
        auto it = ctx->graphs.find(key);
        if (it == ctx->graphs.end()) {
            if (use_pass_kernel(ctx, w)) {  // device phase table: allocated outside the capture
                const PassPhase* ph = nullptr;
                int n = 0;
                int rc = build_pass_phases(ctx, w, want_logits, &ph, &n);
                if (rc != DD_OK) return rc;
            }
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            int nk = 0;
            int rc = enqueue_pass(ctx, w, want_logits, &nk);
            ctx->graph_kernels[key] = nk;
            cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
            if (rc != DD_OK) return rc;
            CK(e);
            cudaGraphExec_t ge;
            CK(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
            it = ctx->graphs.emplace(key, ge).first;
        }
        CK(cudaGraphLaunch(it->second, ctx->stream));
        ctx->launches += ctx->graph_kernels[key];
    } else {
        int nk = 0;
        int rc = enqueue_pass(ctx, w, want_logits, &nk);
        if (rc != DD_OK) return rc;
        ctx->launches += nk;
    }
    ctx->n_cached += w;
    ctx->last_w = want_logits ? w : 0;
    return DD_OK;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* dd_last_error(const dd_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_last_error.c_str();
}

int dd_ctx_create(const dd_model_desc* desc, int cuda_device, dd_ctx** out) {
    return dd_ctx_create_tp(desc, cuda_device, 0, 1, out);
}

int dd_ctx_create_tp(const dd_model_desc* desc, int cuda_device, int tp_rank, int tp_size,
                     dd_ctx** out) {
    dd_ctx* ctx = nullptr;
    if (!desc || !out) return ctx_fail(nullptr, DD_E_ARG, "null argument");
    *out = nullptr;
    const dd_model_desc& d = *desc;
    const int n_kv = d.n_kv_heads > 0 ? d.n_kv_heads : d.n_heads;
    if (tp_size < 1 || tp_size > kMaxTp || tp_rank < 0 || tp_rank >= tp_size)
        return ctx_fail(nullptr, DD_E_ARG, "bad tensor-parallel rank / size");
    // Megatron split: whole heads (q and kv) and 64-feature FFN blocks per rank
    if (d.n_heads % tp_size || n_kv % tp_size || d.ffn_dim % (64 * tp_size) ||
        d.vocab / 128 < tp_size)
        return ctx_fail(nullptr, DD_E_ARG, "shape does not split over the tensor-parallel ranks");
    const int h_l = d.n_heads / tp_size, kv_l = n_kv / tp_size, ffn_l = d.ffn_dim / tp_size;
    if (d.precision != DD_PREC_BF16 && d.precision != DD_PREC_FP32ACC)
        return ctx_fail(nullptr, DD_E_ARG, "unknown precision mode");
    if (d.precision == DD_PREC_FP32ACC && (tp_size != 1 || d.max_seq > kMaxF32AttnKeys))
        return ctx_fail(nullptr, DD_E_ARG, "fp32-accumulate mode needs tp_size 1 and max_seq <= 49152");
    if (d.n_layers < 1 || d.d_model % 128 || d.head_dim % 32 || d.head_dim > 256 ||
        d.n_heads % std::max(1, n_kv) || (tp_size == 1 && d.ffn_dim % 128) || d.vocab % 128 ||
        (h_l * d.head_dim) % 128 || (kv_l * d.head_dim) % 128 ||
        (d.head_dim != 64 && d.head_dim != 128) || d.max_seq < 1)
        return ctx_fail(nullptr, DD_E_ARG,
                        "unsupported shape (d_model, ffn_dim, vocab must be multiples of 128; "
                        "head_dim 64/128; per-rank q and kv widths multiples of 128)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cuda_device)
        return ctx_fail(nullptr, DD_E_CUDA, "no CUDA device available (no CPU fallback exists)");
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess || prop.major != 10)
        return ctx_fail(nullptr, DD_E_CUDA, "device is not sm_100 (Blackwell)");
    ctx = new dd_ctx();
    ctx->device = cuda_device;
    ctx->fp32acc = d.precision == DD_PREC_FP32ACC;
    ctx->sm_count = prop.multiProcessorCount;
    CK(cudaSetDevice(cuda_device));
    {
        // Load every kernel of the library now: with lazy module loading a
        // kernel's first launch loads its module and synchronises the device,
        // which deadlocks tensor-parallel ranks driven from one thread (a rank
        // blocks in the load while its own queued reduction waits for a peer
        // whose work is not yet issued).
        static bool loaded[kMaxDevices] = {};
        const int slot = current_device_slot();
        if (!loaded[slot]) {
            preload_accept_kernels();
            preload_attention_kernels();
            preload_attention_f32_kernels();
            preload_gemm_kernels();
            preload_gemm_wide_kernels();
            preload_model_kernels();
            preload_tp_kernels();
            preload_pass_kernels();
            CK(cudaGetLastError());
            loaded[slot] = true;
        }
    }
    ctx->tp_rank = tp_rank;
    ctx->tp_size = tp_size;
    ctx->vocab = d.vocab;
    ctx->tp_v0.resize(tp_size + 1);
    for (int r = 0; r <= tp_size; ++r)  // whole 128-row head tiles per rank
        ctx->tp_v0[r] = 128 * static_cast<int>(static_cast<int64_t>(d.vocab / 128) * r / tp_size);
    ModelDims& m = ctx->m;
    m.n_layers = d.n_layers;
    m.d = d.d_model;
    m.n_heads = h_l;
    m.n_kv_heads = kv_l;
    m.head_dim = d.head_dim;
    m.ffn = ffn_l;
    m.vocab = ctx->tp_v0[tp_rank + 1] - ctx->tp_v0[tp_rank];
    m.eps = d.rms_eps;
    m.rope_theta = d.rope_theta;
    ctx->page_size = d.page_size > 0 ? d.page_size : 16;
    ctx->n_pages = (d.max_seq + ctx->page_size - 1) / ctx->page_size;
    ctx->max_seq = ctx->n_pages * ctx->page_size;
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->q_ready, cudaEventDisableTiming));
    for (int i = 0; i < kPsRing; ++i) CK(cudaEventCreateWithFlags(&ctx->ps_done[i], cudaEventDisableTiming));

    // weights
    const size_t d_ = m.d;
    CK(cudaMalloc(&ctx->emb, sizeof(__nv_bfloat16) * ctx->vocab * d_));  // replicated
    CK(cudaMalloc(&ctx->head, sizeof(__nv_bfloat16) * m.vocab * d_));
    ctx->layers.resize(m.n_layers);
    for (auto& L : ctx->layers) {
        CK(cudaMalloc(&L.qkv, sizeof(__nv_bfloat16) * m.qkv_rows() * d_));
        CK(cudaMalloc(&L.o, sizeof(__nv_bfloat16) * d_ * m.q_dim()));
        CK(cudaMalloc(&L.gu, sizeof(__nv_bfloat16) * 2 * m.ffn * d_));
        CK(cudaMalloc(&L.dn, sizeof(__nv_bfloat16) * d_ * m.ffn));
    }
    const int gain_n = std::max(m.d, m.ffn);
    CK(cudaMalloc(&ctx->gain_ones, sizeof(float) * gain_n));
    launch_fill_f32(ctx->gain_ones, gain_n, 1.0f, ctx->stream);

    // activations (kMaxPassTokens rows so every TMA box stays in bounds)
    const size_t R = kMaxPrefillTokens;  // activation rows: one prefill pass (logits keep kMaxPassTokens)
    CK(cudaMalloc(&ctx->x, sizeof(float) * R * d_));
    CK(cudaMalloc(&ctx->h, sizeof(__nv_bfloat16) * R * d_));
    CK(cudaMalloc(&ctx->q, sizeof(float) * R * m.q_dim()));
    CK(cudaMalloc(&ctx->o, sizeof(__nv_bfloat16) * R * m.q_dim()));
    CK(cudaMalloc(&ctx->a, sizeof(__nv_bfloat16) * R * m.ffn));
    CK(cudaMemset(ctx->h, 0, sizeof(__nv_bfloat16) * R * d_));
    CK(cudaMemset(ctx->o, 0, sizeof(__nv_bfloat16) * R * m.q_dim()));
    CK(cudaMemset(ctx->a, 0, sizeof(__nv_bfloat16) * R * m.ffn));
    if (make_tmap_bf16(&ctx->map_h, ctx->h, R, d_, 16) ||
        make_tmap_bf16(&ctx->map_o, ctx->o, R, m.q_dim(), 16) ||
        make_tmap_bf16(&ctx->map_a, ctx->a, R, m.ffn, 16) ||
        make_tmap_bf16(&ctx->map_h128, ctx->h, R, d_, 128) ||
        make_tmap_bf16(&ctx->map_o128, ctx->o, R, m.q_dim(), 128) ||
        make_tmap_bf16(&ctx->map_a128, ctx->a, R, m.ffn, 128))
        return ctx_fail(ctx, DD_E_CUDA, "cuTensorMapEncodeTiled failed");
    if (ctx->fp32acc) {
        CK(cudaMalloc(&ctx->h_lo, sizeof(__nv_bfloat16) * R * d_));
        CK(cudaMalloc(&ctx->o_lo, sizeof(__nv_bfloat16) * R * m.q_dim()));
        CK(cudaMalloc(&ctx->a_lo, sizeof(__nv_bfloat16) * R * m.ffn));
        CK(cudaMemset(ctx->h_lo, 0, sizeof(__nv_bfloat16) * R * d_));
        CK(cudaMemset(ctx->o_lo, 0, sizeof(__nv_bfloat16) * R * m.q_dim()));
        CK(cudaMemset(ctx->a_lo, 0, sizeof(__nv_bfloat16) * R * m.ffn));
        if (make_tmap_bf16(&ctx->map_h_lo, ctx->h_lo, R, d_, 16) ||
            make_tmap_bf16(&ctx->map_o_lo, ctx->o_lo, R, m.q_dim(), 16) ||
            make_tmap_bf16(&ctx->map_a_lo, ctx->a_lo, R, m.ffn, 16))
            return ctx_fail(ctx, DD_E_CUDA, "cuTensorMapEncodeTiled failed");
    }
    size_t ws_floats = 0;
    for (int id = 0; id < kNumGemm; ++id) {
        int n_out, k;
        gemm_shape(ctx, id, &n_out, &k);
        for (int nt = 16; nt <= kMaxPassTokens; nt += 16) {
            const GemmPlan& p = plan_for(ctx, id, nt);
            ws_floats = std::max(ws_floats, gemm_ws_floats(p, nt));
        }
    }
    CK(cudaMalloc(&ctx->ws, sizeof(float) * ws_floats));
    {
        // tokens-on-M prefill GEMM: every shape must split into 256-row tiles
        bool ok = true;
        size_t wide_floats = 0;
        for (int id = 0; id < kNumGemm; ++id) {
            int n_out, k;
            gemm_shape(ctx, id, &n_out, &k);
            ok = ok && n_out % 128 == 0;
            if (!ok) break;
            ctx->wide_plans[id] = plan_gemm_wide(n_out, k);
            wide_floats = std::max(wide_floats, gemm_wide_ws_floats(ctx->wide_plans[id]));
        }
        // (fp32-accumulate mode runs every width on the split-activation GEMM)
        if (ok && !ctx->fp32acc) CK(cudaMalloc(&ctx->ws_wide, sizeof(float) * wide_floats));
    }
    CK(cudaMalloc(&ctx->counters, sizeof(int) * 4096));
    CK(cudaMemset(ctx->counters, 0, sizeof(int) * 4096));
    CK(cudaMalloc(&ctx->ss, sizeof(float) * R * (m.d / 128)));
    CK(cudaMalloc(&ctx->logits, sizeof(float) * kMaxPassTokens * ctx->vocab));
    if (tp_size > 1) {
        int max_lv = 0;
        for (int r = 0; r < tp_size; ++r) max_lv = std::max(max_lv, ctx->tp_v0[r + 1] - ctx->tp_v0[r]);
        ctx->tp_lay = tp_layout(m.d, max_lv);
        CK(cudaMalloc(&ctx->tp_xbuf, ctx->tp_lay.bytes));
        CK(cudaMemset(ctx->tp_xbuf, 0, ctx->tp_lay.bytes));
        TpPeers& P = ctx->tp_peers;
        P.rank = tp_rank;
        P.size = tp_size;
        for (int r = 0; r <= tp_size; ++r) P.v0[r] = ctx->tp_v0[r];
    }

    // paged KV cache (all pages reserved up front; page table maps logical->physical)
    const size_t kv_elems = static_cast<size_t>(ctx->n_pages) * m.n_layers * 2 * m.n_kv_heads *
                            ctx->page_size * m.head_dim;
    CK(cudaMalloc(&ctx->kv_pool, sizeof(__nv_bfloat16) * (ctx->fp32acc ? 1 : kv_elems)));
    if (ctx->fp32acc) CK(cudaMalloc(&ctx->kv_f32, sizeof(float) * kv_elems));
    if (!ctx->fp32acc) {
        // finite everywhere: whole-page TMA staging reads rows past the last
        // key, which reach the PV product with P = 0
        CK(cudaMemset(ctx->kv_pool, 0, sizeof(__nv_bfloat16) * kv_elems));
        if (m.head_dim == 128 && ctx->page_size >= 16 && ctx->page_size <= 128 && 128 % ctx->page_size == 0) {
            if (make_tmap_bf16(&ctx->map_kv, ctx->kv_pool, kv_elems / 128, 128,
                               static_cast<uint32_t>(ctx->page_size)))
                return ctx_fail(ctx, DD_E_CUDA, "cuTensorMapEncodeTiled failed (KV pool)");
            ctx->has_map_kv = true;
        }
    }
    std::vector<int32_t> pt(ctx->n_pages);
    for (int i = 0; i < ctx->n_pages; ++i) pt[i] = i;
    CK(cudaMalloc(&ctx->page_table, sizeof(int32_t) * ctx->n_pages));
    CK(cudaMemcpy(ctx->page_table, pt.data(), sizeof(int32_t) * ctx->n_pages,
                  cudaMemcpyHostToDevice));

    // persistent pass kernel scratch
    {
        const char* env = getenv("DD_PASS_KERNEL");
        // the persistent pass kernel has no cross-rank reduction (tp.h): sharded
        // contexts run one launch per GEMM / attention / reduction
        // (fp32-accumulate mode: split activations run on the per-launch GEMM; a
        // partitioned device with fewer SMs than the persistent grid cannot
        // co-schedule its 148 CTAs)
        ctx->use_pass_kernel = !(env && env[0] == '0') && !ctx->fp32acc && ctx->sm_count >= kNumSMs;
        // embed + per layer (qkv, attention, o, gate/up, down) + head
        const size_t per_layer = m.qkv_rows() / 128 + m.n_heads * 16 + m.d / 128 + 2 * m.ffn / 128 + m.d / 128;
        const size_t n_flags = m.d / 128 + per_layer * m.n_layers + m.vocab / 128;
        ctx->pass_flag_count = n_flags;
        const size_t bytes = sizeof(int) * n_flags * kFlagReplicas * kFlagStride;
        CK(cudaMalloc(&ctx->pass_flags, bytes));
        CK(cudaMemset(ctx->pass_flags, 0, bytes));
        size_t half = 0;
        for (int id = 0; id < kNumGemm; ++id) half = std::max(half, pass_ws_floats(ctx, id));
        ctx->pass_ws_half = half;
        CK(cudaMalloc(&ctx->pass_ws, sizeof(float) * 2 * half));
        CK(cudaMalloc(&ctx->pass_counters, sizeof(int) * 2 * 512 * kCounterStride));
        CK(cudaMemset(ctx->pass_counters, 0, sizeof(int) * 2 * 512 * kCounterStride));
        CK(cudaMalloc(&ctx->attn_part, sizeof(float) * pass_attn_part_floats(m)));
        CK(cudaMalloc(&ctx->attn_cnt, sizeof(int) * pass_attn_cnt_ints(m)));
        CK(cudaMemset(ctx->attn_cnt, 0, sizeof(int) * pass_attn_cnt_ints(m)));
    }

    // RoPE tables in double precision -> fp32 (shared with the oracle)
    const int half = m.head_dim / 2;
    std::vector<float> cs(static_cast<size_t>(ctx->max_seq) * half), sn(cs.size());
    for (int p = 0; p < ctx->max_seq; ++p)
        for (int i = 0; i < half; ++i) {
            const double inv = std::pow(static_cast<double>(m.rope_theta),
                                        -2.0 * i / static_cast<double>(m.head_dim));
            const double ang = static_cast<double>(p) * inv;
            cs[static_cast<size_t>(p) * half + i] = static_cast<float>(std::cos(ang));
            sn[static_cast<size_t>(p) * half + i] = static_cast<float>(std::sin(ang));
        }
    CK(cudaMalloc(&ctx->rope_cos, sizeof(float) * cs.size()));
    CK(cudaMalloc(&ctx->rope_sin, sizeof(float) * sn.size()));
    CK(cudaMemcpy(ctx->rope_cos, cs.data(), sizeof(float) * cs.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->rope_sin, sn.data(), sizeof(float) * sn.size(), cudaMemcpyHostToDevice));

    // pass state ring + acceptance scratch
    CK(cudaMalloc(&ctx->d_ps, sizeof(PassState)));
    CK(cudaHostAlloc(&ctx->h_ps, sizeof(PassState) * kPsRing, cudaHostAllocDefault));
    CK(cudaMalloc(&ctx->row_m, sizeof(double) * (kMaxPassTokens + 1)));
    CK(cudaMalloc(&ctx->row_sum, sizeof(double) * (kMaxPassTokens + 1)));
    CK(cudaMalloc(&ctx->row_argmax, sizeof(int) * (kMaxPassTokens + 1)));
    CK(cudaMalloc(&ctx->ticket, sizeof(unsigned)));
    CK(cudaMemset(ctx->ticket, 0, sizeof(unsigned)));
    CK(cudaMalloc(&ctx->d_out, sizeof(dd_verify_out)));
    CK(cudaHostAlloc(&ctx->h_out, sizeof(dd_verify_out), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->h_out_dev), ctx->h_out, 0));
    std::memset(ctx->h_out, 0, sizeof(dd_verify_out));
    CK(cudaMalloc(&ctx->q_rows, sizeof(float) * kMaxPassTokens * ctx->vocab));
    CK(cudaMalloc(&ctx->d_tail, sizeof(int32_t) * kMaxPassTokens));
    CK(cudaMalloc(&ctx->d_compact_dst, sizeof(int32_t) * kMaxPassTokens));
    CK(cudaHostAlloc(&ctx->h_q_stage, sizeof(float) * kMaxPassTokens * ctx->vocab,
                     cudaHostAllocDefault));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->use_graphs = true;
    *out = ctx;
    return DD_OK;
}

void dd_ctx_destroy(dd_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : ctx->pass_phases) cudaFree(kv.second);
    for (int* b : ctx->pass_begins) cudaFree(b);
    if (ctx->attn_rank_d) cudaFree(ctx->attn_rank_d);
    for (auto& L : ctx->layers) {
        cudaFree(L.qkv);
        cudaFree(L.o);
        cudaFree(L.gu);
        cudaFree(L.dn);
    }
    for (cudaEvent_t e : {ctx->t_start, ctx->t_end, ctx->t_first})
        if (e) cudaEventDestroy(e);
    void* dev[] = {ctx->emb, ctx->head, ctx->gain_ones, ctx->x, ctx->h, ctx->q, ctx->o, ctx->a,
                   ctx->ws, ctx->logits, ctx->kv_pool, ctx->page_table, ctx->rope_cos,
                   ctx->rope_sin, ctx->d_ps, ctx->row_m, ctx->row_sum, ctx->row_argmax,
                   ctx->ticket, ctx->d_out, ctx->q_rows, ctx->d_tail, ctx->d_probs,
                   ctx->counters, ctx->ss, ctx->ws_wide, ctx->pass_flags, ctx->pass_ws, ctx->pass_counters,
                   ctx->attn_part, ctx->attn_cnt, ctx->sk_prefix_d, ctx->rank_of_smid_d,
                   ctx->h_lo, ctx->o_lo, ctx->a_lo, ctx->kv_f32, ctx->d_compact_dst};
    for (void* p : dev)
        if (p) cudaFree(p);
    for (void* p : ctx->tp_opened) cudaIpcCloseMemHandle(p);
    if (ctx->tp_xbuf) cudaFree(ctx->tp_xbuf);
    if (ctx->h_ps) cudaFreeHost(ctx->h_ps);
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    if (ctx->h_q_stage) cudaFreeHost(ctx->h_q_stage);
    for (int i = 0; i < kPsRing; ++i)
        if (ctx->ps_done[i]) cudaEventDestroy(ctx->ps_done[i]);
    if (ctx->q_ready) cudaEventDestroy(ctx->q_ready);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
}

int dd_weights_init(dd_ctx* ctx, uint64_t weight_seed, const dd_plant_desc* plant) {
    if (!ctx) return ctx_fail(nullptr, DD_E_ARG, "null ctx");
    CK(cudaSetDevice(ctx->device));
    const ModelDims& m = ctx->m;
    const float amp_proj = static_cast<float>(0.02 * std::sqrt(3.0));
    const float amp_out = static_cast<float>(0.02 / std::sqrt(2.0 * m.n_layers) * std::sqrt(3.0));
    PlantTable pt = make_plant_table(ctx->vocab, m.d, plant);
    const float amp_emb = static_cast<float>(pt.emb_std * std::sqrt(3.0));
    cudaStream_t s = ctx->stream;
    const uint64_t d_ = m.d;
    launch_init_matrix(ctx->emb, ctx->vocab, d_, derive_seed(weight_seed, kTensorEmb), amp_emb, s, 0,
                       0);  // gathered, row-major
    int32_t* d_src = nullptr;
    if (pt.any) {
        CK(cudaMalloc(&d_src, sizeof(int32_t) * ctx->vocab));
        CK(cudaMemcpyAsync(d_src, pt.src.data(), sizeof(int32_t) * ctx->vocab, cudaMemcpyHostToDevice,
                           s));
    }
    launch_init_head(ctx->head, ctx->emb, d_src, m.vocab, d_, derive_seed(weight_seed, kTensorHead),
                     amp_proj, pt.coef, s, ctx->tp_v0[ctx->tp_rank]);
    // this rank's rows (column-parallel) or columns (row-parallel) of every
    // full generated tensor, so any tp_size reproduces the same model
    const uint64_t r = ctx->tp_rank, tp = ctx->tp_size;
    for (int l = 0; l < m.n_layers; ++l) {
        LayerW& L = ctx->layers[l];
        const uint64_t qd = m.q_dim(), kvd = m.kv_dim(), f = m.ffn;
        launch_init_matrix(L.qkv, qd, d_, derive_seed(weight_seed, tensor_id(l, kWq)), amp_proj, s, 0,
                           1, SrcWindow{r * qd, 0, 0});
        launch_init_matrix(L.qkv, kvd, d_, derive_seed(weight_seed, tensor_id(l, kWk)), amp_proj, s,
                           qd, 1, SrcWindow{r * kvd, 0, 0});
        launch_init_matrix(L.qkv, kvd, d_, derive_seed(weight_seed, tensor_id(l, kWv)), amp_proj, s,
                           qd + kvd, 1, SrcWindow{r * kvd, 0, 0});
        launch_init_matrix(L.o, d_, qd, derive_seed(weight_seed, tensor_id(l, kWo)), amp_out, s, 0, 1,
                           SrcWindow{0, r * qd, qd * tp});
        launch_init_matrix_interleaved(L.gu, f, d_, derive_seed(weight_seed, tensor_id(l, kWg)),
                                       amp_proj, 0, s, r * f);
        launch_init_matrix_interleaved(L.gu, f, d_, derive_seed(weight_seed, tensor_id(l, kWu)),
                                       amp_proj, 64, s, r * f);
        launch_init_matrix(L.dn, d_, f, derive_seed(weight_seed, tensor_id(l, kWd)), amp_out, s, 0, 1,
                           SrcWindow{0, r * f, f * tp});
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    if (d_src) cudaFree(d_src);
    ctx->weights_ready = true;
    // SM-weighted stream-K partition: opt-in (measured no faster on the pool's
    // B200s: the slow SMs share a saturated resource)
    const char* bal = getenv("DD_PASS_BALANCE");
    if (ctx->use_pass_kernel && bal && bal[0] == '1') return dd_pass_balance(ctx);
    return DD_OK;
}

static void tp_set_peer(dd_ctx* ctx, int r, char* base) {
    TpPeers& P = ctx->tp_peers;
    P.flags[r] = reinterpret_cast<int*>(base + ctx->tp_lay.flags_off);
    P.part[r] = reinterpret_cast<float*>(base + ctx->tp_lay.part_off);
    P.lg[r] = reinterpret_cast<float*>(base + ctx->tp_lay.lg_off);
    P.pflags[r] = reinterpret_cast<int*>(base + ctx->tp_lay.pflag_off);
    P.pxch[r] = reinterpret_cast<float*>(base + ctx->tp_lay.pxch_off);
}

int dd_tp_export(dd_ctx* ctx, void* ipc_handle) {
    if (!ctx || !ipc_handle) return ctx_fail(ctx, DD_E_ARG, "null argument");
    if (ctx->tp_size < 2) return ctx_fail(ctx, DD_E_STATE, "context is not tensor-parallel");
    CK(cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, ctx->tp_xbuf));
    std::memcpy(ipc_handle, &h, sizeof(h));
    return DD_OK;
}

int dd_tp_connect(dd_ctx* ctx, const void* ipc_handles) {
    if (!ctx || !ipc_handles) return ctx_fail(ctx, DD_E_ARG, "null argument");
    if (ctx->tp_size < 2 || ctx->tp_connected)
        return ctx_fail(ctx, DD_E_STATE, "context is not tensor-parallel or already connected");
    static_assert(sizeof(cudaIpcMemHandle_t) == DD_TP_HANDLE_BYTES, "IPC handle size");
    CK(cudaSetDevice(ctx->device));
    const char* hb = static_cast<const char*>(ipc_handles);
    for (int r = 0; r < ctx->tp_size; ++r) {
        if (r == ctx->tp_rank) {
            tp_set_peer(ctx, r, static_cast<char*>(ctx->tp_xbuf));
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb + static_cast<size_t>(r) * DD_TP_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        ctx->tp_opened.push_back(p);
        tp_set_peer(ctx, r, static_cast<char*>(p));
    }
    ctx->tp_connected = true;
    return DD_OK;
}

int dd_tp_connect_local(dd_ctx* const* ctxs, int n) {
    if (!ctxs || n < 2 || n > kMaxTp) return ctx_fail(nullptr, DD_E_ARG, "bad rank list");
    for (int r = 0; r < n; ++r)
        if (!ctxs[r] || ctxs[r]->tp_size != n || ctxs[r]->tp_rank != r || ctxs[r]->tp_connected)
            return ctx_fail(ctxs[r], DD_E_ARG, "ctxs[r] must be unconnected rank r of an n-way split");
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            dd_ctx* ctx = ctxs[i];  // error target of CK
            const int di = ctxs[i]->device, dj = ctxs[j]->device;
            if (di == dj) continue;
            int ok = 0;
            CK(cudaDeviceCanAccessPeer(&ok, di, dj));
            if (!ok) return ctx_fail(ctxs[i], DD_E_CUDA, "no peer access between the ranks' GPUs");
            CK(cudaSetDevice(di));
            cudaError_t e = cudaDeviceEnablePeerAccess(dj, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else if (e != cudaSuccess) {
                return ctx_fail(ctxs[i], DD_E_CUDA, cudaGetErrorString(e));
            }
        }
    bool shared = true;
    for (int i = 1; i < n; ++i) shared = shared && ctxs[i]->device == ctxs[0]->device;
    for (int i = 0; i < n; ++i) {
        for (int r = 0; r < n; ++r) tp_set_peer(ctxs[i], r, static_cast<char*>(ctxs[r]->tp_xbuf));
        ctxs[i]->tp_peers.shared = shared ? 1 : 0;
        if (shared) {
            // the ranks' persistent pass kernels must be resident together
            ctxs[i]->pass_ctas = kNumSMs / n;
            for (auto& kv : ctxs[i]->pass_phases) cudaFree(kv.second);
            ctxs[i]->pass_phases.clear();
            ctxs[i]->pass_nphases.clear();
            // Every rank's kernels share one GPU: a rank's TP wait kernels (at most
            // 8 CTAs, above) spin while its peers' GEMMs run, so the tokens-on-M
            // GEMMs, whose stream-K reducers wait for segments of their own grid,
            // are planned on 16 fewer SMs; graphs captured before are dropped.
            dd_ctx* ctx = ctxs[i];
            for (int id = 0; id < kNumGemm; ++id) {
                int n_out, k;
                gemm_shape(ctx, id, &n_out, &k);
                if (ctx->wide_plans[id].tiles > 0) ctx->wide_plans[id] = plan_gemm_wide(n_out, k, kNumSMs - 16);
            }
            CK(cudaStreamSynchronize(ctx->stream));
            for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
            ctx->graphs.clear();
        }
        ctxs[i]->tp_connected = true;
    }
    return DD_OK;
}

int dd_prefill(dd_ctx* ctx, const int32_t* tokens, int n) {
    if (!ctx || (!tokens && n > 0) || n < 0) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (!ctx->weights_ready) return ctx_fail(ctx, DD_E_STATE, "weights not initialised");
    CK(cudaSetDevice(ctx->device));
    if (use_big_prefill(ctx, n)) {
        // long prompt: passes of up to kMaxPrefillTokens, equal sizes (weights
        // streamed once per pass, not once per 128-token chunk)
        const int passes = (n + kMaxPrefillTokens - 1) / kMaxPrefillTokens;
        for (int i = 0, p = 0; p < passes; ++p) {
            const int w = (n - i) / (passes - p);
            int rc = run_prefill_big(ctx, tokens + i, w);
            if (rc != DD_OK) return rc;
            i += w;
        }
        return DD_OK;
    }
    for (int i = 0; i < n; i += kPrefillChunk) {
        const int w = std::min(kPrefillChunk, n - i);
        int rc = run_pass(ctx, tokens + i, w, false);
        if (rc != DD_OK) return rc;
    }
    return DD_OK;
}

int dd_score(dd_ctx* ctx, const int32_t* tokens, int w) {
    if (!ctx || !tokens) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (!ctx->weights_ready) return ctx_fail(ctx, DD_E_STATE, "weights not initialised");
    CK(cudaSetDevice(ctx->device));
    return run_pass(ctx, tokens, w, true);
}

int dd_kv_len(const dd_ctx* ctx, int* n) {
    if (!ctx || !n) return DD_E_ARG;
    *n = ctx->n_cached;
    return DD_OK;
}

int dd_kv_truncate(dd_ctx* ctx, int n_valid) {
    if (!ctx) return ctx_fail(nullptr, DD_E_ARG, "null ctx");
    if (n_valid < 0 || n_valid > ctx->n_cached)
        return ctx_fail(ctx, DD_E_ARG, "truncate length outside [0, n_cached]");
    ctx->n_cached = n_valid;  // pages stay reserved; slots past n_valid are dead
    return DD_OK;
}

int dd_kv_compact(dd_ctx* ctx, const int32_t* src_pos, const int32_t* dst_pos, int n) {
    if (!ctx || n < 0 || (n > 0 && (!src_pos || !dst_pos)))
        return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (n > kMaxPassTokens) return ctx_fail(ctx, DD_E_CAPACITY, "at most 256 moves per compaction");
    for (int i = 0; i < n; ++i) {
        if (src_pos[i] < 0 || src_pos[i] >= ctx->n_cached || dst_pos[i] < 0 ||
            dst_pos[i] >= ctx->n_cached)
            return ctx_fail(ctx, DD_E_ARG, "compaction slot outside the cache");
        if (dst_pos[i] > src_pos[i] || (i > 0 && dst_pos[i] <= dst_pos[i - 1]))
            return ctx_fail(ctx, DD_E_ARG, "compaction needs strictly increasing dst <= src");
    }
    if (n == 0) return DD_OK;
    CK(cudaSetDevice(ctx->device));
    // moves staged through the (idle between passes) tail-token buffers
    int32_t* stage = ctx->h_ps[ctx->ps_slot].tokens;
    CK(cudaEventSynchronize(ctx->ps_done[ctx->ps_slot]));
    std::memcpy(stage, src_pos, sizeof(int32_t) * n);
    CK(cudaMemcpyAsync(ctx->d_tail, stage, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::memcpy(stage, dst_pos, sizeof(int32_t) * n);
    CK(cudaMemcpyAsync(ctx->d_compact_dst, stage, sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
    launch_kv_compact(ctx->kv_pool, ctx->kv_f32, ctx->page_table, ctx->page_size, ctx->m, ctx->d_tail,
                      ctx->d_compact_dst, n, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return DD_OK;
}

int dd_read_logits(dd_ctx* ctx, float* host, int row0, int rows) {
    if (!ctx || !host) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (ctx->last_w == 0) return ctx_fail(ctx, DD_E_STATE, "no scored pass");
    if (row0 < 0 || rows < 0 || row0 + rows > ctx->last_w)
        return ctx_fail(ctx, DD_E_ARG, "rows outside the last pass");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemcpyAsync(host, ctx->logits + static_cast<size_t>(row0) * ctx->vocab,
                       sizeof(float) * rows * ctx->vocab, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return DD_OK;
}

int dd_upload_q(dd_ctx* ctx, const float* q_rows, int rows, int vocab) {
    if (!ctx || (!q_rows && rows > 0)) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    // vocab may be below the model's for dd_verify_probs (Markov-table rows)
    if (vocab < 1 || vocab > ctx->vocab || rows < 0 || rows > kMaxPassTokens)
        return ctx_fail(ctx, DD_E_ARG, "q rows shape mismatch");
    CK(cudaSetDevice(ctx->device));
    const size_t bytes = sizeof(float) * static_cast<size_t>(rows) * vocab;
    CK(cudaStreamSynchronize(ctx->copy_stream));  // staging buffer reuse
    std::memcpy(ctx->h_q_stage, q_rows, bytes);
    CK(cudaMemcpyAsync(ctx->q_rows, ctx->h_q_stage, bytes, cudaMemcpyHostToDevice,
                       ctx->copy_stream));
    ctx->h2d_bytes += bytes;
    CK(cudaEventRecord(ctx->q_ready, ctx->copy_stream));
    ctx->q_rows_valid = rows;
    return DD_OK;
}

static int verify_common(dd_ctx* ctx, AcceptParams& p, const dd_verify_args* args,
                         dd_verify_out* out) {
    p.mode = args->mode;
    p.s = args->n_firsts;
    p.greedy = args->greedy;
    p.q_onehot = args->q_onehot;
    p.inv_temp = args->greedy ? 1.0 : 1.0 / args->temperature;
    p.seed = args->seed;
    p.counter = args->counter;
    for (int i = 0; i < 16; ++i) p.firsts[i] = i < args->n_firsts ? args->firsts[i] : -1;
    p.q = ctx->q_rows;
    p.row_m = ctx->row_m;
    p.row_sum = ctx->row_sum;
    p.row_argmax = ctx->row_argmax;
    p.ticket = ctx->ticket;
    p.out = ctx->h_out_dev;
    ctx->verify_seq = ctx->verify_seq == INT_MAX ? 1 : ctx->verify_seq + 1;
    p.seq = ctx->verify_seq;
    if (!p.q_onehot && p.mode != DD_MODE_VANILLA && p.L > 0) {
        if (ctx->q_rows_valid < p.L) return ctx_fail(ctx, DD_E_STATE, "q rows not uploaded");
        CK(cudaStreamWaitEvent(ctx->stream, ctx->q_ready, 0));
    }
    CK(launch_accept(p, ctx->stream));
    ctx->launches += 1;
    ctx->d2h_bytes += sizeof(dd_verify_out);
    // spin on the mapped result's sequence word (the kernel writes it after a
    // system fence); every 1024 polls ask the stream whether it failed
    volatile const int* seqw = &ctx->h_out->pad;
    for (unsigned spins = 1; *seqw != p.seq; ++spins) {
        if ((spins & 1023u) == 0) {
            const cudaError_t e = cudaStreamQuery(ctx->stream);
            if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
            if (e == cudaSuccess && *seqw != p.seq)
                return ctx_fail(ctx, DD_E_CUDA, "acceptance result missing after the stream drained");
        }
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    const volatile int* src = reinterpret_cast<const volatile int*>(ctx->h_out);
    int* dst = reinterpret_cast<int*>(out);
    for (size_t i = 0; i < sizeof(dd_verify_out) / sizeof(int); ++i) dst[i] = src[i];
    return DD_OK;
}

static int check_verify_args(dd_ctx* ctx, const dd_verify_args* args) {
    if (args->mode < DD_MODE_DUO || args->mode > DD_MODE_VANILLA)
        return ctx_fail(ctx, DD_E_ARG, "unknown verify mode");
    if (args->n_firsts < 0 || args->n_firsts > 16)
        return ctx_fail(ctx, DD_E_ARG, "bundle size must be in [0, 16]");
    if (!args->greedy && !(args->temperature > 0.0))
        return ctx_fail(ctx, DD_E_ARG, "temperature must be positive");
    if (args->tail_len < 0 || (args->mode == DD_MODE_VANILLA && args->tail_len != 0))
        return ctx_fail(ctx, DD_E_ARG, "bad tail length");
    for (int i = 0; i < args->n_firsts; ++i)
        if (args->firsts[i] < 0 || args->firsts[i] >= ctx->vocab)
            return ctx_fail(ctx, DD_E_ARG, "bundle token outside vocabulary");
    return DD_OK;
}

int dd_verify(dd_ctx* ctx, const dd_verify_args* args, dd_verify_out* out) {
    if (!ctx || !args || !out) return ctx_fail(ctx, DD_E_ARG, "null argument");
    int rc = check_verify_args(ctx, args);
    if (rc) return rc;
    if (ctx->last_w == 0) return ctx_fail(ctx, DD_E_STATE, "no scored pass to verify");
    const int L = args->tail_len;
    if (L + 1 > ctx->last_w) return ctx_fail(ctx, DD_E_ARG, "tail longer than the scored pass");
    CK(cudaSetDevice(ctx->device));
    AcceptParams p{};
    p.V = ctx->vocab;
    p.L = L;
    p.row0 = ctx->last_w - 1 - L;
    p.logits = ctx->logits;
    p.probs = nullptr;
    p.tail = ctx->d_ps->tokens + (ctx->last_w - L);
    return verify_common(ctx, p, args, out);
}

int dd_verify_probs(dd_ctx* ctx, const double* p_rows, const int32_t* tail_tokens, int vocab,
                    const dd_verify_args* args, dd_verify_out* out) {
    if (!ctx || !args || !out || !p_rows) return ctx_fail(ctx, DD_E_ARG, "null argument");
    int rc = check_verify_args(ctx, args);
    if (rc) return rc;
    const int L = args->tail_len;
    if (L > kMaxPassTokens - 1 || vocab < 1) return ctx_fail(ctx, DD_E_ARG, "bad shape");
    CK(cudaSetDevice(ctx->device));
    const size_t need = static_cast<size_t>(L + 1) * vocab;
    if (need > ctx->probs_cap) {
        if (ctx->d_probs) cudaFree(ctx->d_probs);
        CK(cudaMalloc(&ctx->d_probs, sizeof(double) * need));
        ctx->probs_cap = need;
    }
    CK(cudaMemcpyAsync(ctx->d_probs, p_rows, sizeof(double) * need, cudaMemcpyHostToDevice,
                       ctx->stream));
    if (L > 0)
        CK(cudaMemcpyAsync(ctx->d_tail, tail_tokens, sizeof(int32_t) * L, cudaMemcpyHostToDevice,
                           ctx->stream));
    AcceptParams p{};
    p.V = vocab;
    p.L = L;
    p.row0 = 0;
    p.logits = nullptr;
    p.probs = ctx->d_probs;
    p.tail = ctx->d_tail;
    return verify_common(ctx, p, args, out);
}

int dd_time_pass(dd_ctx* ctx, int w, int trials, float* median_ms) {
    if (!ctx || !median_ms || trials < 1) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    std::vector<int32_t> toks(w, 0);
    const int n0 = ctx->n_cached;
    std::vector<float> ms;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int t = 0; t < trials; ++t) {
        CK(cudaEventRecord(a, ctx->stream));
        int rc = run_pass(ctx, toks.data(), w, true);
        if (rc) return rc;
        CK(cudaEventRecord(b, ctx->stream));
        CK(cudaEventSynchronize(b));
        float x = 0;
        CK(cudaEventElapsedTime(&x, a, b));
        ms.push_back(x);
        ctx->n_cached = n0;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    ctx->last_w = 0;
    std::sort(ms.begin(), ms.end());
    const size_t n = ms.size();
    *median_ms = n % 2 ? ms[n / 2] : 0.5f * (ms[n / 2 - 1] + ms[n / 2]);
    return DD_OK;
}

int dd_profile_pass(dd_ctx* ctx, int w, float* ms4) {
    if (!ctx || !ms4 || w < 1 || w > kMaxPassTokens) return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (ctx->n_cached + w > ctx->max_seq) return ctx_fail(ctx, DD_E_CAPACITY, "cache full");
    CK(cudaSetDevice(ctx->device));
    const int n0 = ctx->n_cached;
    const int slot = ctx->ps_slot;
    ctx->ps_slot = (slot + 1) % kPsRing;
    CK(cudaEventSynchronize(ctx->ps_done[slot]));
    PassState* hp = ctx->h_ps + slot;
    hp->n_cached = n0;
    hp->w = w;
    hp->epoch = ++ctx->epoch;
    for (int i = 0; i < w; ++i) hp->tokens[i] = 0;
    CK(cudaMemcpyAsync(ctx->d_ps, hp, sizeof(PassState), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->ps_done[slot], ctx->stream));
    std::vector<cudaEvent_t> ev;
    std::vector<int> cls;
    auto mark = [&](int c) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, ctx->stream);
        ev.push_back(e);
        cls.push_back(c);
    };
    mark(-1);
    int rc = enqueue_pass_impl(ctx, w, true, mark);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    for (int i = 0; i < 4; ++i) ms4[i] = 0.0f;
    for (size_t i = 1; i < ev.size(); ++i) {
        float x = 0;
        cudaEventElapsedTime(&x, ev[i - 1], ev[i]);
        ms4[cls[i]] += x;
        ms4[3] += x;
    }
    for (auto e : ev) cudaEventDestroy(e);
    ctx->n_cached = n0;
    ctx->last_w = 0;
    return DD_OK;
}

// The GEMM launches of one pass (4 per layer + LM head), back to back; with
// `trace` each launch records per-CTA stamps at trace + launch * stride.
static int enqueue_gemm_sequence(dd_ctx* ctx, int w, unsigned long long* trace, size_t stride,
                                 int* n_launch) {
    const ModelDims& m = ctx->m;
    const int nt = round_nt(w);
    GemmEpiParams e{};
    e.counters = ctx->counters;
    e.ps = ctx->d_ps;
    e.rope_cos = ctx->rope_cos;
    e.rope_sin = ctx->rope_sin;
    e.q_out = ctx->q;
    e.kv_pool = ctx->kv_pool;
    e.page_table = ctx->page_table;
    e.page_size = ctx->page_size;
    e.m = m;
    e.ss_in = ctx->ss;
    e.ss_tiles = m.d / 128;
    e.eps = m.eps;
    e.norm_d = m.d;
    int n = 0;
    auto one = [&](int id, const __nv_bfloat16* W, const CUtensorMap* mx,
                   const GemmEpiParams& ep) -> cudaError_t {
        int n_out, k;
        gemm_shape(ctx, id, &n_out, &k);
        gemm_set_trace(trace ? trace + stride * n : nullptr);
        ++n;
        return launch_gemm(W, mx, n_out, k, w, nt, plan_for(ctx, id, nt), ctx->ws, ep, ctx->stream);
    };
    for (int l = 0; l < m.n_layers; ++l) {
        const LayerW& L = ctx->layers[l];
        GemmEpiParams eq = e;
        eq.kind = kEpiQkvRope;
        eq.layer = l;
        CK(one(kGQkv, L.qkv, &ctx->map_h, eq));
        GemmEpiParams er = e;
        er.kind = kEpiResidual;
        er.out = ctx->x;
        er.ss_in = nullptr;
        er.u_out = ctx->h;
        er.gain = ctx->gain_ones;
        er.ss_out = ctx->ss;
        CK(one(kGO, L.o, &ctx->map_o, er));
        GemmEpiParams eg = e;
        eg.kind = kEpiSwiGLU;
        eg.out_bf = ctx->a;
        CK(one(kGGu, L.gu, &ctx->map_h, eg));
        CK(one(kGDown, L.dn, &ctx->map_a, er));
    }
    GemmEpiParams el = e;
    el.kind = kEpiStore;
    el.out = ctx->logits;
    CK(one(kGHead, ctx->head, &ctx->map_h, el));
    gemm_set_trace(nullptr);
    if (n_launch) *n_launch = n;
    return DD_OK;
}

static int upload_dummy_pass(dd_ctx* ctx, int w) {
    const int slot = ctx->ps_slot;
    ctx->ps_slot = (slot + 1) % kPsRing;
    CK(cudaEventSynchronize(ctx->ps_done[slot]));
    PassState* hp = ctx->h_ps + slot;
    hp->n_cached = ctx->n_cached;
    hp->w = w;
    hp->epoch = ++ctx->epoch;
    for (int i = 0; i < w; ++i) hp->tokens[i] = 0;
    CK(cudaMemcpyAsync(ctx->d_ps, hp, sizeof(PassState), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->ps_done[slot], ctx->stream));
    return DD_OK;
}

int dd_debug_pass_trace(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_launch,
                        int* ctas_per_launch) {
    if (!ctx || !trace || w < 1 || w > kMaxPassTokens) return ctx_fail(ctx, DD_E_ARG, "bad args");
    CK(cudaSetDevice(ctx->device));
    int rc = upload_dummy_pass(ctx, w);
    if (rc) return rc;
    int maxc = 0;
    for (int id = 0; id < kNumGemm; ++id) maxc = std::max(maxc, plan_for(ctx, id, round_nt(w)).ctas);
    const size_t stride = 8 * static_cast<size_t>(maxc);
    const size_t need = stride * (4 * ctx->m.n_layers + 1);
    if (need > max_entries) return ctx_fail(ctx, DD_E_CAPACITY, "trace buffer too small");
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long) * need));
    CK(cudaMemset(d, 0, sizeof(unsigned long long) * need));
    rc = enqueue_gemm_sequence(ctx, w, nullptr, 0, nullptr);  // warm-up
    if (rc) return rc;
    rc = enqueue_gemm_sequence(ctx, w, d, stride, n_launch);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(trace, d, sizeof(unsigned long long) * need, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *ctas_per_launch = maxc;
    ctx->last_w = 0;
    return DD_OK;
}

int dd_time_gemms(dd_ctx* ctx, int w, int trials, float* median_ms, int* launches) {
    if (!ctx || !median_ms || w < 1 || w > kMaxPassTokens || trials < 1)
        return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    if (ctx->n_cached + w > ctx->max_seq) return ctx_fail(ctx, DD_E_CAPACITY, "cache full");
    CK(cudaSetDevice(ctx->device));
    int rc = upload_dummy_pass(ctx, w);
    if (rc) return rc;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ms;
    int n_launch = 0;
    for (int t = 0; t < trials + 1; ++t) {
        CK(cudaEventRecord(a, ctx->stream));
        rc = enqueue_gemm_sequence(ctx, w, nullptr, 0, &n_launch);
        if (rc) return rc;
        CK(cudaEventRecord(b, ctx->stream));
        CK(cudaEventSynchronize(b));
        float x = 0.0f;
        CK(cudaEventElapsedTime(&x, a, b));
        if (t > 0) ms.push_back(x);  // first run warms up
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(ms.begin(), ms.end());
    const size_t n = ms.size();
    *median_ms = n % 2 ? ms[n / 2] : 0.5f * (ms[n / 2 - 1] + ms[n / 2]);
    if (launches) *launches = n_launch;
    ctx->last_w = 0;
    return DD_OK;
}

uint64_t dd_pass_weight_bytes(const dd_ctx* ctx) {
    if (!ctx) return 0;
    const ModelDims& m = ctx->m;
    const uint64_t per_layer = static_cast<uint64_t>(m.qkv_rows()) * m.d +
                               static_cast<uint64_t>(m.d) * m.q_dim() +
                               2ull * m.ffn * m.d + static_cast<uint64_t>(m.d) * m.ffn;
    return 2ull * (per_layer * m.n_layers + static_cast<uint64_t>(m.vocab) * m.d);
}

int dd_read_weights(dd_ctx* ctx, int which, int layer, uint16_t* host, size_t n) {
    if (!ctx || !host) return ctx_fail(ctx, DD_E_ARG, "null argument");
    const ModelDims& m = ctx->m;
    if (which >= 2 && (layer < 0 || layer >= m.n_layers))
        return ctx_fail(ctx, DD_E_ARG, "layer out of range");
    const void* src = nullptr;
    size_t count = 0;
    const size_t d_ = m.d;
    switch (which) {
        case 0: src = ctx->emb; count = static_cast<size_t>(ctx->vocab) * d_; break;
        case 1: src = ctx->head; count = static_cast<size_t>(m.vocab) * d_; break;
        case 2: src = ctx->layers[layer].qkv; count = static_cast<size_t>(m.qkv_rows()) * d_; break;
        case 3: src = ctx->layers[layer].o; count = d_ * m.q_dim(); break;
        case 4: src = ctx->layers[layer].gu; count = 2 * static_cast<size_t>(m.ffn) * d_; break;
        case 5: src = ctx->layers[layer].dn; count = d_ * m.ffn; break;
        default: return ctx_fail(ctx, DD_E_ARG, "unknown tensor");
    }
    if (n != count) return ctx_fail(ctx, DD_E_ARG, "element count mismatch");
    CK(cudaSetDevice(ctx->device));
    if (which == 0) {  // embedding: plain row-major
        CK(cudaMemcpy(host, src, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost));
        return DD_OK;
    }
    // GEMM operands are stored pre-tiled (common.cuh tiled_offset); the fused
    // gate/up matrix is also interleaved in 64-row blocks.  Return logical layout.
    std::vector<uint16_t> tmp(n);
    CK(cudaMemcpy(tmp.data(), src, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost));
    const size_t cols = (which == 3) ? static_cast<size_t>(m.q_dim())
                        : (which == 5) ? static_cast<size_t>(m.ffn) : d_;
    const size_t rows = n / cols;
    for (size_t pr = 0; pr < rows; ++pr) {
        size_t lr = pr;
        if (which == 4) {
            const size_t blk = pr / 128, off = pr % 128;
            lr = off < 64 ? blk * 64 + off : m.ffn + blk * 64 + (off - 64);
        }
        for (size_t c = 0; c < cols; ++c) host[lr * cols + c] = tmp[tiled_offset(pr, c, cols)];
    }
    return DD_OK;
}

int dd_debug_gemm_trace(dd_ctx* ctx, int which, int w, uint64_t* trace, int max_ctas,
                        int* n_ctas) {
    // one launch of GEMM `which` (0 qkv, 1 o, 2 gate/up, 3 down, 4 head) of layer 0
    if (!ctx || !trace || !n_ctas || w < 1 || w > kMaxPassTokens || which < 0 || which > 4)
        return ctx_fail(ctx, DD_E_ARG, "bad arguments");
    CK(cudaSetDevice(ctx->device));
    const int nt = round_nt(w);
    const GemmPlan& p = plan_for(ctx, which, nt);
    const int ctas = p.ctas;
    if (ctas > max_ctas) return ctx_fail(ctx, DD_E_CAPACITY, "trace buffer too small");
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long) * 8 * ctas));
    CK(cudaMemset(d, 0, sizeof(unsigned long long) * 8 * ctas));
    int n_out, k;
    gemm_shape(ctx, which, &n_out, &k);
    const LayerW& L = ctx->layers[0];
    const __nv_bfloat16* W = which == 0 ? L.qkv : which == 1 ? L.o : which == 2 ? L.gu
                             : which == 3 ? L.dn : ctx->head;
    const CUtensorMap* mx = which == 1 ? &ctx->map_o : which == 3 ? &ctx->map_a : &ctx->map_h;
    GemmEpiParams e{};
    e.kind = kEpiStore;
    e.counters = ctx->counters;
    e.out = ctx->ws;  // scratch destination
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
        gemm_set_trace(rep ? d : nullptr);
        CK(launch_gemm(W, mx, n_out, k, w, nt, p, ctx->ws, e, ctx->stream));
    }
    gemm_set_trace(nullptr);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(trace, d, sizeof(unsigned long long) * 8 * ctas, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *n_ctas = ctas;
    return DD_OK;
}

void* dd_debug_pass_progress(void) { return pass_debug_enable(1); }

// one prefill-width pass (17..128 tokens, per-launch path) with per-CTA stamps of
// its wide GEMM launches: trace[launch][cta][8]
int dd_debug_prefill_trace(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_launch) {
    if (!ctx || !trace || !n_launch || w <= 48 || w > 128) return ctx_fail(ctx, DD_E_ARG, "bad args");
    CK(cudaSetDevice(ctx->device));
    const size_t need = static_cast<size_t>(4 * ctx->m.n_layers + 1) * 8 * kNumSMs;
    if (need > max_entries) return ctx_fail(ctx, DD_E_CAPACITY, "trace buffer too small");
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long) * need));
    CK(cudaMemset(d, 0, sizeof(unsigned long long) * need));
    int rc = upload_dummy_pass(ctx, w);
    if (rc) return rc;
    rc = enqueue_pass_impl(ctx, w, true, [](int) {});  // warm-up
    if (rc) return rc;
    rc = upload_dummy_pass(ctx, w);
    if (rc) return rc;
    gemm_wide_set_trace(d);
    rc = enqueue_pass_impl(ctx, w, true, [](int) {});
    gemm_wide_set_trace(nullptr);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(trace, d, sizeof(unsigned long long) * need, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *n_launch = 4 * ctx->m.n_layers + 1;
    ctx->last_w = 0;
    return DD_OK;
}

// one pass of width w (logits on) with per-CTA, per-phase globaltimer stamps:
// trace[cta][phase][8] = weight producer start, inputs ready, MMA done,
// epilogue done, flags polled, acquire fence done, last flag published
// (0 where a role had no work)
int dd_debug_pass_timeline(dd_ctx* ctx, int w, uint64_t* trace, size_t max_entries, int* n_phases) {
    if (!ctx || !trace || !n_phases || w < 1 || w > kMaxPassTokens) return ctx_fail(ctx, DD_E_ARG, "bad args");
    CK(cudaSetDevice(ctx->device));
    const PassPhase* ph = nullptr;
    int n = 0;
    int rc = build_pass_phases(ctx, w, true, &ph, &n);
    if (rc) return rc;
    const size_t need = static_cast<size_t>(kNumSMs) * n * 12;
    if (need > max_entries) return ctx_fail(ctx, DD_E_CAPACITY, "trace buffer too small");
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long) * need));
    CK(cudaMemset(d, 0, sizeof(unsigned long long) * need));
    for (int rep = 0; rep < 2; ++rep) {
        rc = upload_dummy_pass(ctx, w);
        if (rc) return rc;
        rc = enqueue_pass_kernel(ctx, w, true, rep ? d : nullptr);
        if (rc) return rc;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(trace, d, sizeof(unsigned long long) * need, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *n_phases = n;
    ctx->last_w = 0;
    return DD_OK;
}

// Weighted stream-K partition for the persistent pass kernel: time every SM's
// streaming of the gate/up phases (the largest) over a few decode passes and
// give each SM a share proportional to its speed.  Runs once,
// before any pass graph is captured; the phase tables are rebuilt afterwards.
int dd_pass_balance(dd_ctx* ctx) {
    if (!ctx || !ctx->weights_ready) return ctx_fail(ctx, DD_E_STATE, "weights not initialised");
    CK(cudaSetDevice(ctx->device));
    const int w = 8;
    const int L = ctx->m.n_layers;
    const int nph_exp = 5 * L + 2;
    const size_t need = static_cast<size_t>(kNumSMs) * nph_exp * 12;
    std::vector<uint64_t> tr(need);
    std::vector<double> span(1024, 0.0);
    std::vector<int> seen(1024, 0);
    const int n0 = ctx->n_cached;
    for (int rep = 0; rep < 3; ++rep) {
        int nph = 0;
        int rc = dd_debug_pass_timeline(ctx, w, tr.data(), need, &nph);
        if (rc) return rc;
        if (rep == 0) continue;  // warm-up
        for (int b = 0; b < kNumSMs; ++b) {
            const int smid = static_cast<int>(tr[(static_cast<size_t>(b) * nph + 0) * 12 + 10]);
            if (smid < 0 || smid >= 1024) continue;
            for (int l = 1; l + 1 < L || (L <= 2 && l < L); ++l) {
                const size_t base = (static_cast<size_t>(b) * nph + 1 + 5 * l + 3) * 12;
                if (tr[base + 1] == 0 || tr[base + 2] <= tr[base + 1]) continue;
                span[smid] += static_cast<double>(tr[base + 2] - tr[base + 1]);
                seen[smid] += 1;
            }
        }
    }
    ctx->n_cached = n0;
    std::vector<int> smids;
    double mean = 0.0;
    for (int i = 0; i < 1024; ++i)
        if (seen[i]) {
            smids.push_back(i);
            span[i] /= seen[i];
            mean += span[i];
        }
    if (static_cast<int>(smids.size()) != kNumSMs) return DD_OK;  // keep the uniform partition
    mean /= smids.size();
    std::vector<int> rank_of(1024, 0), prefix(kNumSMs + 1, 0);
    for (int r = 0; r < kNumSMs; ++r) {
        const int sm = smids[r];
        rank_of[sm] = r;
        const int wgt = std::max(40, std::min(96, static_cast<int>(std::lround(64.0 * mean / span[sm]))));
        prefix[r + 1] = prefix[r] + wgt;
    }
    if (!ctx->sk_prefix_d) {
        CK(cudaMalloc(&ctx->sk_prefix_d, sizeof(int) * (kNumSMs + 1)));
        CK(cudaMalloc(&ctx->rank_of_smid_d, sizeof(int) * 1024));
    }
    CK(cudaMemcpy(ctx->sk_prefix_d, prefix.data(), sizeof(int) * prefix.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->rank_of_smid_d, rank_of.data(), sizeof(int) * rank_of.size(), cudaMemcpyHostToDevice));
    ctx->sk_prefix_h = prefix;
    // phase tables and partial buffers depend on the partition: rebuild
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second);
    ctx->graphs.clear();
    for (auto& kv : ctx->pass_phases) cudaFree(kv.second);
    ctx->pass_phases.clear();
    for (int* b : ctx->pass_begins) cudaFree(b);
    ctx->pass_begins.clear();
    ctx->attn_rank_ctas = 0;
    ctx->pass_nphases.clear();
    size_t half = 0;
    for (int id = 0; id < kNumGemm; ++id) half = std::max(half, pass_ws_floats(ctx, id));
    if (half > ctx->pass_ws_half) {
        cudaFree(ctx->pass_ws);
        ctx->pass_ws_half = half;
        CK(cudaMalloc(&ctx->pass_ws, sizeof(float) * 2 * half));
    }
    return DD_OK;
}

int dd_test_gemm(const uint16_t* W, const uint16_t* X, int n_out, int k, int w, float* Y) {
    dd_ctx* ctx = nullptr;
    if (!W || !X || !Y || n_out % 128 || k % 64 || w < 1 || w > kMaxPassTokens)
        return ctx_fail(nullptr, DD_E_ARG, "bad gemm shape");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
        return ctx_fail(nullptr, DD_E_CUDA, "no CUDA device available");
    const int nt = round_nt(w);
    void *dW = nullptr, *dX = nullptr;
    float* dws = nullptr;
    float* dY = nullptr;
    CK(cudaMalloc(&dW, sizeof(uint16_t) * n_out * static_cast<size_t>(k)));
    CK(cudaMalloc(&dX, sizeof(uint16_t) * kMaxPassTokens * static_cast<size_t>(k)));
    CK(cudaMemset(dX, 0, sizeof(uint16_t) * kMaxPassTokens * static_cast<size_t>(k)));
    {
        std::vector<uint16_t> tiled(static_cast<size_t>(n_out) * k);
        for (size_t r = 0; r < static_cast<size_t>(n_out); ++r)
            for (size_t c = 0; c < static_cast<size_t>(k); ++c)
                tiled[tiled_offset(r, c, k)] = W[r * k + c];
        CK(cudaMemcpy(dW, tiled.data(), sizeof(uint16_t) * tiled.size(), cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(dX, X, sizeof(uint16_t) * w * static_cast<size_t>(k), cudaMemcpyHostToDevice));
    CUtensorMap mx;
    if (make_tmap_bf16(&mx, dX, kMaxPassTokens, k, 16))
        return ctx_fail(nullptr, DD_E_CUDA, "cuTensorMapEncodeTiled failed");
    GemmPlan p = plan_gemm(n_out, k, nt);
    CK(cudaMalloc(&dws, sizeof(float) * gemm_ws_floats(p, w)));
    CK(cudaMalloc(&dY, sizeof(float) * static_cast<size_t>(w) * n_out));
    int* dcnt = nullptr;
    CK(cudaMalloc(&dcnt, sizeof(int) * p.tiles));
    CK(cudaMemset(dcnt, 0, sizeof(int) * p.tiles));
    GemmEpiParams ep{};
    ep.kind = kEpiStore;
    ep.counters = dcnt;
    ep.out = dY;
    CK(launch_gemm(static_cast<const __nv_bfloat16*>(dW), &mx, n_out, k, w, nt, p, dws, ep, 0));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(Y, dY, sizeof(float) * static_cast<size_t>(w) * n_out, cudaMemcpyDeviceToHost));
    cudaFree(dW);
    cudaFree(dX);
    cudaFree(dws);
    cudaFree(dY);
    cudaFree(dcnt);
    return DD_OK;
}

}  // extern "C"
