/*
 * oracle/llama_ref.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the target forward contract that the reference leaves
 * abstract: ModelSpec::forward / forward_scored (reference
 * proj/include/duodec/model.hpp:57-65, proj/src/model.cpp:286-320) and
 * scored_with_next (proj/src/engine.cpp:36-43): row i of a pass is the
 * next-token distribution after tokens[0..i].  The reference's model is a
 * Markov table; the north star replaces it by a Llama-2-shape transformer with
 * seeded random-init weights, so this file is the logit-level oracle.  Its
 * Llama math is cross-checked against transformers' LlamaForCausalLM
 * (tests/test_oracle_llama.py); PARITY NOTE: the forward itself has no
 * reference arithmetic to pin against.
 *
 * Numerics mirror the GPU pass (paper_2503_00784_b200/csrc/model.cu): fp32
 * residual stream, bf16 rounding of every GEMM input (h, o, a) and of cached
 * K/V, fp32 accumulation, q kept fp32, RoPE from a double-precision table.
 * Only tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() load it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>

/* ------------------------------------------------------------ threads */
typedef void (*range_fn)(void* arg, int64_t lo, int64_t hi);
typedef struct {
    range_fn fn;
    void* arg;
    int64_t lo, hi;
} par_job;
static int g_threads = 1;
/* per calling thread: the model being run sets its own thread count, so a
 * target and a draft can run concurrently from two host threads (the
 * threaded duo loop of oracle/cpu_engine.py) */
static __thread int tl_threads = 0;
static void* par_entry(void* p) {
    par_job* j = (par_job*)p;
    j->fn(j->arg, j->lo, j->hi);
    return NULL;
}
/* static partition of [0, n) over g_threads pthreads */
static void par_range(int64_t n, range_fn fn, void* arg) {
    int nt = tl_threads > 0 ? tl_threads : g_threads;
    if (nt > n) nt = (int)n;
    if (nt <= 1) {
        fn(arg, 0, n);
        return;
    }
    pthread_t th[256];
    par_job jobs[256];
    for (int i = 0; i < nt; ++i) {
        jobs[i].fn = fn;
        jobs[i].arg = arg;
        jobs[i].lo = n * i / nt;
        jobs[i].hi = n * (i + 1) / nt;
        if (i > 0) pthread_create(&th[i], NULL, par_entry, &jobs[i]);
    }
    par_entry(&jobs[0]);
    for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------ generator */
static inline uint64_t mix(uint64_t seed, uint64_t m) { /* random.hpp:16-21 */
    uint64_t z = seed + m * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t derive(uint64_t base, uint64_t index) { /* random.hpp:38-43 */
    uint64_t z = base + (index + 1) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 30)) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline float unit(uint64_t seed, uint64_t e) {
    const uint64_t x = mix(seed, e + 1);
    return (float)(int32_t)(x >> 40) * 0x1.0p-23f - 1.0f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even (finite inputs) */
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static inline float bf2f(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static inline float bfr(float f) { return bf2f(f2bf(f)); }

enum { T_WQ = 0, T_WK = 1, T_WV = 2, T_WO = 3, T_WG = 4, T_WU = 5, T_WD = 6 };
static uint64_t tensor_id(int layer, int kind) { return 2 + (uint64_t)layer * 8 + (uint64_t)kind; }

typedef struct {
    uint16_t* dst;
    uint64_t seed;
    float amp;
} gen_arg;
static void gen_range(void* p, int64_t lo, int64_t hi) {
    gen_arg* a = (gen_arg*)p;
    for (int64_t e = lo; e < hi; ++e) a->dst[e] = f2bf(unit(a->seed, (uint64_t)e) * a->amp);
}
static void gen_matrix(uint16_t* dst, uint64_t n, uint64_t seed, float amp) {
    gen_arg a = {dst, seed, amp};
    par_range((int64_t)n, gen_range, &a);
}

/* plant table: identical recipe to paper_2503_00784_b200/csrc/plant.cpp */
static int make_plant(int vocab, int d, uint64_t plant_seed, double alpha, float gain,
                      float emb_std, int32_t* src, float* coef) {
    int any = 0;
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * vocab);
    for (int i = 0; i < vocab; ++i) {
        perm[i] = i;
        src[i] = -1;
    }
    *coef = 0.0f;
    if (alpha > 0.0) {
        uint64_t counter = 0;
        for (int i = vocab - 1; i >= 1; --i) {
            const uint64_t j = mix(plant_seed, ++counter) % (uint64_t)(i + 1);
            const int32_t t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
        const uint64_t sel = derive(plant_seed, 1);
        for (int tok = 0; tok < vocab; ++tok) {
            const double u = (double)(mix(sel, (uint64_t)tok + 1) >> 11) * 0x1.0p-53;
            if (u < alpha) {
                src[perm[tok]] = tok;
                any = 1;
            }
        }
        *coef = (float)((double)gain / ((double)emb_std * sqrt((double)d)));
    }
    free(perm);
    return any;
}

/* ------------------------------------------------------------ model */
typedef struct {
    int rows, cols;
    int8_t* q;      /* [rows][cols] */
    float* scale;   /* [rows] */
} orc_qmat;

typedef struct {
    uint16_t *qkv, *o, *gu, *dn;
    orc_qmat qqkv, qo, qgu, qdn; /* W8A8 draft mode */
} orc_layer;

typedef struct orc_llama {
    int L, d, H, Hkv, hd, F, V, max_seq, n_cached, n_threads;
    float eps, theta;
    uint16_t *emb, *head;
    orc_layer* layers;
    uint16_t* kv; /* [L][2][Hkv][max_seq][hd] */
    float *rope_cos, *rope_sin;
    int32_t* plant_src;
    int32_t* plant_perm;
    int quant;      /* 1: W8A8 matmuls (the product CPU draft's numerics) */
    int p_bf16;     /* 1: softmax weights rounded to bf16 before P.V (diagnostic) */
    int fp32;       /* 1: fp32 activations and KV cache (the GPU's fp32acc mode) */
    float* kvf;     /* fp32 KV cache of fp32 mode, same indexing as kv */
    orc_qmat qhead;
} orc_llama;

static size_t kv_idx(const orc_llama* m, int layer, int kv, int h, int pos) {
    return ((((size_t)layer * 2 + kv) * m->Hkv + h) * m->max_seq + pos) * m->hd;
}

typedef struct {
    orc_llama* m;
    uint64_t seed;
    float amp, coef;
    int any;
} head_arg;
static void head_range(void* p, int64_t lo, int64_t hi) {
    head_arg* a = (head_arg*)p;
    const int d = a->m->d;
    for (int64_t e = lo; e < hi; ++e) {
        float w = unit(a->seed, (uint64_t)e) * a->amp;
        const int64_t v = e / d, i = e % d;
        const int32_t t = a->any ? a->m->plant_src[v] : -1;
        if (t >= 0) w = fmaf(a->coef, bf2f(a->m->emb[(size_t)t * d + i]), w);
        a->m->head[e] = f2bf(w);
    }
}

orc_llama* orc_llama_create(int n_layers, int d, int n_heads, int n_kv_heads, int head_dim,
                            int ffn, int vocab, float eps, float theta, int max_seq,
                            uint64_t weight_seed, uint64_t plant_seed, double alpha, float gain,
                            float emb_std, int n_threads) {
    orc_llama* m = (orc_llama*)calloc(1, sizeof(orc_llama));
    m->L = n_layers;
    m->d = d;
    m->H = n_heads;
    m->Hkv = n_kv_heads > 0 ? n_kv_heads : n_heads;
    m->hd = head_dim;
    m->F = ffn;
    m->V = vocab;
    m->eps = eps;
    m->theta = theta;
    m->max_seq = max_seq;
    m->n_threads = n_threads;
    g_threads = n_threads > 0 ? (n_threads > 256 ? 256 : n_threads) : 1;
    if (!(emb_std > 0.0f)) emb_std = 0.02f;
    const int qd = m->H * m->hd, kvd = m->Hkv * m->hd;
    const float amp_proj = (float)(0.02 * sqrt(3.0));
    const float amp_out = (float)(0.02 / sqrt(2.0 * n_layers) * sqrt(3.0));
    const float amp_emb = (float)(emb_std * sqrt(3.0));
    m->emb = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)vocab * d);
    m->head = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)vocab * d);
    gen_matrix(m->emb, (uint64_t)vocab * d, derive(weight_seed, 0), amp_emb);
    m->plant_src = (int32_t*)malloc(sizeof(int32_t) * vocab);
    float coef = 0.0f;
    const int any = make_plant(vocab, d, plant_seed, alpha, gain, emb_std, m->plant_src, &coef);
    {
        head_arg ha = {m, derive(weight_seed, 1), amp_proj, coef, any};
        par_range((int64_t)vocab * d, head_range, &ha);
    }
    m->layers = (orc_layer*)calloc(n_layers, sizeof(orc_layer));
    for (int l = 0; l < n_layers; ++l) {
        orc_layer* Ly = &m->layers[l];
        Ly->qkv = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(qd + 2 * kvd) * d);
        Ly->o = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)d * qd);
        Ly->gu = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)2 * ffn * d);
        Ly->dn = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)d * ffn);
        gen_matrix(Ly->qkv, (uint64_t)qd * d, derive(weight_seed, tensor_id(l, T_WQ)), amp_proj);
        gen_matrix(Ly->qkv + (size_t)qd * d, (uint64_t)kvd * d,
                   derive(weight_seed, tensor_id(l, T_WK)), amp_proj);
        gen_matrix(Ly->qkv + (size_t)(qd + kvd) * d, (uint64_t)kvd * d,
                   derive(weight_seed, tensor_id(l, T_WV)), amp_proj);
        gen_matrix(Ly->o, (uint64_t)d * qd, derive(weight_seed, tensor_id(l, T_WO)), amp_out);
        gen_matrix(Ly->gu, (uint64_t)ffn * d, derive(weight_seed, tensor_id(l, T_WG)), amp_proj);
        gen_matrix(Ly->gu + (size_t)ffn * d, (uint64_t)ffn * d,
                   derive(weight_seed, tensor_id(l, T_WU)), amp_proj);
        gen_matrix(Ly->dn, (uint64_t)d * ffn, derive(weight_seed, tensor_id(l, T_WD)), amp_out);
    }
    m->kv = (uint16_t*)calloc((size_t)n_layers * 2 * m->Hkv * max_seq * head_dim, sizeof(uint16_t));
    const int half = head_dim / 2;
    m->rope_cos = (float*)malloc(sizeof(float) * (size_t)max_seq * half);
    m->rope_sin = (float*)malloc(sizeof(float) * (size_t)max_seq * half);
    for (int p = 0; p < max_seq; ++p)
        for (int i = 0; i < half; ++i) {
            const double inv = pow((double)theta, -2.0 * i / (double)head_dim);
            const double ang = (double)p * inv;
            m->rope_cos[(size_t)p * half + i] = (float)cos(ang);
            m->rope_sin[(size_t)p * half + i] = (float)sin(ang);
        }
    return m;
}

void orc_llama_free(orc_llama* m) {
    if (!m) return;
    for (int l = 0; l < m->L; ++l) {
        free(m->layers[l].qkv);
        free(m->layers[l].o);
        free(m->layers[l].gu);
        free(m->layers[l].dn);
    }
    free(m->layers);
    free(m->emb);
    free(m->head);
    free(m->kv);
    free(m->kvf);
    free(m->rope_cos);
    free(m->rope_sin);
    free(m->plant_src);
    free(m);
}

/* Per-row symmetric int8 weights (scale = max|w|/127, round-half-even) and
 * per-token int8 activations: restates the product CPU draft
 * (paper_2503_00784_b200/csrc/draft.cpp quantize / quantize_acts / qdot_rows);
 * the integer dot products are exact, so logits match bit-for-bit up to the
 * float epilogue order. */
static orc_qmat quantize_rows_levels(const uint16_t* w, int rows, int cols, int levels) {
    orc_qmat m;
    m.rows = rows;
    m.cols = cols;
    m.q = (int8_t*)malloc((size_t)rows * cols);
    m.scale = (float*)malloc(sizeof(float) * rows);
    for (int r = 0; r < rows; ++r) {
        const uint16_t* src = w + (size_t)r * cols;
        float mx = 0.0f;
        for (int c = 0; c < cols; ++c) {
            const float a = fabsf(bf2f(src[c]));
            if (a > mx) mx = a;
        }
        const float sc = mx > 0.0f ? mx / (float)levels : 1.0f;
        for (int c = 0; c < cols; ++c) {
            int v = (int)nearbyintf(bf2f(src[c]) / sc);
            v = v < -levels ? -levels : (v > levels ? levels : v);
            m.q[(size_t)r * cols + c] = (int8_t)v;
        }
        m.scale[r] = sc;
    }
    return m;
}
static orc_qmat quantize_rows(const uint16_t* w, int rows, int cols) {
    return quantize_rows_levels(w, rows, cols, 127);
}

void orc_llama_set_pbf16(orc_llama* m, int on) { m->p_bf16 = on; }

/* dd_kv_compact restated: move cache slots src[i] -> dst[i] for every layer,
 * K and V, kv head, in list order (the caller truncates afterwards). */
void orc_llama_kv_compact(orc_llama* m, const int32_t* src, const int32_t* dst, int n) {
    for (int k = 0; k < n; ++k)
        for (int l = 0; l < m->L; ++l)
            for (int kv = 0; kv < 2; ++kv)
                for (int h = 0; h < m->Hkv; ++h) {
                    const size_t a = kv_idx(m, l, kv, h, src[k]), b = kv_idx(m, l, kv, h, dst[k]);
                    for (int i = 0; i < m->hd; ++i) {
                        m->kv[b + i] = m->kv[a + i];
                        if (m->kvf) m->kvf[b + i] = m->kvf[a + i];
                    }
                }
}

/* fp32 mode (the GPU's DD_PREC_FP32ACC): activations are not rounded to bf16
 * anywhere (GEMM inputs h / o / a, the QK^T query) and the KV cache is fp32;
 * weights stay the generated bf16 values.  Set before the first forward. */
int orc_llama_set_fp32(orc_llama* m, int on) {
    if (m->n_cached != 0) return -1;
    m->fp32 = on;
    if (on && !m->kvf)
        m->kvf = (float*)calloc((size_t)m->L * 2 * m->Hkv * m->max_seq * m->hd, sizeof(float));
    return 0;
}

static inline float act(const orc_llama* m, float v) { return m->fp32 ? v : bfr(v); }
static inline float kv_get(const orc_llama* m, size_t i) { return m->fp32 ? m->kvf[i] : bf2f(m->kv[i]); }
static inline void kv_put(orc_llama* m, size_t i, float v) {
    if (m->fp32) m->kvf[i] = v;
    else m->kv[i] = f2bf(v);
}

void orc_llama_set_quant(orc_llama* m, int on) {
    if (!on || m->quant) return;
    const int qd = m->H * m->hd, kvd = m->Hkv * m->hd;
    for (int l = 0; l < m->L; ++l) {
        orc_layer* Ly = &m->layers[l];
        const char* ab = getenv("DD_DRAFT_ATTN_BITS");
        const int a4 = ab && atoi(ab) == 4 && m->d % 128 == 0 && qd % 128 == 0;
        Ly->qqkv = quantize_rows_levels(Ly->qkv, qd + 2 * kvd, m->d, a4 ? 7 : 127);
        Ly->qo = quantize_rows_levels(Ly->o, m->d, qd, a4 ? 7 : 127);
        /* the draft's gate/up and down are 4-bit (draft.cpp) unless DD_DRAFT_FFN_BITS=8 */
        const char* fb = getenv("DD_DRAFT_FFN_BITS");
        const int f4 = !(fb && atoi(fb) == 8) && m->d % 128 == 0 && m->F % 128 == 0;
        Ly->qgu = quantize_rows_levels(Ly->gu, 2 * m->F, m->d, f4 ? 7 : 127);
        Ly->qdn = quantize_rows_levels(Ly->dn, m->d, m->F, f4 ? 7 : 127);
    }
    /* the draft's LM head is 4-bit (draft.cpp quantize4) when d is a multiple of 128 */
    const char* hb = getenv("DD_DRAFT_HEAD_BITS");
    const int w4 = m->d % 128 == 0 && !(hb && atoi(hb) == 8);
    m->qhead = quantize_rows_levels(m->head, m->V, m->d, w4 ? 7 : 127);
    m->quant = 1;
}

typedef struct {
    const orc_qmat* m;
    const int8_t* xq;
    const float* xs;
    int w;
    float* y;
} qmm_arg;
static void qmm_range(void* p, int64_t lo, int64_t hi) {
    qmm_arg* a = (qmm_arg*)p;
    const int k = a->m->cols;
    for (int64_t n = lo; n < hi; ++n)
        for (int t = 0; t < a->w; ++t) {
            int64_t dot = 0;
            const int8_t* wq = a->m->q + (size_t)n * k;
            const int8_t* xq = a->xq + (size_t)t * k;
            for (int i = 0; i < k; ++i) dot += (int64_t)wq[i] * xq[i];
            a->y[(size_t)t * a->m->rows + n] = (float)(int32_t)dot * (a->xs[t] * a->m->scale[n]);
        }
}
/* x: [w][k] float values that are exactly bf16 */
static void matmul_q(const orc_qmat* m, const float* x, int w, float* y) {
    const int k = m->cols;
    int8_t* xq = (int8_t*)malloc((size_t)w * k);
    float* xs = (float*)malloc(sizeof(float) * w);
    for (int t = 0; t < w; ++t) {
        float mx = 0.0f;
        for (int i = 0; i < k; ++i) {
            const float a = fabsf(x[(size_t)t * k + i]);
            if (a > mx) mx = a;
        }
        const float sc = mx > 0.0f ? mx / 127.0f : 1.0f;
        for (int i = 0; i < k; ++i) {
            int v = (int)nearbyintf(x[(size_t)t * k + i] / sc);
            xq[(size_t)t * k + i] = (int8_t)(v < -127 ? -127 : (v > 127 ? 127 : v));
        }
        xs[t] = sc;
    }
    qmm_arg a = {m, xq, xs, w, y};
    par_range(m->rows, qmm_range, &a);
    free(xq);
    free(xs);
}

int orc_llama_len(const orc_llama* m) { return m->n_cached; }
void orc_llama_truncate(orc_llama* m, int n) {
    if (n >= 0 && n <= m->n_cached) m->n_cached = n;
}
/* raw bf16 bits of a weight tensor: which 0 emb, 1 head, 2 qkv, 3 o, 4 gu, 5 down */
const uint16_t* orc_llama_tensor(const orc_llama* m, int which, int layer) {
    switch (which) {
        case 0: return m->emb;
        case 1: return m->head;
        case 2: return m->layers[layer].qkv;
        case 3: return m->layers[layer].o;
        case 4: return m->layers[layer].gu;
        default: return m->layers[layer].dn;
    }
}
const int32_t* orc_llama_plant_src(const orc_llama* m) { return m->plant_src; }

/* fp32 dot of a bf16 weight row with an fp32 activation row (16 partial sums) */
static inline float dot_bf16(const uint16_t* w, const float* x, int k) {
    float acc[16] = {0};
    int i = 0;
    for (; i + 16 <= k; i += 16)
        for (int j = 0; j < 16; ++j) acc[j] += bf2f(w[i + j]) * x[i + j];
    for (; i < k; ++i) acc[i & 15] += bf2f(w[i]) * x[i];
    float s = 0.0f;
    for (int j = 0; j < 16; ++j) s += acc[j];
    return s;
}

/* y[t][n] = W[n,:] . x[t,:]  for t < w, n < rows */
typedef struct {
    const uint16_t* W;
    int rows, k, w;
    const float* x;
    float* y;
} mm_arg;
static inline float dot_f32(const float* w, const float* x, int k) {
    float acc[16] = {0};
    int i = 0;
    for (; i + 16 <= k; i += 16)
        for (int j = 0; j < 16; ++j) acc[j] += w[i + j] * x[i + j];
    for (; i < k; ++i) acc[i & 15] += w[i] * x[i];
    float s = 0.0f;
    for (int j = 0; j < 16; ++j) s += acc[j];
    return s;
}
static void mm_range(void* p, int64_t lo, int64_t hi) {
    mm_arg* a = (mm_arg*)p;
    if (a->w == 1) {
        for (int64_t n = lo; n < hi; ++n)
            a->y[n] = dot_bf16(a->W + (size_t)n * a->k, a->x, a->k);
        return;
    }
    float* wr = (float*)malloc(sizeof(float) * a->k);  /* row converted once */
    for (int64_t n = lo; n < hi; ++n) {
        const uint16_t* src = a->W + (size_t)n * a->k;
        for (int i = 0; i < a->k; ++i) wr[i] = bf2f(src[i]);
        for (int t = 0; t < a->w; ++t)
            a->y[(size_t)t * a->rows + n] = dot_f32(wr, a->x + (size_t)t * a->k, a->k);
    }
    free(wr);
}
static void matmul(const uint16_t* W, int rows, int k, const float* x, int w, float* y) {
    mm_arg a = {W, rows, k, w, x, y};
    par_range(rows, mm_range, &a);
}

/* Deferred RMSNorm (mirrors the GPU pass): h = bf16(x * g) and the scale
 * r = 1/sqrt(mean(x^2) + eps) is applied to the consuming GEMM's fp32 output,
 * since W.(x*r*g) == r * (W.(x*g)).  Gains are 1. */
/* Deterministic exp used by the W8A8 (CPU-draft) numerics: Cody-Waite range
 * reduction + degree-6 Taylor polynomial, fp32 with fused multiply-adds.  The
 * product CPU draft (paper_2503_00784_b200/csrc/draft.cpp dd_exp16) runs the
 * same operations in AVX-512 lanes, so the two agree bit for bit. */
static float orc_exp_poly(float x) {
    x = fminf(fmaxf(x, -87.0f), 88.0f);
    const float n = nearbyintf(x * 1.44269504f);
    float r = fmaf(n, -0.693145751953125f, x);
    r = fmaf(n, -1.428606765330187e-06f, r);
    float p = 1.3888889e-03f;
    p = fmaf(p, r, 8.3333333e-03f);
    p = fmaf(p, r, 4.1666667e-02f);
    p = fmaf(p, r, 1.6666667e-01f);
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    const int32_t e = ((int32_t)n + 127) << 23;
    float sc;
    memcpy(&sc, &e, 4);
    return p * sc;
}

static float rmsnorm_bf(const orc_llama* m, const float* x, int d, float eps, float* h) {
    float ss = 0.0f;
    for (int i = 0; i < d; ++i) ss = fmaf(x[i], x[i], ss);
    for (int i = 0; i < d; ++i) h[i] = act(m, x[i] * 1.0f);
    return 1.0f / sqrtf(ss / (float)d + eps);
}
static void scale_rows(float* y, int w, int n, const float* r) {
    for (int t = 0; t < w; ++t)
        for (int i = 0; i < n; ++i) y[(size_t)t * n + i] *= r[t];
}

typedef struct {
    orc_llama* m;
    int l, n0, w;
    const float* q;
    float* o;
    float scale;
} attn_arg;
static void attn_range(void* p, int64_t lo, int64_t hi) {
    attn_arg* a = (attn_arg*)p;
    orc_llama* m = a->m;
    const int hd = m->hd, H = m->H, Hkv = m->Hkv, qd = H * hd, l = a->l;
    for (int64_t job = lo; job < hi; ++job) {
        const int head = (int)(job / a->w), t = (int)(job % a->w);
        const int pos = a->n0 + t, nk = pos + 1;
        const int kvh = head / (H / Hkv);
        const float* qv = a->q + (size_t)t * qd + head * hd;
        float* sc = (float*)malloc(sizeof(float) * nk);
        /* the GPU target feeds bf16(q) to its tensor-core QK^T (attention.cu);
         * the CPU draft (W8A8 mode) keeps q in fp32 */
        float qr[256];
        for (int i = 0; i < hd; ++i) qr[i] = m->quant ? qv[i] : act(m, qv[i]);
        float mx = -INFINITY;
        for (int j = 0; j < nk; ++j) {
            const size_t kr = kv_idx(m, l, 0, kvh, j);
            float acc = 0.0f;
            for (int i = 0; i < hd; ++i) acc = fmaf(qr[i], kv_get(m, kr + i), acc);
            sc[j] = acc * a->scale;
            if (sc[j] > mx) mx = sc[j];
        }
        float sum = 0.0f;
        if (m->quant) {
            /* the CPU draft's order: 16 lane partials over full 16-key blocks,
             * lanes summed 0..15, then the tail keys in order */
            const int nb = nk & ~15;
            float lanes[16] = {0};
            for (int j = 0; j < nb; ++j) {
                sc[j] = orc_exp_poly(sc[j] - mx);
                lanes[j & 15] += sc[j];
            }
            for (int l = 0; l < 16; ++l) sum += lanes[l];
            for (int j = nb; j < nk; ++j) {
                sc[j] = orc_exp_poly(sc[j] - mx);
                sum += sc[j];
            }
        } else {
            for (int j = 0; j < nk; ++j) {
                sc[j] = expf(sc[j] - mx);
                sum += sc[j];
            }
        }
        const float inv = 1.0f / sum;
        if (m->p_bf16)
            for (int j = 0; j < nk; ++j) sc[j] = bfr(sc[j]);
        for (int i = 0; i < hd; ++i) {
            float acc = 0.0f;
            for (int j = 0; j < nk; ++j) acc = fmaf(sc[j], kv_get(m, kv_idx(m, l, 1, kvh, j) + i), acc);
            a->o[(size_t)t * qd + head * hd + i] = act(m, acc * inv);
        }
        free(sc);
    }
}

/* One scored pass of w tokens at positions n_cached..; logits [w][V] (or only
 * the last row when last_only, written at logits[0..V)). */
int orc_llama_forward(orc_llama* m, const int32_t* tokens, int w, float* logits, int last_only) {
    if (w < 1 || m->n_cached + w > m->max_seq) return -1;
    tl_threads = m->n_threads > 0 ? (m->n_threads > 256 ? 256 : m->n_threads) : 1;
    const int d = m->d, hd = m->hd, H = m->H, Hkv = m->Hkv, F = m->F, V = m->V;
    const int qd = H * hd, kvd = Hkv * hd, rows = qd + 2 * kvd, half = hd / 2;
    const int n0 = m->n_cached;
    float* x = (float*)malloc(sizeof(float) * (size_t)w * d);
    float* h = (float*)malloc(sizeof(float) * (size_t)w * d);
    float* qkv = (float*)malloc(sizeof(float) * (size_t)w * rows);
    float* q = (float*)malloc(sizeof(float) * (size_t)w * qd);
    float* o = (float*)malloc(sizeof(float) * (size_t)w * qd);
    float* y = (float*)malloc(sizeof(float) * (size_t)w * (2 * F > d ? 2 * F : d));
    float* a = (float*)malloc(sizeof(float) * (size_t)w * F);
    float* rn = (float*)malloc(sizeof(float) * (size_t)w);
    for (int t = 0; t < w; ++t) {
        if (tokens[t] < 0 || tokens[t] >= V) return -2;
        for (int i = 0; i < d; ++i) x[(size_t)t * d + i] = bf2f(m->emb[(size_t)tokens[t] * d + i]);
        rn[t] = rmsnorm_bf(m, x + (size_t)t * d, d, m->eps, h + (size_t)t * d);
    }
    const float scale = (float)(1.0 / sqrt((double)hd));
    for (int l = 0; l < m->L; ++l) {
        const orc_layer* Ly = &m->layers[l];
        if (m->quant) matmul_q(&Ly->qqkv, h, w, qkv);
        else matmul(Ly->qkv, rows, d, h, w, qkv);
        scale_rows(qkv, w, rows, rn);
        for (int t = 0; t < w; ++t) {
            const int pos = n0 + t;
            const float* cs = m->rope_cos + (size_t)pos * half;
            const float* sn = m->rope_sin + (size_t)pos * half;
            const float* r = qkv + (size_t)t * rows;
            for (int head = 0; head < H + Hkv; ++head)
                for (int i = 0; i < half; ++i) {
                    const float av = r[head * hd + i], bv = r[head * hd + i + half];
                    const float lo = fmaf(av, cs[i], -(bv * sn[i]));
                    const float hi = fmaf(bv, cs[i], av * sn[i]);
                    if (head < H) {
                        q[(size_t)t * qd + head * hd + i] = lo;
                        q[(size_t)t * qd + head * hd + i + half] = hi;
                    } else {
                        const size_t kd = kv_idx(m, l, 0, head - H, pos);
                        kv_put(m, kd + i, lo);
                        kv_put(m, kd + i + half, hi);
                    }
                }
            for (int e = 0; e < kvd; ++e)
                kv_put(m, kv_idx(m, l, 1, e / hd, pos) + e % hd, r[qd + kvd + e]);
        }
        /* attention: query t (pos n0+t) over keys 0..pos */
        {
            attn_arg aa = {m, l, n0, w, q, o, scale};
            par_range((int64_t)H * w, attn_range, &aa);
        }
        if (m->quant) matmul_q(&Ly->qo, o, w, y);
        else matmul(Ly->o, d, qd, o, w, y);
        for (int t = 0; t < w; ++t) {
            for (int i = 0; i < d; ++i) x[(size_t)t * d + i] += y[(size_t)t * d + i];
            rn[t] = rmsnorm_bf(m, x + (size_t)t * d, d, m->eps, h + (size_t)t * d);
        }
        if (m->quant) matmul_q(&Ly->qgu, h, w, y);
        else matmul(Ly->gu, 2 * F, d, h, w, y);
        scale_rows(y, w, 2 * F, rn);
        for (int t = 0; t < w; ++t)
            for (int f = 0; f < F; ++f) {
                const float g = y[(size_t)t * 2 * F + f], u = y[(size_t)t * 2 * F + F + f];
                const float silu = g / (1.0f + (m->quant ? orc_exp_poly(-g) : expf(-g)));
                a[(size_t)t * F + f] = act(m, silu * u);
            }
        if (m->quant) matmul_q(&Ly->qdn, a, w, y);
        else matmul(Ly->dn, d, F, a, w, y);
        for (int t = 0; t < w; ++t) {
            for (int i = 0; i < d; ++i) x[(size_t)t * d + i] += y[(size_t)t * d + i];
            rn[t] = rmsnorm_bf(m, x + (size_t)t * d, d, m->eps, h + (size_t)t * d);
        }
    }
    if (logits) {
        if (last_only) {
            if (m->quant) matmul_q(&m->qhead, h + (size_t)(w - 1) * d, 1, logits);
            else matmul(m->head, V, d, h + (size_t)(w - 1) * d, 1, logits);
            scale_rows(logits, 1, V, rn + (w - 1));
        } else {
            if (m->quant) matmul_q(&m->qhead, h, w, logits);
            else matmul(m->head, V, d, h, w, logits);
            scale_rows(logits, w, V, rn);
        }
    }
    m->n_cached += w;
    free(x);
    free(h);
    free(qkv);
    free(q);
    free(o);
    free(y);
    free(a);
    free(rn);
    return 0;
}
