// CPU draft model: Llama-family forward on pinned host cores, W8A8 (per-row
// int8 weights, per-token int8 activations, AVX-512 VNNI dot products).
//
// This is the draft side of DuoDecoding (north star: "the draft model runs on
// host CPU cores in a concurrent thread").  The reference's draft is a
// ModelSpec table (proj/src/model.cpp:286-320) queried by draft_dynamic
// (proj/src/drafting.cpp:71-136); here it is a Llama-68M-shape transformer
// with the same synthetic-weight generator as the GPU target and the oracle
// (oracle/llama_ref.c), so its logits are checked against the oracle too.
// The KV cache follows the draft context: logits(ctx) keeps the longest
// cached prefix of ctx and runs only the new tokens (branch forks of
// draft_dynamic re-run one token).
#include "draft.h"

#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include "plant.h"

namespace dd {

namespace {

inline uint64_t mix(uint64_t seed, uint64_t m) {
    uint64_t z = seed + m * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t derive(uint64_t base, uint64_t index) {
    uint64_t z = base + (index + 1) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 30)) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline float unit(uint64_t seed, uint64_t e) {
    return static_cast<float>(static_cast<int32_t>(mix(seed, e + 1) >> 40)) * 0x1.0p-23f - 1.0f;
}
inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
inline float bf2f(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
uint64_t tensor_id(int layer, int kind) { return 2 + static_cast<uint64_t>(layer) * 8 + kind; }

void gen(SpinPool& pool, std::vector<uint16_t>& dst, uint64_t offset, uint64_t n, uint64_t seed,
         float amp) {
    pool.run([&](int tid, int nt) {
        const uint64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
        for (uint64_t e = lo; e < hi; ++e) dst[offset + e] = f2bf(unit(seed, e) * amp);
    });
}

// Per-row symmetric int8 quantisation of a bf16 matrix (mirrored bit-for-bit
// by oracle/llama_ref.c orc_quantize_rows).
QMat quantize(const std::vector<uint16_t>& w, int rows, int cols, SpinPool& pool, int levels = 127) {
    QMat m;
    m.rows = rows;
    m.cols = cols;
    m.q.resize(static_cast<size_t>(rows) * cols);
    m.scale.resize(rows);
    m.rowsum.resize(rows);
    pool.run([&](int tid, int nt) {
        const int lo = static_cast<int>(static_cast<int64_t>(rows) * tid / nt);
        const int hi = static_cast<int>(static_cast<int64_t>(rows) * (tid + 1) / nt);
        for (int r = lo; r < hi; ++r) {
            const uint16_t* src = &w[static_cast<size_t>(r) * cols];
            float mx = 0.0f;
            for (int c = 0; c < cols; ++c) mx = std::max(mx, std::fabs(bf2f(src[c])));
            const float sc = mx > 0.0f ? mx / static_cast<float>(levels) : 1.0f;
            int32_t sum = 0;
            int8_t* dst = &m.q[static_cast<size_t>(r) * cols];
            for (int c = 0; c < cols; ++c) {
                int v = static_cast<int>(std::nearbyint(bf2f(src[c]) / sc));
                v = std::max(-levels, std::min(levels, v));
                dst[c] = static_cast<int8_t>(v);
                sum += v;
            }
            m.scale[r] = sc;
            m.rowsum[r] = sum;
        }
    });
    if (rows % 32 == 0 && cols % 64 == 0) {
        m.amx.resize(static_cast<size_t>(rows) * cols);
        const int kb_n = cols / 64;
        pool.run([&](int tid, int nt) {
            for (int nb = tid; nb < rows / 16; nb += nt)
                for (int kb = 0; kb < kb_n; ++kb) {
                    int8_t* tile = &m.amx[(static_cast<size_t>(nb) * kb_n + kb) * 1024];
                    for (int r = 0; r < 16; ++r)      // k / 4 within the block
                        for (int n = 0; n < 16; ++n)  // output row within the block
                            for (int j = 0; j < 4; ++j)
                                tile[r * 64 + n * 4 + j] =
                                    m.q[static_cast<size_t>(nb * 16 + n) * cols + kb * 64 + 4 * r + j];
                }
        });
    }
    return m;
}

// W4 head quantisation (Q4Mat): scale = max|w| / 7, values in [-7, 7]
// (mirrored bit-for-bit by oracle/llama_ref.c quantize_rows with 7 levels).
Q4Mat quantize4(const std::vector<uint16_t>& w, int rows, int cols, SpinPool& pool) {
    Q4Mat m;
    m.rows = rows;
    m.cols = cols;
    m.q.resize(static_cast<size_t>(rows) * cols / 2);
    m.scale.resize(rows);
    m.rowsum.resize(rows);
    pool.run([&](int tid, int nt) {
        const int lo = static_cast<int>(static_cast<int64_t>(rows) * tid / nt);
        const int hi = static_cast<int>(static_cast<int64_t>(rows) * (tid + 1) / nt);
        std::vector<int> v(cols);
        for (int r = lo; r < hi; ++r) {
            const uint16_t* src = &w[static_cast<size_t>(r) * cols];
            float mx = 0.0f;
            for (int c = 0; c < cols; ++c) mx = std::max(mx, std::fabs(bf2f(src[c])));
            const float sc = mx > 0.0f ? mx / 7.0f : 1.0f;
            int32_t sum = 0;
            for (int c = 0; c < cols; ++c) {
                v[c] = std::max(-7, std::min(7, static_cast<int>(std::nearbyint(bf2f(src[c]) / sc))));
                sum += v[c];
            }
            uint8_t* dst = &m.q[static_cast<size_t>(r) * cols / 2];
            for (int b = 0; b < cols / 128; ++b)
                for (int j = 0; j < 64; ++j)
                    dst[b * 64 + j] = static_cast<uint8_t>((v[b * 128 + j] + 8) | ((v[b * 128 + 64 + j] + 8) << 4));
            m.scale[r] = sc;
            m.rowsum[r] = sum;
        }
    });
    return m;
}

// Nibble copy (Q4Mat layout of quantize4) of an int8 QMat quantised with 7
// levels: the decode path streams half the bytes, the int8 copy serves the
// prefill (VNNI / AMX) - the same integers, so the same results.
Q4Mat pack4(const QMat& s8, SpinPool& pool) {
    Q4Mat m;
    m.rows = s8.rows;
    m.cols = s8.cols;
    m.q.resize(static_cast<size_t>(m.rows) * m.cols / 2);
    m.scale = s8.scale;
    m.rowsum = s8.rowsum;
    pool.run([&](int tid, int nt) {
        const int lo = static_cast<int>(static_cast<int64_t>(m.rows) * tid / nt);
        const int hi = static_cast<int>(static_cast<int64_t>(m.rows) * (tid + 1) / nt);
        for (int r = lo; r < hi; ++r) {
            const int8_t* v = &s8.q[static_cast<size_t>(r) * m.cols];
            uint8_t* dst = &m.q[static_cast<size_t>(r) * m.cols / 2];
            for (int b = 0; b < m.cols / 128; ++b)
                for (int j = 0; j < 64; ++j)
                    dst[b * 64 + j] = static_cast<uint8_t>((v[b * 128 + j] + 8) | ((v[b * 128 + 64 + j] + 8) << 4));
        }
    });
    return m;
}

// Per-token symmetric int8 activation quantisation, stored as u8 = q + 128.
void quantize_acts(SpinPool& pool, const uint16_t* X, int w, int k, std::vector<uint8_t>& xq,
                   std::vector<float>& xs) {
    xq.resize(static_cast<size_t>(w) * k);
    xs.resize(w);
    auto one = [&](int t) {
        const uint16_t* x = X + static_cast<size_t>(t) * k;
        float mx = 0.0f;
        for (int i = 0; i < k; ++i) mx = std::max(mx, std::fabs(bf2f(x[i])));
        const float sc = mx > 0.0f ? mx / 127.0f : 1.0f;
        for (int i = 0; i < k; ++i) {
            int v = static_cast<int>(std::nearbyint(bf2f(x[i]) / sc));
            v = std::max(-127, std::min(127, v));
            xq[static_cast<size_t>(t) * k + i] = static_cast<uint8_t>(v + 128);
        }
        xs[t] = sc;
    };
    if (w < 8) {
        for (int t = 0; t < w; ++t) one(t);
    } else {
        pool.run([&](int tid, int nt) {
            for (int t = tid; t < w; t += nt) one(t);
        });
    }
}

// Y[t][n] = (sum_k xq[t][k] * q[n][k]) * (xs[t] * scale[n]) for a block of
// TB tokens x RB weight rows: TB*RB independent vpdpbusd chains, each
// activation and weight load shared across the block (the weights of a row
// block stay in L1 across the token blocks of a prefill).  Integer dots are
// exact, so the blocking does not change any result.
template <int TB, int RB>
__attribute__((target("avx512f,avx512bw,avx512vnni"), always_inline)) inline void qdot_block(
    const QMat& m, const uint8_t* xq, const float* xs, int t0, int n0, float* Y) {
    const int k = m.cols;
    __m512i acc[TB][RB];
#pragma GCC unroll 8
    for (int t = 0; t < TB; ++t)
#pragma GCC unroll 8
        for (int r = 0; r < RB; ++r) acc[t][r] = _mm512_setzero_si512();
    for (int i = 0; i < k; i += 64) {
        __m512i xv[TB];
#pragma GCC unroll 8
        for (int t = 0; t < TB; ++t)
            xv[t] = _mm512_loadu_si512(xq + static_cast<size_t>(t0 + t) * k + i);
#pragma GCC unroll 8
        for (int r = 0; r < RB; ++r) {
            const __m512i wv = _mm512_loadu_si512(&m.q[static_cast<size_t>(n0 + r) * k + i]);
#pragma GCC unroll 8
            for (int t = 0; t < TB; ++t) acc[t][r] = _mm512_dpbusd_epi32(acc[t][r], xv[t], wv);
        }
    }
#pragma GCC unroll 8
    for (int t = 0; t < TB; ++t)
#pragma GCC unroll 8
        for (int r = 0; r < RB; ++r) {
            const int32_t dot = _mm512_reduce_add_epi32(acc[t][r]) - 128 * m.rowsum[n0 + r];
            Y[static_cast<size_t>(t0 + t) * m.rows + n0 + r] =
                static_cast<float>(dot) * (xs[t0 + t] * m.scale[n0 + r]);
        }
}

__attribute__((target("avx512f,avx512bw,avx512vnni"))) void qdot_rows(
    const QMat& m, const uint8_t* xq, const float* xs, int w, int lo, int hi, float* Y) {
    if (w >= 4) {
        // prefill: 4 tokens x 6 rows (24 accumulators + 4 activations + 1 weight)
        int n = lo;
        for (; n + 6 <= hi; n += 6) {
            int t = 0;
            for (; t + 4 <= w; t += 4) qdot_block<4, 6>(m, xq, xs, t, n, Y);
            for (; t < w; ++t) qdot_block<1, 6>(m, xq, xs, t, n, Y);
        }
        for (; n < hi; ++n) {
            int t = 0;
            for (; t + 4 <= w; t += 4) qdot_block<4, 1>(m, xq, xs, t, n, Y);
            for (; t < w; ++t) qdot_block<1, 1>(m, xq, xs, t, n, Y);
        }
        return;
    }
    for (int t = 0; t < w; ++t) {
        int n = lo;
        for (; n + 8 <= hi; n += 8) qdot_block<1, 8>(m, xq, xs, t, n, Y);
        for (; n < hi; ++n) qdot_block<1, 1>(m, xq, xs, t, n, Y);
    }
}

__attribute__((target("avx512f,avx512bw,avx512vnni"), always_inline)) inline void q4_finish(
    const Q4Mat& m, int n, __m512i acc, int32_t xsum, float xs, float* Y) {
    const int32_t dot = _mm512_reduce_add_epi32(acc) - 8 * xsum - 128 * m.rowsum[n];
    Y[n] = static_cast<float>(dot) * (xs * m.scale[n]);
}

// One token against the W4 head.  With u8 activations a = q + 128 and
// offset-binary weights b = w + 8, dpbusd sums a.b = q.w + 8 sum(q) + 128 sum(w)
// + 1024 k, so q.w = a.b - 8 sum(a) - 128 sum(w): exact integers.
__attribute__((target("avx512f,avx512bw,avx512vnni"))) void qdot4_rows(
    const Q4Mat& m, const uint8_t* xq, float xs, int32_t xsum, int lo, int hi, float* Y) {
    const int nb = m.cols / 128;
    const size_t rb = static_cast<size_t>(m.cols) / 2;
    const __m512i mask = _mm512_set1_epi8(0x0F);
    int n = lo;
    for (; n + 8 <= hi; n += 8) {
        __m512i acc[8];
#pragma GCC unroll 8
        for (int r = 0; r < 8; ++r) acc[r] = _mm512_setzero_si512();
        for (int b = 0; b < nb; ++b) {
            const __m512i x0 = _mm512_loadu_si512(xq + b * 128), x1 = _mm512_loadu_si512(xq + b * 128 + 64);
#pragma GCC unroll 8
            for (int r = 0; r < 8; ++r) {
                const __m512i v = _mm512_loadu_si512(&m.q[(n + r) * rb + b * 64]);
                acc[r] = _mm512_dpbusd_epi32(acc[r], x0, _mm512_and_si512(v, mask));
                acc[r] = _mm512_dpbusd_epi32(acc[r], x1, _mm512_and_si512(_mm512_srli_epi16(v, 4), mask));
            }
        }
#pragma GCC unroll 8
        for (int r = 0; r < 8; ++r) q4_finish(m, n + r, acc[r], xsum, xs, Y);
    }
    for (; n < hi; ++n) {
        __m512i acc = _mm512_setzero_si512();
        for (int b = 0; b < nb; ++b) {
            const __m512i v = _mm512_loadu_si512(&m.q[n * rb + b * 64]);
            acc = _mm512_dpbusd_epi32(acc, _mm512_loadu_si512(xq + b * 128), _mm512_and_si512(v, mask));
            acc = _mm512_dpbusd_epi32(acc, _mm512_loadu_si512(xq + b * 128 + 64),
                                      _mm512_and_si512(_mm512_srli_epi16(v, 4), mask));
        }
        q4_finish(m, n, acc, xsum, xs, Y);
    }
}

void matmul4(SpinPool& pool, const Q4Mat& m, const uint16_t* x, float* Y, std::vector<uint8_t>& xq,
             std::vector<float>& xs) {
    quantize_acts(pool, x, 1, m.cols, xq, xs);
    int32_t xsum = 0;
    for (int i = 0; i < m.cols; ++i) xsum += xq[i];
    const int blocks = (m.rows + 7) / 8;
    pool.run([&](int tid, int nt) {
        const int lo = std::min(m.rows, static_cast<int>(static_cast<int64_t>(blocks) * tid / nt) * 8);
        const int hi = std::min(m.rows, static_cast<int>(static_cast<int64_t>(blocks) * (tid + 1) / nt) * 8);
        if (lo < hi) qdot4_rows(m, xq.data(), xs[0], xsum, lo, hi, Y);
    });
}

// ---- AMX (TDPBUSD) prefill matmul: the same u8 x s8 integer dot products as
// the VNNI path (exact), 32 tokens x 32 rows per step in four int32 tiles.
bool amx_ready() {
    static const bool ok = [] {
        const char* env = getenv("DD_DRAFT_AMX");
        if ((env && env[0] == '0') || !__builtin_cpu_supports("amx-int8")) return false;
        constexpr long kArchReqXcompPerm = 0x1023, kXfeatureXtiledata = 18;  // Linux arch_prctl
        return syscall(SYS_arch_prctl, kArchReqXcompPerm, kXfeatureXtiledata) == 0;
    }();
    return ok;
}

struct alignas(64) TileCfg {
    uint8_t palette = 1, start_row = 0, pad[14] = {};
    uint16_t colsb[16] = {};
    uint8_t rows[16] = {};
};

__attribute__((target("amx-tile,amx-int8,avx512f"))) void qdot_amx(
    const QMat& m, const uint8_t* xq, const float* xs, int w, int n_lo, int n_hi, float* Y) {
    TileCfg cfg;
    for (int t = 0; t < 8; ++t) {
        cfg.colsb[t] = 64;
        cfg.rows[t] = 16;
    }
    _tile_loadconfig(&cfg);
    const int k = m.cols, kb_n = k / 64;
    alignas(64) int32_t c[4][16][16];
    for (int n0 = n_lo; n0 < n_hi; n0 += 32) {
        const int8_t* b0 = &m.amx[static_cast<size_t>(n0 / 16) * kb_n * 1024];
        const int8_t* b1 = b0 + static_cast<size_t>(kb_n) * 1024;
        for (int t0 = 0; t0 < w; t0 += 32) {  // xq holds a multiple of 32 rows
            _tile_zero(0);
            _tile_zero(1);
            _tile_zero(2);
            _tile_zero(3);
            for (int kb = 0; kb < kb_n; ++kb) {
                _tile_loadd(4, xq + static_cast<size_t>(t0) * k + kb * 64, k);
                _tile_loadd(5, xq + static_cast<size_t>(t0 + 16) * k + kb * 64, k);
                _tile_loadd(6, b0 + static_cast<size_t>(kb) * 1024, 64);
                _tile_loadd(7, b1 + static_cast<size_t>(kb) * 1024, 64);
                _tile_dpbusd(0, 4, 6);
                _tile_dpbusd(1, 4, 7);
                _tile_dpbusd(2, 5, 6);
                _tile_dpbusd(3, 5, 7);
            }
            _tile_stored(0, c[0], 64);
            _tile_stored(1, c[1], 64);
            _tile_stored(2, c[2], 64);
            _tile_stored(3, c[3], 64);
            for (int q = 0; q < 4; ++q) {
                const int tb = t0 + (q >> 1) * 16, nb = n0 + (q & 1) * 16;
                for (int i = 0; i < 16 && tb + i < w; ++i)
                    for (int j = 0; j < 16; ++j) {
                        const int32_t dot = c[q][i][j] - 128 * m.rowsum[nb + j];
                        Y[static_cast<size_t>(tb + i) * m.rows + nb + j] =
                            static_cast<float>(dot) * (xs[tb + i] * m.scale[nb + j]);
                    }
            }
        }
    }
    _tile_release();
}

void matmul(SpinPool& pool, const QMat& m, const uint16_t* X, int w, float* Y,
            std::vector<uint8_t>& xq, std::vector<float>& xs) {
    quantize_acts(pool, X, w, m.cols, xq, xs);
    if (w >= 16 && !m.amx.empty() && amx_ready()) {
        // pad the activation rows to a multiple of 32 (rows past w are never stored)
        const int wp = (w + 31) & ~31;
        if (xq.size() < static_cast<size_t>(wp) * m.cols) xq.resize(static_cast<size_t>(wp) * m.cols, 128);
        const int units = m.rows / 32;
        pool.run([&](int tid, int nt) {
            const int lo = static_cast<int>(static_cast<int64_t>(units) * tid / nt) * 32;
            const int hi = static_cast<int>(static_cast<int64_t>(units) * (tid + 1) / nt) * 32;
            if (lo < hi) qdot_amx(m, xq.data(), xs.data(), w, lo, hi, Y);
        });
        return;
    }
    const int gran = w >= 4 ? 6 : 8;
    const int blocks = (m.rows + gran - 1) / gran;
    pool.run([&](int tid, int nt) {
        const int lo = std::min(m.rows, static_cast<int>(static_cast<int64_t>(blocks) * tid / nt) * gran);
        const int hi = std::min(m.rows, static_cast<int>(static_cast<int64_t>(blocks) * (tid + 1) / nt) * gran);
        if (lo < hi) qdot_rows(m, xq.data(), xs.data(), w, lo, hi, Y);
    });
}

// deferred RMSNorm (same formulation as the GPU target and the oracle):
// h = bf16(x * g), r applied to the consuming matmul's fp32 output
float rmsnorm_bf(const float* x, int d, float eps, uint16_t* h) {
    float ss = 0.0f;
    for (int i = 0; i < d; ++i) ss = std::fmaf(x[i], x[i], ss);
    for (int i = 0; i < d; ++i) h[i] = f2bf(x[i]);
    return 1.0f / std::sqrt(ss / static_cast<float>(d) + eps);
}

}  // namespace

// ------------------------------------------------------------------ pool
SpinPool::SpinPool(int n_threads, const std::vector<int>& cpus)
    : n_(std::max(1, n_threads)), done_(new Done[std::max(1, n_threads)]) {
    // workers 1..n-1 are pinned to cpus[1..]; the calling thread (tid 0, the
    // engine's draft worker) pins itself to cpus[0]
    for (int i = 1; i < n_; ++i) {
        th_.emplace_back([this, i] { worker(i); });
        if (!cpus.empty()) {
            cpu_set_t set;
            CPU_ZERO(&set);
            CPU_SET(cpus[static_cast<size_t>(i) % cpus.size()], &set);
            pthread_setaffinity_np(th_.back().native_handle(), sizeof(set), &set);
        }
    }
}

SpinPool::~SpinPool() {
    stop_.store(true, std::memory_order_release);
    gen_.fetch_add(1, std::memory_order_acq_rel);
    gen_.notify_all();
    for (auto& t : th_) t.join();
}

void SpinPool::worker(int tid) {
    uint64_t seen = 0;
    for (;;) {
        // spin ~50 us (the engine issues back-to-back jobs), then sleep in a
        // futex wait so an idle draft does not steal host cores
        int spins = 0;
        while (gen_.load(std::memory_order_acquire) == seen) {
            if (++spins < 20000) {
                _mm_pause();
            } else {
                sleepers_.fetch_add(1, std::memory_order_acq_rel);
                gen_.wait(seen, std::memory_order_acquire);
                sleepers_.fetch_sub(1, std::memory_order_acq_rel);
            }
        }
        seen = gen_.load(std::memory_order_acquire);
        if (stop_.load(std::memory_order_acquire)) return;
        (*job_)(tid, n_);
        done_[tid].gen.store(seen, std::memory_order_release);
    }
}

void SpinPool::run(const std::function<void(int, int)>& fn) {
    if (n_ == 1) {
        fn(0, 1);
        return;
    }
    job_ = &fn;
    const uint64_t g = gen_.fetch_add(1, std::memory_order_acq_rel) + 1;
    if (sleepers_.load(std::memory_order_acquire) > 0) gen_.notify_all();
    fn(0, n_);
    for (int t = 1; t < n_; ++t)
        while (done_[t].gen.load(std::memory_order_acquire) != g) _mm_pause();
}

// ------------------------------------------------------------------ model
CpuLlama::CpuLlama(const dd_model_desc& d, uint64_t weight_seed, const dd_plant_desc* plant,
                   int n_threads, const std::vector<int>& cpus)
    : L_(d.n_layers), d_(d.d_model), H_(d.n_heads), Hkv_(d.n_kv_heads > 0 ? d.n_kv_heads : d.n_heads),
      hd_(d.head_dim), F_(d.ffn_dim), V_(d.vocab), max_seq_(d.max_seq), eps_(d.rms_eps) {
    pool_ = std::make_unique<SpinPool>(n_threads, cpus);
    const int qd = H_ * hd_, kvd = Hkv_ * hd_;
    const float amp_proj = static_cast<float>(0.02 * std::sqrt(3.0));
    const float amp_out = static_cast<float>(0.02 / std::sqrt(2.0 * L_) * std::sqrt(3.0));
    PlantTable pt = make_plant_table(V_, d_, plant);
    const float amp_emb = static_cast<float>(pt.emb_std * std::sqrt(3.0));
    const uint64_t D = static_cast<uint64_t>(d_);
    emb_.resize(static_cast<size_t>(V_) * D);
    std::vector<uint16_t> head_bf(static_cast<size_t>(V_) * D);
    gen(*pool_, emb_, 0, V_ * D, derive(weight_seed, 0), amp_emb);
    {
        const uint64_t hs = derive(weight_seed, 1);
        const uint64_t n = V_ * D;
        pool_->run([&](int tid, int nt) {
            const uint64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
            for (uint64_t e = lo; e < hi; ++e) {
                float w = unit(hs, e) * amp_proj;
                const int32_t t = pt.any ? pt.src[e / D] : -1;
                if (t >= 0) w = std::fmaf(pt.coef, bf2f(emb_[static_cast<size_t>(t) * D + e % D]), w);
                head_bf[e] = f2bf(w);
            }
        });
        const char* hb = getenv("DD_DRAFT_HEAD_BITS");
        head_w4_ = d_ % 128 == 0 && !(hb && atoi(hb) == 8);
        if (head_w4_) {
            head4_ = quantize4(head_bf, V_, d_, *pool_);
        } else {
            head_ = quantize(head_bf, V_, d_, *pool_);
        }
    }
    layers_.resize(L_);
    for (int l = 0; l < L_; ++l) {
        DraftLayer& Ly = layers_[l];
        std::vector<uint16_t> qkv(static_cast<size_t>(qd + 2 * kvd) * D), o(D * qd),
            gu(2 * static_cast<size_t>(F_) * D), dn(D * F_);
        gen(*pool_, qkv, 0, qd * D, derive(weight_seed, tensor_id(l, 0)), amp_proj);
        gen(*pool_, qkv, qd * D, kvd * D, derive(weight_seed, tensor_id(l, 1)), amp_proj);
        gen(*pool_, qkv, (qd + kvd) * D, kvd * D, derive(weight_seed, tensor_id(l, 2)), amp_proj);
        gen(*pool_, o, 0, D * qd, derive(weight_seed, tensor_id(l, 3)), amp_out);
        gen(*pool_, gu, 0, F_ * D, derive(weight_seed, tensor_id(l, 4)), amp_proj);
        gen(*pool_, gu, F_ * D, F_ * D, derive(weight_seed, tensor_id(l, 5)), amp_proj);
        gen(*pool_, dn, 0, D * F_, derive(weight_seed, tensor_id(l, 6)), amp_out);
        // DD_DRAFT_ATTN_BITS=4: QKV and O 4-bit as well (same scheme as the FFN below)
        static const bool attn4 = getenv("DD_DRAFT_ATTN_BITS") && atoi(getenv("DD_DRAFT_ATTN_BITS")) == 4;
        Ly.a4 = attn4 && d_ % 128 == 0 && qd % 128 == 0;
        Ly.qkv = quantize(qkv, qd + 2 * kvd, d_, *pool_, Ly.a4 ? 7 : 127);
        Ly.o = quantize(o, d_, qd, *pool_, Ly.a4 ? 7 : 127);
        if (Ly.a4) {
            Ly.qkv4 = pack4(Ly.qkv, *pool_);
            Ly.o4 = pack4(Ly.o, *pool_);
        }
        // gate/up and down quantised to 7 levels (4-bit) and streamed as nibbles by
        // decode - 2/3 of the layer bytes, so a drafted token reads 24 instead of 31 MB
        // (c 16.1 -> 20.8 on the B200 host, tokens per iteration unchanged, config 2
        // 1542 -> 1595 tok/s); DD_DRAFT_FFN_BITS=8 keeps them int8.  The oracle's
        // W8A8 mode mirrors it.
        static const bool ffn4 = !(getenv("DD_DRAFT_FFN_BITS") && atoi(getenv("DD_DRAFT_FFN_BITS")) == 8);
        Ly.w4 = ffn4 && d_ % 128 == 0 && F_ % 128 == 0;
        Ly.gu = quantize(gu, 2 * F_, d_, *pool_, Ly.w4 ? 7 : 127);
        Ly.dn = quantize(dn, d_, F_, *pool_, Ly.w4 ? 7 : 127);
        if (Ly.w4) {
            Ly.gu4 = pack4(Ly.gu, *pool_);
            Ly.dn4 = pack4(Ly.dn, *pool_);
        }
    }
    kv_.assign(static_cast<size_t>(L_) * 2 * Hkv_ * ((max_seq_ + 15) & ~15) * hd_, 0);
    const int half = hd_ / 2;
    rope_cos_.resize(static_cast<size_t>(max_seq_) * half);
    rope_sin_.resize(rope_cos_.size());
    for (int p = 0; p < max_seq_; ++p)
        for (int i = 0; i < half; ++i) {
            const double inv = std::pow(static_cast<double>(d.rope_theta), -2.0 * i / hd_);
            rope_cos_[static_cast<size_t>(p) * half + i] = static_cast<float>(std::cos(p * inv));
            rope_sin_[static_cast<size_t>(p) * half + i] = static_cast<float>(std::sin(p * inv));
        }
    logits_tmp_.resize(V_);
}

bool CpuLlama::logits(const int32_t* ctx, int n, float* out) {
    if (n < 1 || n > max_seq_) {
        err = "draft context length out of range";
        return false;
    }
    for (int i = 0; i < n; ++i)
        if (ctx[i] < 0 || ctx[i] >= V_) {
            err = "draft token outside vocabulary";
            return false;
        }
    // keep the longest cached prefix, always re-running at least the last token
    int keep = 0;
    const int lim = std::min<int>(static_cast<int>(tokens_.size()), n - 1);
    while (keep < lim && tokens_[keep] == ctx[keep]) ++keep;
    tokens_.resize(keep);
    int pos = keep;
    while (pos < n) {
        const int w = std::min(256, n - pos);
        forward(ctx + pos, w, out);
        pos += w;
    }
    return true;
}

namespace {
// Deterministic exp (Cody-Waite + degree-6 Taylor, fp32 FMA), 16 lanes; the
// oracle's orc_exp_poly (oracle/llama_ref.c) is the same operation sequence
// in scalar code, so draft and oracle agree bit for bit.
__attribute__((target("avx512f"), always_inline)) inline __m512 dd_exp16(__m512 x) {
    x = _mm512_min_ps(_mm512_max_ps(x, _mm512_set1_ps(-87.0f)), _mm512_set1_ps(88.0f));
    const __m512 n = _mm512_roundscale_ps(_mm512_mul_ps(x, _mm512_set1_ps(1.44269504f)),
                                          _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    __m512 r = _mm512_fmadd_ps(n, _mm512_set1_ps(-0.693145751953125f), x);
    r = _mm512_fmadd_ps(n, _mm512_set1_ps(-1.428606765330187e-06f), r);
    __m512 p = _mm512_set1_ps(1.3888889e-03f);
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(8.3333333e-03f));
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(4.1666667e-02f));
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.6666667e-01f));
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(0.5f));
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f));
    p = _mm512_fmadd_ps(p, r, _mm512_set1_ps(1.0f));
    const __m512i e = _mm512_slli_epi32(
        _mm512_add_epi32(_mm512_cvtps_epi32(n), _mm512_set1_epi32(127)), 23);
    return _mm512_mul_ps(p, _mm512_castsi512_ps(e));
}
__attribute__((target("avx512f"))) float dd_exp1(float x) {
    alignas(64) float t[16];
    _mm512_store_ps(t, dd_exp16(_mm512_set1_ps(x)));
    return t[0];
}

// 16 bf16 -> 16 fp32 (exact)
__attribute__((target("avx512f,avx512bw"), always_inline)) inline __m512 load_bf16x16(
    const uint16_t* p) {
    const __m512i v = _mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(p)));
    return _mm512_castsi512_ps(_mm512_slli_epi32(v, 16));
}

// One (head, query) of causal attention over keys 0..nk-1.  K is stored in
// 16-key blocks, dim-major inside a block (kt[pos/16][i][pos%16]) so 16 keys' scores are computed in 16 lanes, each
// lane accumulating over the head dims in order: exactly the scalar
// acc = fma(q[i], k[i], acc) chain of the oracle.  PV accumulates over keys in
// order with the head dims in lanes.  Bit-identical to the scalar loop.
__attribute__((target("avx512f,avx512bw"))) void attend_one(
    const float* qv, const uint16_t* kt, const uint16_t* v, int nk, int hd, int max_seq,
    float scale, std::vector<float>& sc, uint16_t* out) {
    sc.resize(static_cast<size_t>(nk) + 16);
    int j = 0;
    const __m512 vs = _mm512_set1_ps(scale);
    for (; j + 64 <= nk; j += 64) {  // four independent 16-key chains
        const uint16_t* kb = kt + static_cast<size_t>(j) * hd;
        const size_t bs = static_cast<size_t>(hd) * 16;
        __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
        for (int i = 0; i < hd; ++i) {
            const __m512 qb = _mm512_set1_ps(qv[i]);
            a0 = _mm512_fmadd_ps(qb, load_bf16x16(kb + i * 16), a0);
            a1 = _mm512_fmadd_ps(qb, load_bf16x16(kb + bs + i * 16), a1);
            a2 = _mm512_fmadd_ps(qb, load_bf16x16(kb + 2 * bs + i * 16), a2);
            a3 = _mm512_fmadd_ps(qb, load_bf16x16(kb + 3 * bs + i * 16), a3);
        }
        _mm512_storeu_ps(&sc[j], _mm512_mul_ps(a0, vs));
        _mm512_storeu_ps(&sc[j + 16], _mm512_mul_ps(a1, vs));
        _mm512_storeu_ps(&sc[j + 32], _mm512_mul_ps(a2, vs));
        _mm512_storeu_ps(&sc[j + 48], _mm512_mul_ps(a3, vs));
    }
    for (; j + 16 <= nk; j += 16) {
        const uint16_t* kb = kt + static_cast<size_t>(j) * hd;  // block j/16
        __m512 acc = _mm512_setzero_ps();
        for (int i = 0; i < hd; ++i)
            acc = _mm512_fmadd_ps(_mm512_set1_ps(qv[i]), load_bf16x16(kb + i * 16), acc);
        _mm512_storeu_ps(&sc[j], _mm512_mul_ps(acc, _mm512_set1_ps(scale)));
    }
    for (; j < nk; ++j) {
        float acc = 0.0f;
        for (int i = 0; i < hd; ++i)
            acc = std::fmaf(qv[i], bf2f(kt[static_cast<size_t>(j >> 4) * hd * 16 + i * 16 + (j & 15)]), acc);
        sc[j] = acc * scale;
    }
    // max is order-free; the sum uses the oracle's fixed order: 16 lane
    // partials over the full 16-key blocks, lanes added 0..15, then the tail
    const int nb = nk & ~15;
    float mx = -INFINITY;
    {
        __m512 vmx = _mm512_set1_ps(-INFINITY);
        for (int jj = 0; jj < nb; jj += 16) vmx = _mm512_max_ps(vmx, _mm512_loadu_ps(&sc[jj]));
        mx = _mm512_reduce_max_ps(vmx);
        for (int jj = nb; jj < nk; ++jj) mx = std::max(mx, sc[jj]);
    }
    float sum = 0.0f;
    {
        const __m512 vm = _mm512_set1_ps(mx);
        __m512 vsum = _mm512_setzero_ps();
        for (int jj = 0; jj < nb; jj += 16) {
            const __m512 e = dd_exp16(_mm512_sub_ps(_mm512_loadu_ps(&sc[jj]), vm));
            _mm512_storeu_ps(&sc[jj], e);
            vsum = _mm512_add_ps(vsum, e);
        }
        alignas(64) float lanes[16];
        _mm512_store_ps(lanes, vsum);
        for (int l = 0; l < 16; ++l) sum += lanes[l];
        for (int jj = nb; jj < nk; ++jj) {
            sc[jj] = dd_exp1(sc[jj] - mx);
            sum += sc[jj];
        }
    }
    const float inv = 1.0f / sum;
    if (hd % 16 == 0 && hd <= 256) {
        __m512 acc[16];
        const int nv = hd / 16;
        for (int c = 0; c < nv; ++c) acc[c] = _mm512_setzero_ps();
        for (int jj = 0; jj < nk; ++jj) {
            const __m512 p = _mm512_set1_ps(sc[jj]);
            const uint16_t* vr = v + static_cast<size_t>(jj) * hd;
            for (int c = 0; c < nv; ++c) acc[c] = _mm512_fmadd_ps(p, load_bf16x16(vr + 16 * c), acc[c]);
        }
        alignas(64) float tmp[256];
        for (int c = 0; c < nv; ++c) _mm512_store_ps(tmp + 16 * c, acc[c]);
        for (int i = 0; i < hd; ++i) out[i] = f2bf(tmp[i] * inv);
    } else {
        float acc[256];
        for (int i = 0; i < hd; ++i) acc[i] = 0.0f;
        for (int jj = 0; jj < nk; ++jj) {
            const uint16_t* vr = v + static_cast<size_t>(jj) * hd;
            for (int i = 0; i < hd; ++i) acc[i] = std::fmaf(sc[jj], bf2f(vr[i]), acc[i]);
        }
        for (int i = 0; i < hd; ++i) out[i] = f2bf(acc[i] * inv);
    }
}
// a[f] = bf16(silu(g) * u), g = gu[f] * r, u = gu[F + f] * r (oracle order)
__attribute__((target("avx512f"))) void swiglu_row(const float* gu, float r, int F, uint16_t* a) {
    const __m512 vr = _mm512_set1_ps(r), one = _mm512_set1_ps(1.0f);
    alignas(64) float tmp[16];
    int f = 0;
    for (; f + 16 <= F; f += 16) {
        const __m512 g = _mm512_mul_ps(_mm512_loadu_ps(gu + f), vr);
        const __m512 u = _mm512_mul_ps(_mm512_loadu_ps(gu + F + f), vr);
        const __m512 e = dd_exp16(_mm512_sub_ps(_mm512_setzero_ps(), g));
        _mm512_store_ps(tmp, _mm512_mul_ps(_mm512_div_ps(g, _mm512_add_ps(one, e)), u));
        for (int i = 0; i < 16; ++i) a[f + i] = f2bf(tmp[i]);
    }
    for (; f < F; ++f) {
        const float g = gu[f] * r, u = gu[F + f] * r;
        a[f] = f2bf(g / (1.0f + dd_exp1(-g)) * u);
    }
}
}  // namespace

void CpuLlama::forward(const int32_t* toks, int w, float* logits_last) {
    const int n0 = static_cast<int>(tokens_.size());
    const int qd = H_ * hd_, kvd = Hkv_ * hd_, rows = qd + 2 * kvd, half = hd_ / 2;
    const size_t W = static_cast<size_t>(w);
    x_.resize(W * d_);
    hb_.resize(W * d_);
    qkv_.resize(W * rows);
    q_.resize(W * qd);
    ob_.resize(W * qd);
    gu_.resize(W * 2 * F_);
    ab_.resize(W * F_);
    y_.resize(W * std::max(d_, 2 * F_));
    std::vector<float> rn(W);
    // per-token elementwise work: on the pool for prefill-sized w
    auto per_token = [&](const std::function<void(int)>& fn) {
        if (w < 8) {
            for (int t = 0; t < w; ++t) fn(t);
        } else {
            pool_->run([&](int tid, int nt) {  // contiguous chunks: no false sharing
                const int lo = w * tid / nt, hi = w * (tid + 1) / nt;
                for (int t = lo; t < hi; ++t) fn(t);
            });
        }
    };
    per_token([&](int t) {
        for (int i = 0; i < d_; ++i)
            x_[t * d_ + i] = bf2f(emb_[static_cast<size_t>(toks[t]) * d_ + i]);
        rn[t] = rmsnorm_bf(&x_[t * d_], d_, eps_, &hb_[t * d_]);
    });
    const size_t ms16 = static_cast<size_t>((max_seq_ + 15) & ~15);
    // K in 16-key blocks, dim-major inside a block: [l][h][pos/16][i][16];
    // V row-major [l][h][pos][i]
    auto ktp = [&](int l, int h) {
        return &kv_[((static_cast<size_t>(l) * 2 + 0) * Hkv_ + h) * ms16 * hd_];
    };
    auto kt_at = [&](int i, int pos) {
        return static_cast<size_t>(pos >> 4) * hd_ * 16 + static_cast<size_t>(i) * 16 + (pos & 15);
    };
    auto vp = [&](int l, int h, int pos) {
        return &kv_[(((static_cast<size_t>(l) * 2 + 1) * Hkv_ + h) * ms16 + pos) * hd_];
    };
    const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(hd_)));
    for (int l = 0; l < L_; ++l) {
        const DraftLayer& Ly = layers_[l];
        if (Ly.a4 && w == 1) matmul4(*pool_, Ly.qkv4, hb_.data(), qkv_.data(), xq_, xs_);
        else matmul(*pool_, Ly.qkv, hb_.data(), w, qkv_.data(), xq_, xs_);
        per_token([&](int t) {
            float* r = &qkv_[static_cast<size_t>(t) * rows];
            for (int i = 0; i < rows; ++i) r[i] *= rn[t];
            const int pos = n0 + t;
            const float* cs = &rope_cos_[static_cast<size_t>(pos) * half];
            const float* sn = &rope_sin_[static_cast<size_t>(pos) * half];
            for (int head = 0; head < H_ + Hkv_; ++head)
                for (int i = 0; i < half; ++i) {
                    const float av = r[head * hd_ + i], bv = r[head * hd_ + i + half];
                    const float lo = std::fmaf(av, cs[i], -(bv * sn[i]));
                    const float hi = std::fmaf(bv, cs[i], av * sn[i]);
                    if (head < H_) {
                        q_[t * qd + head * hd_ + i] = lo;
                        q_[t * qd + head * hd_ + i + half] = hi;
                    } else {
                        uint16_t* kt = ktp(l, head - H_);
                        kt[kt_at(i, pos)] = f2bf(lo);
                        kt[kt_at(i + half, pos)] = f2bf(hi);
                    }
                }
            for (int e = 0; e < kvd; ++e) vp(l, e / hd_, pos)[e % hd_] = f2bf(r[qd + kvd + e]);
        });
        pool_->run([&](int tid, int nt) {
            std::vector<float> sc;
            const int jobs = H_ * w;
            // balance the causal triangle: long (late) queries first, strided
            for (int jb = tid; jb < jobs; jb += nt) {
                const int job = jobs - 1 - jb;
                const int t = job / H_, head = job % H_;
                const int pos = n0 + t, kvh = head / (H_ / Hkv_);
                attend_one(&q_[t * qd + head * hd_], ktp(l, kvh), vp(l, kvh, 0), pos + 1, hd_,
                           max_seq_, scale, sc, &ob_[t * qd + head * hd_]);
            }
        });
        if (Ly.a4 && w == 1) matmul4(*pool_, Ly.o4, ob_.data(), y_.data(), xq_, xs_);
        else matmul(*pool_, Ly.o, ob_.data(), w, y_.data(), xq_, xs_);
        per_token([&](int t) {
            for (int i = 0; i < d_; ++i) x_[t * d_ + i] += y_[t * d_ + i];
            rn[t] = rmsnorm_bf(&x_[t * d_], d_, eps_, &hb_[t * d_]);
        });
        if (Ly.w4 && w == 1) matmul4(*pool_, Ly.gu4, hb_.data(), gu_.data(), xq_, xs_);
        else matmul(*pool_, Ly.gu, hb_.data(), w, gu_.data(), xq_, xs_);
        per_token([&](int t) {
            swiglu_row(&gu_[static_cast<size_t>(t) * 2 * F_], rn[t], F_, &ab_[static_cast<size_t>(t) * F_]);
        });
        if (Ly.w4 && w == 1) matmul4(*pool_, Ly.dn4, ab_.data(), y_.data(), xq_, xs_);
        else matmul(*pool_, Ly.dn, ab_.data(), w, y_.data(), xq_, xs_);
        per_token([&](int t) {
            for (int i = 0; i < d_; ++i) x_[t * d_ + i] += y_[t * d_ + i];
            rn[t] = rmsnorm_bf(&x_[t * d_], d_, eps_, &hb_[t * d_]);
        });
    }
    if (head_w4_) {
        matmul4(*pool_, head4_, &hb_[(W - 1) * d_], logits_last, xq_, xs_);
    } else {
        matmul(*pool_, head_, &hb_[(W - 1) * d_], 1, logits_last, xq_, xs_);
    }
    for (int i = 0; i < V_; ++i) logits_last[i] *= rn[W - 1];
    tokens_.insert(tokens_.end(), toks, toks + w);
}

int CpuLlama::distribution(const float* lg, double temperature, bool greedy, float* q) {
    // argmax, lowest index on ties (kernels_scalar.cpp:40-48)
    const int nt = pool_->size();
    std::vector<float> bestv(nt, -INFINITY);
    std::vector<int> besti(nt, 0);
    std::vector<double> sums(nt, 0.0);
    pool_->run([&](int tid, int n) {
        const int lo = static_cast<int>(static_cast<int64_t>(V_) * tid / n);
        const int hi = static_cast<int>(static_cast<int64_t>(V_) * (tid + 1) / n);
        float bv = -INFINITY;
        int bi = lo;
        for (int i = lo; i < hi; ++i)
            if (lg[i] > bv) {
                bv = lg[i];
                bi = i;
            }
        bestv[tid] = bv;
        besti[tid] = bi;
    });
    float bv = bestv[0];
    int bi = besti[0];
    for (int t = 1; t < nt; ++t)
        if (bestv[t] > bv) {
            bv = bestv[t];
            bi = besti[t];
        }
    if (greedy) {  // one-hot at the argmax (q == nullptr: argmax only)
        if (q != nullptr) {
            std::memset(q, 0, sizeof(float) * V_);
            q[bi] = 1.0f;
        }
        return bi;
    }
    const double inv_t = 1.0 / temperature;
    const double m = static_cast<double>(bv) * inv_t;
    pool_->run([&](int tid, int n) {
        const int lo = static_cast<int>(static_cast<int64_t>(V_) * tid / n);
        const int hi = static_cast<int>(static_cast<int64_t>(V_) * (tid + 1) / n);
        double s = 0.0;
        for (int i = lo; i < hi; ++i) s += std::exp(static_cast<double>(lg[i]) * inv_t - m);
        sums[tid] = s;
    });
    double tot = 0.0;
    for (double s : sums) tot += s;
    const double inv = 1.0 / tot;
    pool_->run([&](int tid, int n) {
        const int lo = static_cast<int>(static_cast<int64_t>(V_) * tid / n);
        const int hi = static_cast<int>(static_cast<int64_t>(V_) * (tid + 1) / n);
        for (int i = lo; i < hi; ++i)
            q[i] = static_cast<float>(std::exp(static_cast<double>(lg[i]) * inv_t - m) * inv);
    });
    return bi;
}

int CpuLlama::sample(const float* q, double u) {
    const int nt = pool_->size();
    std::vector<double> sums(nt, 0.0);
    std::vector<int> last(nt, -1);
    pool_->run([&](int tid, int n) {
        const int lo = static_cast<int>(static_cast<int64_t>(V_) * tid / n);
        const int hi = static_cast<int>(static_cast<int64_t>(V_) * (tid + 1) / n);
        double acc = 0.0;
        int ls = -1;
        for (int i = lo; i < hi; ++i)
            if (q[i] > 0.0f) {
                acc += q[i];
                ls = i;
            }
        sums[tid] = acc;
        last[tid] = ls;
    });
    double prefix = 0.0;
    int last_support = 0;
    for (int t = 0; t < nt; ++t) {
        if (last[t] >= 0) last_support = last[t];
        if (sums[t] > 0.0 && u < prefix + sums[t]) {
            const int lo = static_cast<int>(static_cast<int64_t>(V_) * t / nt);
            const int hi = static_cast<int>(static_cast<int64_t>(V_) * (t + 1) / nt);
            double acc = prefix;
            for (int i = lo; i < hi; ++i) {
                if (!(q[i] > 0.0f)) continue;
                acc += q[i];
                if (u < acc) return i;
            }
            return last[t];
        }
        prefix += sums[t];
    }
    return last_support;  // u in the rounding slack past the accumulated mass
}

void CpuLlama::top_k(const float* q, int k, int32_t* out) {
    // partial selection keeping "descending probability, then ascending id"
    // (ranked_tokens, proj/src/distribution.cpp:80-87) without a full sort
    const int nt = pool_->size();
    std::vector<std::vector<int32_t>> part(nt);
    auto better = [&](int32_t a, int32_t b) { return q[a] > q[b] || (q[a] == q[b] && a < b); };
    pool_->run([&](int tid, int n) {
        const int lo = static_cast<int>(static_cast<int64_t>(V_) * tid / n);
        const int hi = static_cast<int>(static_cast<int64_t>(V_) * (tid + 1) / n);
        std::vector<int32_t>& p = part[tid];
        p.clear();
        for (int i = lo; i < hi; ++i) {
            if (static_cast<int>(p.size()) < k) {
                p.push_back(i);
                std::push_heap(p.begin(), p.end(), better);  // heap top = worst kept
            } else if (better(i, p.front())) {
                std::pop_heap(p.begin(), p.end(), better);
                p.back() = i;
                std::push_heap(p.begin(), p.end(), better);
            }
        }
    });
    std::vector<int32_t> all;
    for (auto& p : part) all.insert(all.end(), p.begin(), p.end());
    std::sort(all.begin(), all.end(), better);
    for (int i = 0; i < k; ++i) out[i] = all[i];
}

}  // namespace dd

// ------------------------------------------------------------------ C ABI
extern "C" {

int dd_draft_create(const dd_model_desc* desc, uint64_t weight_seed, const dd_plant_desc* plant,
                    int n_threads, const int* cpus, int n_cpus, dd_draft** out) {
    if (!desc || !out) return DD_E_ARG;
    *out = nullptr;
    if (!__builtin_cpu_supports("avx512vnni") || !__builtin_cpu_supports("avx512bw"))
        return DD_E_ARG;  // single native path: AVX-512 VNNI
    const dd_model_desc& d = *desc;
    if (d.n_layers < 1 || d.d_model % 32 || d.ffn_dim % 32 || d.head_dim > 256 || d.max_seq < 2 ||
        d.n_heads % std::max(1, d.n_kv_heads))
        return DD_E_ARG;
    std::vector<int> cl;
    for (int i = 0; i < n_cpus; ++i) cl.push_back(cpus[i]);
    int nt = n_threads;
    if (nt <= 0) nt = !cl.empty() ? static_cast<int>(cl.size())
                                  : std::max(1, static_cast<int>(std::thread::hardware_concurrency()) - 2);
    auto* dr = new dd_draft();
    dr->cpus = cl;
    dr->model = std::make_unique<dd::CpuLlama>(d, weight_seed, plant, nt, cl);
    *out = dr;
    return DD_OK;
}

void dd_draft_destroy(dd_draft* d) { delete d; }

int dd_draft_logits(dd_draft* d, const int32_t* ctx_tokens, int n, float* logits) {
    if (!d || !ctx_tokens || !logits) return DD_E_ARG;
    return d->model->logits(ctx_tokens, n, logits) ? DD_OK : DD_E_ARG;
}

int dd_draft_time_token(dd_draft* d, int trials, float* median_ms) {
    if (!d || !median_ms || trials < 1) return DD_E_ARG;
    // calibrate()'s denominator: the cost of one single-token forward
    // (engine.cpp:559-561), measured the way drafting runs them - a run of 8
    // consecutive tokens after an 8-token context, per-token mean - so the pool
    // threads are as warm as in draft_dynamic; median over the trials
    constexpr int kRun = 8;
    std::vector<int32_t> ctx(8 + kRun, 0);
    std::vector<float> lg(d->model->vocab());
    std::vector<double> ms;
    for (int i = 0; i < 3 + trials; ++i) {
        for (int j = 0; j < kRun; ++j) ctx[8 + j] = (i * kRun + j) % 7 + 1;
        d->model->logits(ctx.data(), 8, lg.data());  // cache holds 8 tokens
        const auto t0 = std::chrono::steady_clock::now();
        for (int j = 1; j <= kRun; ++j) d->model->logits(ctx.data(), 8 + j, lg.data());  // one new token each
        const double x =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / kRun;
        if (i >= 3) ms.push_back(x);
    }
    std::sort(ms.begin(), ms.end());
    const size_t n = ms.size();
    *median_ms = static_cast<float>(n % 2 ? ms[n / 2] : 0.5 * (ms[n / 2 - 1] + ms[n / 2]));
    return DD_OK;
}

}  // extern "C"
