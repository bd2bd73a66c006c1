// Host decoding engine: run_vanilla / run_sps / run_duo over the GPU target
// (dd_ctx) and the CPU draft (dd_draft), restating the reference loop
// (proj/src/engine.cpp:273-512) with the verification on the device.
//
// Target-side state machine: the KV cache always holds
// every verified token except the last committed one, c; each scored pass is
// [c] ++ tail (W = 1 + L) and after verification the cache is truncated to
// |verified| - 1 (KV rollback of a rejected tail).  Draft side: draft_dynamic
// (proj/src/drafting.cpp:71-136) on host cores in a concurrent worker thread
// (engine.cpp:425-440) exchanging one request/reply per iteration through a
// lock-free single-slot channel (replacing the mutex/condvar DuoChannel,
// engine.cpp:162-226).  RNG draw order per role is the reference's, so the
// threaded and sequential executions emit identical tokens.
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/duodec_b200.h"
#include "draft.h"

#include "ctx.h"

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct EngineError : std::runtime_error {
    int code;
    EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(int rc, dd_ctx* ctx) {
    if (rc != DD_OK) throw EngineError(rc, dd_last_error(ctx));
}

void jitter(const dd_engine_config& c, int iter, int role);

// RandomStream (proj/include/duodec/random.hpp:11-34)
struct Rng {
    uint64_t seed = 0, counter = 0;
    uint64_t next_u64() {
        uint64_t z = seed + (++counter) * 0x9e3779b97f4a7c15ULL;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
};

// sample() over fp32 probabilities (proj/src/distribution.cpp:61-78)
int sample_f32(const float* p, int V, double u) {
    double acc = 0.0;
    int last = 0;
    for (int i = 0; i < V; ++i) {
        const double v = p[i];
        if (v <= 0.0) continue;
        acc += v;
        last = i;
        if (u < acc) return i;
    }
    return last;
}

struct DraftSeq {
    std::vector<int32_t> tokens;
    std::vector<std::vector<float>> dists;  // empty rows when greedy (one-hot)
};

struct Bundle {
    std::vector<DraftSeq> seqs;
    double threshold = 0.0;
    int forwards = 0;
    double ms = 0.0;
};

// Draft-side q(ctx) with the draft's temperature / greedy rule applied.
struct DraftModel {
    dd::CpuLlama* m;
    double temperature;
    bool greedy;
    std::vector<float> lg;
    int V;
    explicit DraftModel(dd::CpuLlama* mm, double t, bool g)
        : m(mm), temperature(t), greedy(g), lg(mm->vocab()), V(mm->vocab()) {}
    // fills q (fp32 V) and returns the argmax
    int dist(const std::vector<int32_t>& ctx, float* q) {
        if (!m->logits(ctx.data(), static_cast<int>(ctx.size()), lg.data()))
            throw EngineError(DD_E_ARG, m->err);
        return m->distribution(lg.data(), temperature, greedy, q);
    }
};

// draft_dynamic (proj/src/drafting.cpp:71-136): probe step, rank-ordered
// branch admission above theta = p_top * p_second, even budget split with the
// remainder on the top sequence, sampled continuation (rng draws in
// sequence-major order), probe reused for the top sequence's second token.
Bundle draft_dynamic(DraftModel& dm, const std::vector<int32_t>& context, int budget,
                     int max_sequences, Rng& rng) {
    const auto t0 = Clock::now();
    const int V = dm.V;
    Bundle b;
    // greedy: the distributions are one-hot at the argmax, so only the argmax is
    // computed (no V-wide q rows to fill: p_top = probe[a2] = 1)
    std::vector<float> first(dm.greedy ? 0 : V), probe(dm.greedy ? 0 : V);
    const int top = dm.dist(context, dm.greedy ? nullptr : first.data());
    const int s_cap = std::min(max_sequences, budget);
    std::vector<int32_t> ranks(std::min(V, s_cap + 1));
    if (dm.greedy) {
        ranks[0] = top;  // one-hot: no other rank has positive mass
    } else {
        dm.m->top_k(first.data(), static_cast<int>(ranks.size()), ranks.data());
    }
    const double p_top = dm.greedy ? 1.0 : first[top];
    std::vector<int32_t> pctx = context;
    pctx.push_back(top);
    const int a2 = dm.dist(pctx, dm.greedy ? nullptr : probe.data());
    b.threshold = p_top * (dm.greedy ? 1.0 : static_cast<double>(probe[a2]));
    b.forwards = 2;
    std::vector<int32_t> firsts{top};
    if (!dm.greedy) {
        for (size_t r = 1; r < ranks.size() && static_cast<int>(firsts.size()) < s_cap; ++r) {
            if (!(static_cast<double>(first[ranks[r]]) > b.threshold)) break;
            firsts.push_back(ranks[r]);
        }
    }
    const int s = static_cast<int>(firsts.size());
    const int base = budget / s, rem = budget - base * s;
    std::vector<float> d(dm.greedy ? 0 : V);
    for (int i = 0; i < s; ++i) {
        const int len = base + (i == 0 ? rem : 0);
        DraftSeq seq;
        seq.tokens.push_back(firsts[i]);
        seq.dists.push_back(dm.greedy ? std::vector<float>() : first);
        std::vector<int32_t> ctx = context;
        ctx.push_back(firsts[i]);
        for (int pos = 1; pos < len; ++pos) {
            const bool reuse = (i == 0 && pos == 1);
            int am;
            const float* dp;
            if (reuse) {
                am = a2;
                dp = probe.data();
            } else {
                am = dm.dist(ctx, dm.greedy ? nullptr : d.data());
                ++b.forwards;
                dp = d.data();
            }
            const double u = rng.next_uniform();
            const int t = dm.greedy ? am : dm.m->sample(dp, u);
            seq.tokens.push_back(t);
            seq.dists.push_back(dm.greedy ? std::vector<float>() : std::vector<float>(dp, dp + V));
            ctx.push_back(t);
        }
        b.seqs.push_back(std::move(seq));
    }
    b.ms = ms_since(t0);
    return b;
}

// Single-slot lock-free rendezvous: prefix down, bundle up (one pair per iteration).
struct Channel {
    std::atomic<int> state{0};  // 0 idle, 1 request posted, 2 reply posted, 3 stop
    std::vector<int32_t> z;
    Bundle reply;
    std::exception_ptr error;
    std::atomic<bool> failed{false};

    void post_request(std::vector<int32_t> zz) {
        z = std::move(zz);
        state.store(1, std::memory_order_release);
    }
    bool wait_request() {  // worker side
        for (;;) {
            const int s = state.load(std::memory_order_acquire);
            if (s == 1) return true;
            if (s == 3) return false;
            _mm_pause();
        }
    }
    void post_reply(Bundle b) {
        reply = std::move(b);
        int expect = 1;  // a concurrent stop() wins
        state.compare_exchange_strong(expect, 2, std::memory_order_acq_rel);
    }
    Bundle wait_reply() {
        for (;;) {
            if (failed.load(std::memory_order_acquire)) std::rethrow_exception(error);
            if (state.load(std::memory_order_acquire) == 2) break;
            _mm_pause();
        }
        state.store(0, std::memory_order_relaxed);
        return std::move(reply);
    }
    void stop() { state.store(3, std::memory_order_release); }
};

struct Runner {
    dd_ctx* ctx;                // rank 0: acceptance, timing
    std::vector<dd_ctx*> ranks;  // every tensor-parallel rank (ranks[0] == ctx)
    dd_draft* draft;
    dd_engine_config cfg;
    int V = 0;
    int budget = 0;
    std::vector<int32_t> verified;
    std::optional<DraftSeq> tail;
    Rng rng_draft, rng_verify;
    size_t prompt_len = 0;
    std::vector<dd_iteration_record> recs;
    Clock::time_point t_start;
    double ttft = 0.0;
    // Prompt suffix not yet in the cache (ends with c): the first scored pass of
    // vanilla / duo covers it, so the target's forward over the prompt yields
    // iteration 1's distribution directly instead of a prefill plus a
    // one-token pass (the reference's iteration 1 scores the whole prefix).
    std::vector<int32_t> pending;

    int c_token() const { return verified.back(); }

    std::vector<int32_t> first_pass() {
        std::vector<int32_t> p;
        if (pending.empty()) {
            p.push_back(c_token());
        } else {
            p.swap(pending);
        }
        return p;
    }

    // Every rank runs the same passes; each call only enqueues (the ranks'
    // reductions meet on the devices), so issuing them in rank order is safe.
    void score(const std::vector<int32_t>& pass) {
        for (dd_ctx* r : ranks) ck(dd_score(r, pass.data(), static_cast<int>(pass.size())), r);
    }
    void truncate_all(int n) {
        for (dd_ctx* r : ranks) ck(dd_kv_truncate(r, n), r);
    }
    void prefill(const int32_t* tokens, int n) {
        if (ranks.size() == 1) {  // dd_prefill picks the pass sizes (one pass for a long prompt)
            ck(dd_prefill(ctx, tokens, n), ctx);
            return;
        }
        for (int i = 0; i < n; i += dd::kPrefillChunk) {  // chunk-major: no rank runs ahead
            const int w = std::min(dd::kPrefillChunk, n - i);
            for (dd_ctx* r : ranks) ck(dd_prefill(r, tokens + i, w), r);
        }
    }
    void truncate_cache() { truncate_all(static_cast<int>(verified.size()) - 1); }

    void record(dd_iteration_record r) {
        recs.push_back(r);
        if (recs.size() == 1) {
            ttft = ms_since(t_start);
            ck(ctx_mark(ctx, 2), ctx);
        }
    }

    dd_verify_out verify(int mode, int L, const std::vector<int32_t>& firsts, bool q_onehot) {
        dd_verify_args a{};
        a.mode = mode;
        a.tail_len = L;
        a.n_firsts = static_cast<int>(std::min<size_t>(firsts.size(), 16));
        for (int i = 0; i < a.n_firsts; ++i) a.firsts[i] = firsts[i];
        a.seed = rng_verify.seed;
        a.counter = rng_verify.counter;
        a.temperature = cfg.temperature;
        a.greedy = cfg.greedy;
        a.q_onehot = q_onehot ? 1 : 0;
        dd_verify_out o{};
        ck(dd_verify(ctx, &a, &o), ctx);
        rng_verify.counter = o.counter_out;
        return o;
    }

    void upload_rows(const std::vector<std::vector<float>>& rows, size_t from) {
        if (cfg.greedy || rows.size() <= from) return;
        std::vector<float> flat;
        flat.reserve((rows.size() - from) * V);
        for (size_t i = from; i < rows.size(); ++i) flat.insert(flat.end(), rows[i].begin(), rows[i].end());
        ck(dd_upload_q(ctx, flat.data(), static_cast<int>(rows.size() - from), V), ctx);
    }

    void run_vanilla() {  // engine.cpp:273-312
        while (verified.size() - prompt_len < static_cast<size_t>(cfg.max_new_tokens)) {
            const auto t0 = Clock::now();
            score(first_pass());
            const dd_verify_out o = verify(DD_MODE_VANILLA, 0, {}, true);
            verified.push_back(o.next_token);
            truncate_cache();
            dd_iteration_record r{};
            r.target_ms = ms_since(t0);
            r.tokens_processed = 1;
            r.width = 1;
            record(r);
        }
    }

    void run_sps(DraftModel& dm) {  // engine.cpp:314-393
        std::vector<float> q(V);
        while (verified.size() - prompt_len < static_cast<size_t>(cfg.max_new_tokens)) {
            const auto td = Clock::now();
            std::vector<int32_t> toks;
            std::vector<std::vector<float>> dists;
            std::vector<int32_t> c2 = verified;
            for (int k = 0; k < budget; ++k) {
                const int am = dm.dist(c2, q.data());
                const double u = rng_draft.next_uniform();
                const int t = cfg.greedy ? am : dm.m->sample(q.data(), u);
                toks.push_back(t);
                if (!cfg.greedy) dists.push_back(q);
                c2.push_back(t);
            }
            const double draft_ms = ms_since(td);
            const auto tt = Clock::now();
            upload_rows(dists, 0);
            std::vector<int32_t> pass{c_token()};
            pass.insert(pass.end(), toks.begin(), toks.end());
            score(pass);
            const dd_verify_out o = verify(DD_MODE_SPS, budget, {}, cfg.greedy);
            verified.insert(verified.end(), toks.begin(), toks.begin() + o.sps_accepted);
            verified.push_back(o.next_token);
            truncate_cache();
            dd_iteration_record r{};
            r.draft_ms = draft_ms;
            r.target_ms = ms_since(tt);
            r.tokens_processed = o.sps_accepted + 1;
            r.sequence_count = 1;
            r.accepted = o.sps_accepted;
            r.width = budget + 1;
            record(r);
        }
    }

    void run_duo(DraftModel& dm) {  // engine.cpp:395-512
        Channel ch;
        std::thread worker;
        const bool threaded = cfg.threaded != 0;
        if (threaded) {
            // The worker must start on its own core: a thread inherits its creator's
            // affinity, and the creator (the target-role thread, typically pinned to
            // one core) spins in wait_reply, so a worker born on that core would only
            // run after a scheduler tick (~ms of lost draft time in iteration 1, i.e.
            // TTFT).  Create it with the draft core's affinity instead.
            cpu_set_t saved;
            const bool pin = !draft->cpus.empty() &&
                             pthread_getaffinity_np(pthread_self(), sizeof(saved), &saved) == 0;
            if (pin) {
                cpu_set_t set;
                CPU_ZERO(&set);
                CPU_SET(draft->cpus[0], &set);
                pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
            }
            worker = std::thread([&] {
                if (!draft->cpus.empty()) {  // the worker is pool thread 0
                    cpu_set_t set;
                    CPU_ZERO(&set);
                    CPU_SET(draft->cpus[0], &set);
                    pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
                }
                try {
                    for (int it = 0; ch.wait_request(); ++it) {
                        jitter(cfg, it, 0);
                        ch.post_reply(draft_dynamic(dm, ch.z, budget, cfg.max_sequences, rng_draft));
                    }
                } catch (...) {
                    ch.error = std::current_exception();
                    ch.failed.store(true, std::memory_order_release);
                }
            });
            if (pin) pthread_setaffinity_np(pthread_self(), sizeof(saved), &saved);
        }
        try {
            while (verified.size() - prompt_len < static_cast<size_t>(cfg.max_new_tokens)) {
                // both roles start from the identical prefix verified ++ tail
                std::vector<int32_t> z = verified;
                const int L = tail ? static_cast<int>(tail->tokens.size()) : 0;
                if (tail) z.insert(z.end(), tail->tokens.begin(), tail->tokens.end());
                std::vector<int32_t> pass = first_pass();
                if (tail) pass.insert(pass.end(), tail->tokens.begin(), tail->tokens.end());
                Bundle bundle;
                const auto tt = Clock::now();
                double comm = 0.0;
                const int it = static_cast<int>(recs.size());
                if (threaded) {
                    ch.post_request(std::move(z));
                    jitter(cfg, it, 1);
                    score(pass);
                    const auto tw = Clock::now();
                    bundle = ch.wait_reply();  // rendezvous
                    comm = ms_since(tw);
                } else {
                    jitter(cfg, it, 0);
                    bundle = draft_dynamic(dm, z, budget, cfg.max_sequences, rng_draft);
                    jitter(cfg, it, 1);
                    score(pass);
                }
                const auto tv = Clock::now();
                std::vector<int32_t> firsts;
                for (auto& s : bundle.seqs) firsts.push_back(s.tokens[0]);
                const dd_verify_out o = verify(DD_MODE_DUO, L, firsts, cfg.greedy);
                const double target_ms = ms_since(tt);
                // apply_verification (engine.cpp:62-106)
                int committed = 0, accepted = 0;
                bool usable = true;
                if (tail) {
                    if (o.prefix_all_accepted) {
                        verified.insert(verified.end(), tail->tokens.begin(), tail->tokens.end());
                        committed += L;
                        accepted += L;
                    } else {
                        verified.insert(verified.end(), tail->tokens.begin(),
                                        tail->tokens.begin() + o.reject_index);
                        verified.push_back(o.resample);
                        committed += o.reject_index + 1;
                        accepted += o.reject_index;
                        usable = false;
                    }
                    tail.reset();
                }
                if (usable) {
                    if (o.bundle_accepted) {
                        DraftSeq& seq = bundle.seqs[static_cast<size_t>(o.seq_index)];
                        verified.push_back(seq.tokens[0]);
                        committed += 1;
                        accepted += 1;
                        if (seq.tokens.size() > 1) {  // tail_of (engine.cpp:45-51)
                            DraftSeq t;
                            t.tokens.assign(seq.tokens.begin() + 1, seq.tokens.end());
                            if (!cfg.greedy) t.dists.assign(seq.dists.begin() + 1, seq.dists.end());
                            tail = std::move(t);
                        }
                    } else {
                        verified.push_back(o.fallback);
                        committed += 1;
                    }
                }
                truncate_cache();
                if (tail) upload_rows(tail->dists, 0);  // overlaps the next pass
                dd_iteration_record r{};
                r.draft_ms = bundle.ms;
                r.target_ms = target_ms;
                r.verify_ms = ms_since(tv);
                r.comm_ms = comm;
                r.tokens_processed = committed;
                r.sequence_count = static_cast<int>(bundle.seqs.size());
                r.accepted = accepted;
                r.width = L + 1;
                record(r);
            }
        } catch (...) {
            if (threaded) {
                ch.stop();
                worker.join();
            }
            throw;
        }
        if (threaded) {
            ch.stop();
            worker.join();
        }
    }
};

// WorkerHooks jitter (engine.hpp:36-41): role 0 = before_draft, 1 = before_target
void jitter(const dd_engine_config& c, int iter, int role) {
    if (c.jitter_max_us <= 0) return;
    uint64_t z = c.jitter_seed + (2ull * static_cast<uint64_t>(iter) + role + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z ^= z >> 31;
    std::this_thread::sleep_for(
        std::chrono::microseconds(z % (static_cast<uint64_t>(c.jitter_max_us) + 1)));
}

int choose_budget_impl(double c) { return static_cast<int>(std::max<long>(2, std::lround(c))); }

}  // namespace

extern "C" {

int dd_calibrate(dd_ctx* ctx, dd_draft* draft, int probe_len, int trials, int hard_cap,
                 double* cost_coefficient, int* budget) {
    // calibrate (engine.cpp:534-578): median target scored pass at probe_len
    // (CUDA events) over the median single-token CPU draft forward
    if (!ctx || !draft || !cost_coefficient || !budget) return DD_E_ARG;
    if (trials < 10 || probe_len < 1) return DD_E_ARG;
    float t_ms = 0.0f, d_ms = 0.0f;
    int n0 = 0;
    dd_kv_len(ctx, &n0);
    if (n0 < probe_len) {
        std::vector<int32_t> probe(static_cast<size_t>(probe_len - n0), 0);
        int rc = dd_prefill(ctx, probe.data(), static_cast<int>(probe.size()));
        if (rc) return rc;
    }
    int rc = dd_time_pass(ctx, probe_len, trials + 5, &t_ms);
    if (rc) return rc;
    dd_kv_truncate(ctx, n0);
    {
        // time the draft where run_duo runs it: pool thread 0 on the draft's
        // first core (the caller may be pinned to the target-role core)
        cpu_set_t saved;
        const bool pin = !draft->cpus.empty() &&
                         pthread_getaffinity_np(pthread_self(), sizeof(saved), &saved) == 0;
        if (pin) {
            cpu_set_t set;
            CPU_ZERO(&set);
            CPU_SET(draft->cpus[0], &set);
            pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
        }
        // measure the draft in steady state, as run_duo runs it: the first
        // ~second of drafting after the draft's creation runs up to 40% slower
        // on the pool's hosts (clocks, caches), so keep drafting for 1 s first
        // (once per draft: later calibrations reuse the warmed state)
        const auto t_warm = std::chrono::steady_clock::now();
        if (!draft->calib_warmed) {
            do {
                rc = dd_draft_time_token(draft, trials, &d_ms);
            } while (rc == DD_OK &&
                     std::chrono::steady_clock::now() - t_warm < std::chrono::seconds(1));
            draft->calib_warmed = rc == DD_OK;
        }
        if (rc == DD_OK) rc = dd_draft_time_token(draft, trials, &d_ms);
        if (pin) pthread_setaffinity_np(pthread_self(), sizeof(saved), &saved);
    }
    if (rc) return rc;
    if (d_ms < 1e-6f) return DD_E_STATE;  // DegenerateTiming
    *cost_coefficient = static_cast<double>(t_ms) / static_cast<double>(d_ms);
    *budget = std::min(choose_budget_impl(*cost_coefficient), hard_cap);
    return DD_OK;
}

static int engine_run(const std::vector<dd_ctx*>& ranks, dd_draft* draft,
                      const dd_engine_config* cfg, const int32_t* prompt, int n_prompt,
                      dd_generation_result* out) {
    dd_ctx* ctx = ranks[0];
    if (!ctx || !cfg || !prompt || !out || n_prompt < 1) return DD_E_ARG;
    const dd_engine_config& c = *cfg;
    // EngineConfig::validate (engine.cpp:230-249); greedy replaces T > 0
    if (c.budget < 2 || c.budget > c.budget_hard_cap || c.max_sequences < 1 ||
        c.max_new_tokens < 1 || (!c.greedy && !(c.temperature > 0.0)) ||
        (c.budget_policy == DD_BUDGET_CALIBRATED && c.calib_trials < 10) ||
        c.mode < DD_MODE_DUO || c.mode > DD_MODE_VANILLA)
        return ctx_fail(ctx, DD_E_ARG, "invalid engine configuration");
    if (c.mode != DD_MODE_VANILLA && !draft)
        return ctx_fail(ctx, DD_E_ARG, "sps/duo mode requires a draft model");
    // run_sps / run_duo throw ConfigError on a vocabulary mismatch (the
    // acceptance kernel reads q rows at the target's vocabulary stride)
    if (c.mode != DD_MODE_VANILLA)
        for (dd_ctx* k : ranks)
            if (!k || draft->model->vocab() != k->vocab)
                return ctx_fail(ctx, DD_E_ARG, "draft and target vocabularies differ");
    // dd_verify tests at most 16 bundle sequences (verify_bundle's draw
    // schedule would silently lose the rest)
    if (c.max_sequences > 16)
        return ctx_fail(ctx, DD_E_ARG, "max_sequences above the verifier's 16-sequence bundle");
    if (ranks.size() > 1 && c.mode != DD_MODE_VANILLA && c.budget_policy == DD_BUDGET_CALIBRATED)
        return ctx_fail(ctx, DD_E_ARG, "a tensor-parallel group needs a fixed budget");
    Runner r;
    r.ctx = ctx;
    r.ranks = ranks;
    r.draft = draft;
    r.cfg = c;
    try {
        r.budget = c.budget;
        // the reference starts the timeline before resolve_budget
        // (engine.cpp:444-456), so total_ms / ttft_ms / tps include calibration
        r.t_start = Clock::now();
        if (c.mode != DD_MODE_VANILLA && c.budget_policy == DD_BUDGET_CALIBRATED) {
            double coef = 0.0;
            ck(dd_kv_truncate(ctx, 0), ctx);
            ck(dd_calibrate(ctx, draft, c.calib_probe_len, c.calib_trials, c.budget_hard_cap,
                            &coef, &r.budget),
               ctx);
        }
        if (c.mode == DD_MODE_SPS && r.budget + 1 > 256) return DD_E_CAPACITY;
        r.V = draft ? draft->model->vocab() : 0;
        r.verified.assign(prompt, prompt + n_prompt);
        r.prompt_len = static_cast<size_t>(n_prompt);
        r.rng_draft.seed = c.draft_seed;
        r.rng_verify.seed = c.verify_seed;
        for (dd_ctx* k : ranks) k->h2d_bytes = k->d2h_bytes = k->launches = 0;
        ck(ctx_mark(ctx, 0), ctx);
        r.truncate_all(0);
        // SpS drafts before its first pass, so its prefill (overlapping that
        // drafting) stops before c; vanilla and duo score the last prefill chunk.
        int keep = 1;
        if (c.mode != DD_MODE_SPS) keep = (n_prompt - 1) % dd::kPrefillChunk + 1;
        if (n_prompt > keep) r.prefill(prompt, n_prompt - keep);
        if (keep > 1) r.pending.assign(prompt + n_prompt - keep, prompt + n_prompt);
        out->prefill_ms = 0.0;
        if (c.mode == DD_MODE_VANILLA) {
            r.run_vanilla();
        } else {
            DraftModel dm(draft->model.get(), c.temperature, c.greedy != 0);
            if (c.mode == DD_MODE_SPS) {
                r.run_sps(dm);
            } else {
                r.run_duo(dm);
            }
        }
        const double total = ms_since(r.t_start);
        ck(ctx_mark(ctx, 1), ctx);
        out->device_ms = ctx_elapsed_ms(ctx, 1);
        out->device_ttft_ms = ctx_elapsed_ms(ctx, 2);
        out->h2d_bytes = sizeof(int32_t) * static_cast<uint64_t>(n_prompt);
        out->d2h_bytes = 0;
        out->gpu_launches = 0;
        for (dd_ctx* k : ranks) {
            out->h2d_bytes += k->h2d_bytes;
            out->d2h_bytes += k->d2h_bytes;
            out->gpu_launches += k->launches;
        }
        const size_t gen = r.verified.size() - r.prompt_len;
        out->n_tokens = static_cast<int>(gen);
        for (size_t i = 0; i < gen && static_cast<int>(i) < out->max_tokens; ++i)
            out->tokens[i] = r.verified[r.prompt_len + i];
        out->n_iterations = static_cast<int>(r.recs.size());
        for (size_t i = 0; i < r.recs.size() && static_cast<int>(i) < out->max_iterations; ++i)
            out->iterations[i] = r.recs[i];
        out->ttft_ms = r.ttft;
        out->total_ms = total;
        out->tps = total > 0.0 ? static_cast<double>(gen) / (total / 1000.0) : 0.0;  // engine.cpp:117-122
        out->budget_used = r.budget;
        return DD_OK;
    } catch (const EngineError& e) {
        return ctx_fail(ctx, e.code, e.what());
    } catch (const std::exception& e) {
        return ctx_fail(ctx, DD_E_STATE, e.what());
    }
}

int dd_engine_run(dd_ctx* ctx, dd_draft* draft, const dd_engine_config* cfg,
                  const int32_t* prompt, int n_prompt, dd_generation_result* out) {
    return engine_run({ctx}, draft, cfg, prompt, n_prompt, out);
}

int dd_draft_dist(dd_draft* d, const int32_t* ctx_tokens, int n, double temperature, int greedy,
                  float* q, int* argmax) {
    if (!d || !ctx_tokens || n < 1 || !q || !argmax || (!greedy && !(temperature > 0.0)))
        return DD_E_ARG;
    try {
        DraftModel dm(d->model.get(), temperature, greedy != 0);
        *argmax = dm.dist(std::vector<int32_t>(ctx_tokens, ctx_tokens + n), q);
        return DD_OK;
    } catch (const EngineError& e) {
        d->err = e.what();
        return e.code;
    }
}

int dd_draft_dynamic(dd_draft* d, const int32_t* ctx_tokens, int n, int budget,
                     int max_sequences, double temperature, int greedy, uint64_t seed,
                     uint64_t* counter, int32_t* tokens, int32_t* seq_len, int* n_seqs,
                     double* threshold, int* forwards) {
    if (!d || !ctx_tokens || n < 1 || !counter || !tokens || !seq_len || !n_seqs || !threshold ||
        !forwards || budget < 1 || max_sequences < 1 || (!greedy && !(temperature > 0.0)))
        return DD_E_ARG;
    try {
        DraftModel dm(d->model.get(), temperature, greedy != 0);
        Rng rng;
        rng.seed = seed;
        rng.counter = *counter;
        Bundle b = draft_dynamic(dm, std::vector<int32_t>(ctx_tokens, ctx_tokens + n), budget,
                                 max_sequences, rng);
        int k = 0;
        for (size_t i = 0; i < b.seqs.size(); ++i) {
            seq_len[i] = static_cast<int32_t>(b.seqs[i].tokens.size());
            for (int32_t t : b.seqs[i].tokens) tokens[k++] = t;
        }
        *n_seqs = static_cast<int>(b.seqs.size());
        *threshold = b.threshold;
        *forwards = b.forwards;
        *counter = rng.counter;
        return DD_OK;
    } catch (const EngineError& e) {
        d->err = e.what();
        return e.code;
    }
}

int dd_engine_run_tp(dd_ctx* const* ctxs, int n, dd_draft* draft, const dd_engine_config* cfg,
                     const int32_t* prompt, int n_prompt, dd_generation_result* out) {
    if (!ctxs || n < 1) return DD_E_ARG;
    std::vector<dd_ctx*> ranks(ctxs, ctxs + n);
    for (int i = 0; i < n; ++i)
        if (!ranks[i] || (n > 1 && (ranks[i]->tp_size != n || ranks[i]->tp_rank != i ||
                                    !ranks[i]->tp_connected)))
            return ctx_fail(ranks[i], DD_E_ARG, "ctxs[i] must be connected rank i of the group");
    return engine_run(ranks, draft, cfg, prompt, n_prompt, out);
}

}  // extern "C"
