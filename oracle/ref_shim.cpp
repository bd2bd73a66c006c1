// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library, compiled from
// its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libduodec_ref.so.  Python tests load it with ctypes to pin the
// oracle restatement (oracle/protocol.py) and the GPU acceptance kernel to the
// reference's exact decisions, draw counts and engine outputs.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "duodec/distribution.hpp"
#include "duodec/drafting.hpp"
#include "duodec/engine.hpp"
#include "duodec/fidelity.hpp"
#include "duodec/model.hpp"
#include "duodec/random.hpp"
#include "duodec/verify.hpp"

using namespace duodec;

namespace {
thread_local std::string g_err;

RandomStream stream_at(uint64_t seed, uint64_t counter) {
    RandomStream r(seed);
    for (uint64_t i = 0; i < counter; ++i) (void)r.next_u64();  // no counter setter
    return r;
}
Distribution dist(const double* p, int V) {
    return Distribution::unchecked(std::vector<double>(p, p + V));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rng_u64(uint64_t seed, uint64_t skip, int n, uint64_t* out) {
    RandomStream r = stream_at(seed, skip);
    for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform(uint64_t seed, uint64_t skip, int n, double* out) {
    RandomStream r = stream_at(seed, skip);
    for (int i = 0; i < n; ++i) out[i] = r.next_uniform();
}
uint64_t ref_derive_seed(uint64_t base, uint64_t index) { return derive_seed(base, index); }

int ref_sample(const double* p, int V, double u) { return sample(dist(p, V), u); }
int ref_argmax(const double* p, int V) { return argmax(dist(p, V)); }
int ref_accept_test(double p, double q, double r) { return accept_test(p, q, r) ? 1 : 0; }

// residual(); returns 0 ok, 1 ZeroMassError
int ref_residual(const double* p, const double* q, int V, double* out) {
    try {
        Distribution d = residual(dist(p, V), dist(q, V));
        std::memcpy(out, d.probs().data(), sizeof(double) * V);
        return 0;
    } catch (const ZeroMassError&) {
        return 1;
    }
}

// verify_prefix: tail tokens[L], q rows [L][V], p rows [L][V]
void ref_verify_prefix(const int32_t* toks, const double* q_rows, const double* p_rows, int L,
                       int V, uint64_t seed, uint64_t counter, int* all_accepted,
                       int* reject_index, int* resample, uint64_t* counter_out) {
    DraftSequence tail;
    std::vector<Distribution> target;
    for (int j = 0; j < L; ++j) {
        tail.tokens.push_back(toks[j]);
        tail.dists.push_back(dist(q_rows + static_cast<size_t>(j) * V, V));
        target.push_back(dist(p_rows + static_cast<size_t>(j) * V, V));
    }
    if (L > 0) tail.first_token_prob = tail.dists[0][static_cast<size_t>(toks[0])];
    RandomStream r = stream_at(seed, counter);
    PrefixOutcome o = verify_prefix(tail, target, r);
    *all_accepted = o.all_accepted;
    *reject_index = o.reject_index;
    *resample = o.resample;
    *counter_out = r.counter();
}

void ref_verify_bundle(const int32_t* firsts, int s, const double* p_next, int V, uint64_t seed,
                       uint64_t counter, int* accepted, int* seq_index, int* fallback,
                       uint64_t* counter_out) {
    DraftBundle b;
    for (int i = 0; i < s; ++i) {
        DraftSequence seq;
        seq.tokens.push_back(firsts[i]);
        b.sequences.push_back(std::move(seq));
    }
    RandomStream r = stream_at(seed, counter);
    BundleOutcome o = verify_bundle(b, dist(p_next, V), r);
    *accepted = o.accepted;
    *seq_index = o.seq_index;
    *fallback = o.fallback;
    *counter_out = r.counter();
}

void ref_sps_verify(const int32_t* toks, const double* q_rows, const double* p_rows, int L, int V,
                    uint64_t seed, uint64_t counter, int* accepted, int* next_token,
                    uint64_t* counter_out) {
    std::vector<Distribution> q, p;
    for (int j = 0; j < L; ++j) q.push_back(dist(q_rows + static_cast<size_t>(j) * V, V));
    for (int j = 0; j <= L; ++j) p.push_back(dist(p_rows + static_cast<size_t>(j) * V, V));
    RandomStream r = stream_at(seed, counter);
    SpsResult o = sps_verify(std::span<const Token>(toks, static_cast<size_t>(L)), q, p, r);
    *accepted = o.accepted;
    *next_token = o.next_token;
    *counter_out = r.counter();
}

// ---- Markov-model level (text model files, parsed by the reference) ----
void* ref_model_parse(const char* text) {
    try {
        return new ModelSpec(ModelSpec::parse(text));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_model_free(void* m) { delete static_cast<ModelSpec*>(m); }
int ref_model_vocab(void* m) { return static_cast<ModelSpec*>(m)->vocab_size(); }
void ref_model_forward(void* m, const int32_t* ctx, int n, double* out) {
    const auto* ms = static_cast<ModelSpec*>(m);
    const Distribution& d = ms->forward(std::span<const Token>(ctx, static_cast<size_t>(n)));
    std::memcpy(out, d.probs().data(), sizeof(double) * d.size());
}
void* ref_model_with_temperature(void* m, double t) {
    return new ModelSpec(static_cast<ModelSpec*>(m)->with_temperature(t));
}

// draft_dynamic: returns s; fills firsts[s], lens[s], tokens (flattened, budget),
// threshold, forwards, counter_out
int ref_draft_dynamic(void* draft, const int32_t* ctx, int n, int budget, int max_seq,
                      uint64_t seed, uint64_t counter, int32_t* lens, int32_t* tokens,
                      double* first_probs, double* threshold, int* forwards,
                      uint64_t* counter_out) {
    RandomStream r = stream_at(seed, counter);
    DraftBundle b = draft_dynamic(*static_cast<ModelSpec*>(draft),
                                  std::span<const Token>(ctx, static_cast<size_t>(n)), budget,
                                  max_seq, r);
    int off = 0;
    for (int i = 0; i < b.sequence_count(); ++i) {
        const auto& seq = b.sequences[static_cast<size_t>(i)];
        lens[i] = static_cast<int>(seq.size());
        first_probs[i] = seq.first_token_prob;
        for (Token t : seq.tokens) tokens[off++] = t;
    }
    *threshold = b.threshold;
    *forwards = b.forwards_used;
    *counter_out = r.counter();
    return b.sequence_count();
}

// Engine run on a simulated (profile) or wall timeline.
// profile: draft_per_token, base, slope, comm (ignored when wall != 0)
int ref_run(int mode, void* target, void* draft, const int32_t* prompt, int n, int budget,
            int max_sequences, int max_new_tokens, double temperature, uint64_t draft_seed,
            uint64_t verify_seed, int calibrated, int threaded, const double* profile, int wall,
            int32_t* out_tokens, int max_out, int* n_out, double* ttft, double* total,
            double* tps, int* iter_tokens, int* iter_seqs, int* iter_accepted, int max_iters,
            int* n_iters, int* budget_used) {
    try {
        EngineConfig cfg;
        cfg.mode = static_cast<Mode>(mode);
        cfg.budget = budget;
        cfg.max_sequences = max_sequences;
        cfg.max_new_tokens = max_new_tokens;
        cfg.temperature = temperature;
        cfg.draft_seed = draft_seed;
        cfg.verify_seed = verify_seed;
        cfg.budget_policy = calibrated ? BudgetPolicy::calibrated : BudgetPolicy::fixed;
        cfg.duo_execution = threaded ? DuoExecution::threaded : DuoExecution::sequential;
        DeviceProfile prof{profile[0], profile[1], profile[2], profile[3]};
        Timeline tl = wall ? Timeline::wall() : Timeline::simulated(prof);
        if (calibrated && !wall) {
            const double c = calibrate(*static_cast<ModelSpec*>(target),
                                       *static_cast<ModelSpec*>(draft), cfg.calib_probe_len,
                                       cfg.calib_trials, tl);
            *budget_used = std::min(choose_budget(c), cfg.budget_hard_cap);
        } else {
            *budget_used = budget;
        }
        GenerationResult r = run_generation(*static_cast<ModelSpec*>(target),
                                            static_cast<ModelSpec*>(draft),
                                            std::span<const Token>(prompt, static_cast<size_t>(n)),
                                            cfg, tl);
        *n_out = static_cast<int>(r.tokens.size());
        for (int i = 0; i < *n_out && i < max_out; ++i) out_tokens[i] = r.tokens[static_cast<size_t>(i)];
        *ttft = r.ttft_ms;
        *total = r.total_ms;
        *tps = r.tps;
        *n_iters = static_cast<int>(r.iterations.size());
        for (int i = 0; i < *n_iters && i < max_iters; ++i) {
            iter_tokens[i] = r.iterations[static_cast<size_t>(i)].tokens_processed;
            iter_seqs[i] = r.iterations[static_cast<size_t>(i)].sequence_count;
            iter_accepted[i] = r.iterations[static_cast<size_t>(i)].accepted;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

double ref_calibrate_sim(void* target, void* draft, int probe_len, int trials,
                         const double* profile) {
    DeviceProfile prof{profile[0], profile[1], profile[2], profile[3]};
    Timeline tl = Timeline::simulated(prof);
    return calibrate(*static_cast<ModelSpec*>(target), *static_cast<ModelSpec*>(draft), probe_len,
                     trials, tl);
}
int ref_choose_budget(double c) { return choose_budget(c); }

// run_fidelity; returns max TV, fills per-position TV
double ref_run_fidelity(int mode, void* target, void* draft, const int32_t* prompt, int n,
                        int budget, int max_sequences, double temperature, int samples,
                        int positions, double* tv) {
    EngineConfig cfg;
    cfg.budget = budget;
    cfg.max_sequences = max_sequences;
    cfg.temperature = temperature;
    FidelityReport rep = run_fidelity(static_cast<Mode>(mode), *static_cast<ModelSpec*>(target),
                                      static_cast<ModelSpec*>(draft),
                                      std::span<const Token>(prompt, static_cast<size_t>(n)), cfg,
                                      samples, positions);
    for (int i = 0; i < positions; ++i) tv[i] = rep.tv_per_position[static_cast<size_t>(i)];
    return rep.max_tv;
}

}  // extern "C"
