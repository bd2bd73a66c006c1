// gpu_target.hpp — the C++ adapter a maintainer adds to the reference
// (/root/reference/proj) to move its target role onto the B200 path.
//
// It stands in for ModelSpec on the target role of run_duo / run_sps /
// run_vanilla (proj/include/duodec/engine.hpp:102-116): target_step()
// replaces target_step -> scored_with_next -> ModelSpec::forward_scored
// (proj/src/engine.cpp:36-43, 145-157), verify() replaces verify_prefix /
// verify_bundle / sps_verify inside apply_verification (engine.cpp:62-106,
// verify.cpp:41-107) and rollback() replaces the commit/truncate of the
// target's cached prefix.  Only the C ABI of include/duodec_b200.h is used;
// errors surface as the reference's exception types.  Compiled against the
// reference headers by tests/test_integration_adapter.py.
#pragma once

#include <cstdint>
#include <vector>

#include "duodec/engine.hpp"  // ConfigError, EngineConfig
#include "duodec/types.hpp"   // GenerationState, DraftBundle
#include "duodec_b200.h"

namespace duodec_b200 {

class GpuTarget {
public:
    GpuTarget(const dd_model_desc& desc, std::uint64_t weight_seed, int device = 0,
              const dd_plant_desc* plant = nullptr) {
        if (dd_ctx_create(&desc, device, &ctx_) != DD_OK)  // no CPU fallback
            throw duodec::ConfigError(dd_last_error(nullptr));
        if (dd_weights_init(ctx_, weight_seed, plant) != DD_OK) {
            const std::string msg = dd_last_error(ctx_);
            dd_ctx_destroy(ctx_);
            throw duodec::ConfigError(msg);
        }
    }
    ~GpuTarget() { dd_ctx_destroy(ctx_); }
    GpuTarget(const GpuTarget&) = delete;
    GpuTarget& operator=(const GpuTarget&) = delete;

    // Prompt: cache every token but the last (the cache invariant below).
    void prefill(const std::vector<duodec::Token>& prompt) {
        if (prompt.size() > 1) check(dd_prefill(ctx_, to_i32(prompt).data(), static_cast<int>(prompt.size()) - 1));
    }

    // target_step: one scored pass over [c] ++ tail (W = 1 + L); row i is the
    // target distribution after token i (forward_scored rows + p_next).
    void target_step(const duodec::GenerationState& s) {
        std::vector<std::int32_t> pass{static_cast<std::int32_t>(s.verified.back())};
        if (s.unverified)
            for (duodec::Token t : s.unverified->tokens) pass.push_back(static_cast<std::int32_t>(t));
        check(dd_score(ctx_, pass.data(), static_cast<int>(pass.size())));
    }

    // Draft rows of the tail (the q of verify_prefix), uploaded while the pass
    // runs; row t is the draft distribution that produced tail token t.
    void upload_tail_q(const duodec::DraftSequence& tail) {
        if (tail.size() == 0) return;
        const int V = static_cast<int>(tail.dists[0].size());
        std::vector<float> rows(tail.size() * static_cast<std::size_t>(V));
        for (std::size_t t = 0; t < tail.size(); ++t)
            for (int v = 0; v < V; ++v) rows[t * V + v] = static_cast<float>(tail.dists[t][v]);
        check(dd_upload_q(ctx_, rows.data(), static_cast<int>(tail.size()), V));
    }

    // verify_prefix + verify_bundle (duo) on the device; advances the role's
    // RandomStream by exactly the draws the kernel consumed.
    dd_verify_out verify_duo(const duodec::GenerationState& s, const duodec::DraftBundle& b,
                             duodec::RandomStream& rng, double temperature, bool greedy) {
        dd_verify_args a{};
        a.mode = DD_MODE_DUO;
        a.tail_len = s.unverified ? static_cast<int>(s.unverified->size()) : 0;
        a.n_firsts = b.sequence_count();
        if (a.n_firsts > 16) throw duodec::ConfigError("bundle wider than the device verifier (16)");
        for (int i = 0; i < a.n_firsts; ++i) a.firsts[i] = static_cast<std::int32_t>(b.sequences[i].tokens[0]);
        a.seed = rng.seed();
        a.counter = rng.counter();
        a.temperature = temperature;
        a.greedy = greedy ? 1 : 0;
        dd_verify_out o{};
        check(dd_verify(ctx_, &a, &o));
        for (int i = 0; i < o.n_draws; ++i) (void)rng.next_u64();
        return o;
    }

    // After apply_verification commits to s.verified: the cache keeps every
    // verified token except the last committed one.
    void rollback(const duodec::GenerationState& s) {
        check(dd_kv_truncate(ctx_, static_cast<int>(s.verified.size()) - 1));
    }

    // calibrate's target half: median device time of a pass of width w.
    double pass_ms(int w, int trials) {
        float ms = 0.0f;
        check(dd_time_pass(ctx_, w, trials, &ms));
        return ms;
    }

    dd_ctx* raw() const { return ctx_; }

private:
    void check(int rc) const {
        if (rc != DD_OK) throw duodec::ConfigError(dd_last_error(ctx_));
    }
    static std::vector<std::int32_t> to_i32(const std::vector<duodec::Token>& v) {
        return std::vector<std::int32_t>(v.begin(), v.end());
    }
    dd_ctx* ctx_ = nullptr;
};

}  // namespace duodec_b200
