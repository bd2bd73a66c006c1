// CPU draft model (Llama-family, bf16 weights) for the host draft worker.
#pragma once

#include <stdint.h>

#include <atomic>
#include <functional>
#include <string>
#include <thread>
#include <memory>
#include <vector>

#include "../../include/duodec_b200.h"

namespace dd {

// Fixed-size pool of pinned spinning workers; run(fn) calls fn(tid, nthreads)
// on every thread (the caller is tid 0) and returns when all are done.
class SpinPool {
  public:
    SpinPool(int n_threads, const std::vector<int>& cpus);
    ~SpinPool();
    int size() const { return n_; }
    void run(const std::function<void(int, int)>& fn);

  private:
    void worker(int tid);
    int n_;
    std::vector<std::thread> th_;
    std::atomic<uint64_t> gen_{0};
    // per-worker completion word (the job generation it finished), one cache
    // line each: the caller polls them instead of every worker incrementing
    // one contended counter
    struct alignas(64) Done {
        std::atomic<uint64_t> gen{0};
    };
    std::unique_ptr<Done[]> done_;
    std::atomic<int> sleepers_{0};
    std::atomic<bool> stop_{false};
    const std::function<void(int, int)>* job_ = nullptr;
};

// W8A8 weight matrix: per-row symmetric int8 (scale = max|w| / 127) plus the
// row sums used by the unsigned-activation VNNI trick.
struct QMat {
    int rows = 0, cols = 0;
    std::vector<int8_t> q;        // [rows][cols]
    std::vector<float> scale;     // [rows]
    std::vector<int32_t> rowsum;  // [rows] sum of q
    // AMX copy for prefill-sized matmuls (rows % 32 == 0, cols % 64 == 0):
    // [rows / 16][cols / 64] tiles of 16 x 64 bytes, row r of a tile holding
    // the 4 consecutive k of the tile's 16 output rows (TDPBUSD B layout)
    std::vector<int8_t> amx;
};

// W4 LM head (the draft's largest matrix, streamed once per drafted token):
// per-row symmetric 4-bit (scale = max|w| / 7), stored offset-binary (w + 8)
// two per byte - byte j of the 64-byte block b holds k = 128 b + j in its low
// and k = 128 b + 64 + j in its high nibble, so one load and two masks give
// the VNNI operands of two 64-wide activation slices.  Used when cols is a
// multiple of 128 (else the head stays W8).
struct Q4Mat {
    int rows = 0, cols = 0;
    std::vector<uint8_t> q;       // [rows][cols / 2]
    std::vector<float> scale;     // [rows]
    std::vector<int32_t> rowsum;  // [rows] sum of the signed 4-bit values
};

struct DraftLayer {
    QMat qkv, o, gu, dn;  // row-major [out][in]
    Q4Mat gu4, dn4;       // nibble copies of gu / dn (DD_DRAFT_FFN_BITS=4)
    bool w4 = false;
    Q4Mat qkv4, o4;       // nibble copies of qkv / o (DD_DRAFT_ATTN_BITS=4)
    bool a4 = false;
};

// Llama forward on host cores with a KV cache that follows the draft
// context: logits(ctx) reuses the longest cached prefix of ctx.
class CpuLlama {
  public:
    CpuLlama(const dd_model_desc& d, uint64_t weight_seed, const dd_plant_desc* plant,
             int n_threads, const std::vector<int>& cpus);
    int vocab() const { return V_; }
    // next-token logits after ctx (fp32, V); returns false on bad input
    bool logits(const int32_t* ctx, int n, float* out);
    // q = softmax(logits / T) rounded to fp32 (greedy: one-hot at the argmax);
    // also returns the argmax (lowest id on ties)
    int distribution(const float* logits, double temperature, bool greedy, float* q);
    // indices of the k largest q (descending, ties ascending id)
    void top_k(const float* q, int k, int32_t* out);
    // inverse-CDF sample of q with uniform u (distribution.cpp:61-78): pool
    // chunk sums + a sequential walk of the crossing chunk
    int sample(const float* q, double u);
    SpinPool& pool() { return *pool_; }
    int cached() const { return static_cast<int>(tokens_.size()); }
    std::string err;

  private:
    void forward(const int32_t* toks, int w, float* logits_last);
    int L_, d_, H_, Hkv_, hd_, F_, V_, max_seq_;
    float eps_;
    std::vector<uint16_t> emb_;
    QMat head_;
    Q4Mat head4_;
    bool head_w4_ = false;
    std::vector<DraftLayer> layers_;
    std::vector<uint16_t> kv_;  // K: [L][Hkv][max_seq/16][hd][16] (16-key blocks, dim-major inside), V: [L][Hkv][max_seq][hd]; bf16
    std::vector<float> rope_cos_, rope_sin_;
    std::vector<int32_t> tokens_;  // tokens whose K/V are cached
    std::unique_ptr<SpinPool> pool_;
    // scratch
    std::vector<float> x_, qkv_, q_, o_, gu_, a_, y_, logits_tmp_;
    std::vector<uint16_t> hb_, ob_, ab_;
    std::vector<uint8_t> xq_;  // quantised activations (u8 = q + 128)
    std::vector<float> xs_;    // per-token activation scales
};

}  // namespace dd

struct dd_draft {
    std::unique_ptr<dd::CpuLlama> model;
    std::vector<int> cpus;
    std::string err;
    bool calib_warmed = false;  // dd_calibrate's 1 s steady-state warm-up ran
};
