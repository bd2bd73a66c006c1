// Host interface of the fused acceptance kernel (accept.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/duodec_b200.h"

namespace dd {

struct AcceptParams {
    int mode;       // DD_MODE_*
    int V;
    int L;          // tested rows 0..L-1 (tail / draft); row L = p_next / bonus
    int s;          // bundle size (duo)
    int greedy;
    int q_onehot;
    int row0;       // logits row holding target_dists[0]
    double inv_temp;
    uint64_t seed, counter;
    int32_t firsts[16];
    const float* logits;   // [>= row0+L+1][V] fp32 (when probs == nullptr)
    const double* probs;   // [L+1][V] fp64 probabilities, or nullptr
    const float* q;        // [L][V] draft rows (unless q_onehot)
    const int32_t* tail;   // [L] tail / draft tokens (device)
    double* row_m;         // scratch [L+1]
    double* row_sum;       // scratch [L+1]
    int* row_argmax;       // scratch [L+1]
    unsigned int* ticket;  // zero-initialised counter (reset by the kernel)
    dd_verify_out* out;    // mapped-host result: fields, system fence, then out->pad = seq
    int seq;               // completion sequence the host polls for (nonzero)
};

cudaError_t launch_accept(const AcceptParams& p, cudaStream_t stream);

}  // namespace dd
