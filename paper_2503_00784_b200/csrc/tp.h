// Tensor parallelism for the 70B-shape target (BASELINE config 5).
//
// Megatron split, one rank per GPU: QKV / gate-up column-parallel (local heads
// and FFN features), O / down row-parallel, LM head vocabulary-parallel, the
// embedding and the fp32 residual stream replicated.  The two row-parallel
// GEMMs per layer store fp32 partials; tp_reduce_residual then sums every
// rank's partial over peer memory (NVLink P2P loads, rank order 0..N-1 on
// every rank, so the replicated residual stays bit-identical across ranks)
// and applies the residual add + deferred-RMSNorm producer that the unsharded
// GEMM epilogue fuses.  The vocabulary-parallel head writes local logits;
// tp_gather_logits assembles the full rows on every rank, and the acceptance
// kernel runs redundantly on each rank with the same seed and counter (no
// broadcast), as SURVEY.md §8e prescribes.
//
// Synchronisation: every rank owns a symmetric exchange buffer (flags |
// 2 partial buffers | local logits).  Op k of a pass signals by storing
// epoch * ops_per_pass + k + 1 (release, system scope) into flag[rank] of
// every peer, then waits until all flags reach that value (acquire).  The
// partial buffers alternate by op parity: a rank rewrites buffer k % 2 only at
// op k + 2, after it has seen every peer's op k + 1 signal, which each peer
// sends only after finishing its op k reads.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "model.h"

namespace dd {

constexpr int kMaxTp = 8;
constexpr int kTpFlagStride = 32;  // ints: one 128-byte line per source rank
// Persistent pass kernel under TP (pass.cu tp_exchange): the O / down
// reducers exchange their reduced fp32 tile [128 rows][16 tokens] with the
// peers' reducers of the same tile, through 4 rotating slots per tile and one
// flag line per (source rank, tile).
constexpr int kTpPassTiles = 64;  // d_model <= 8192
constexpr int kTpPassSlots = 4;

struct TpPeers {
    float* part[kMaxTp];  // rank r's [2][kMaxPassTokens][d] fp32 partials
    float* lg[kMaxTp];    // rank r's [kMaxPassTokens][v0[r+1] - v0[r]] local logits
    int* flags[kMaxTp];   // rank r's [kMaxTp][kTpFlagStride] arrival flags
    int v0[kMaxTp + 1];   // vocabulary split (multiples of 128)
    int* pflags[kMaxTp];  // rank r's [kMaxTp][kTpPassTiles][kTpFlagStride] pass-kernel tile flags
    float* pxch[kMaxTp];  // rank r's [kTpPassSlots][kTpPassTiles][128][16] reduced tiles
    int rank, size;
    int shared;  // every rank on one device (test harness): the waiting kernels run on few CTAs
};

// exchange-buffer layout (identical on every rank)
struct TpLayout {
    size_t flags_off, part_off, lg_off, pflag_off, pxch_off, bytes;
    size_t part_stride;  // floats per partial buffer
};
TpLayout tp_layout(int d, int max_local_vocab);

// ops_per_pass = 2 * n_layers + 1 (two reductions per layer, then the gather)
void launch_tp_reduce_residual(const TpPeers& P, const PassState* ps, int op, int ops_per_pass,
                               int d, float* x, __nv_bfloat16* u, const float* gain,
                               float* ss_out, cudaStream_t s);
void launch_tp_gather_logits(const TpPeers& P, const PassState* ps, int op, int ops_per_pass,
                             int vocab, float* logits, cudaStream_t s);

}  // namespace dd
