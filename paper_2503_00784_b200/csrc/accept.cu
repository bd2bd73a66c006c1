// Fused logits -> softmax -> speculative-sampling acceptance (sm_100a).
//
// One launch per verification step.  Grid = L+1 CTAs; CTA r reduces row r of
// the scored pass (fp64 max / sum-exp, or the argmax for greedy), then the
// last CTA to finish (global ticket) replays the reference's sequential
// decision procedure with the SAME RandomStream draw schedule:
//
//   duo  : verify_prefix  (proj/src/verify.cpp:41-61)  on rows 0..L-1, then,
//          if the whole tail passed, verify_bundle (verify.cpp:63-90) on row L
//   sps  : sps_verify     (verify.cpp:92-107)
//   vanilla: sample(p, next_uniform) (proj/src/engine.cpp:288-291)
//
// accept_test is the strict r < p/q of verify.cpp:25-28; residual_or_p is
// verify.cpp:13-21 (max(p-q,0), renormalised, p on zero mass); sample() is the
// inverse CDF of distribution.cpp:61-78 (skip p<=0, first i with u < acc,
// else the last support).  The O(V) parts (residual mass, CDF scan) run
// block-parallel: per-thread chunk sums, a block scan, then one thread walks
// the crossing chunk sequentially.  Rows are fp64 p = softmax(logits/T) or,
// for greedy, one-hot at the lowest-index argmax (kernels_scalar.cpp:40-48).
#include <cstddef>

#include "accept.h"
#include "common.cuh"

namespace dd {

namespace {

constexpr int kThreads = 512;
constexpr double kZeroMass = 1e-12;  // kZeroMassThreshold, distribution.hpp:17

struct Ctx {
    const AcceptParams* P;
    __device__ double p_at(int r, int i) const {
        if (P->greedy) return i == P->row_argmax[r] ? 1.0 : 0.0;
        if (P->probs) return P->probs[static_cast<size_t>(r) * P->V + i];
        const double z = static_cast<double>(P->logits[static_cast<size_t>(P->row0 + r) * P->V + i]) *
                         P->inv_temp;
        return exp(z - P->row_m[r]) / P->row_sum[r];
    }
    __device__ double q_at(int j, int i) const {
        if (P->q_onehot) return i == P->tail[j] ? 1.0 : 0.0;
        return static_cast<double>(P->q[static_cast<size_t>(j) * P->V + i]);
    }
};

__device__ double block_sum_d(double v, double* red) {
    v = warp_sum_d(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = lane < kThreads / 32 ? red[lane] : 0.0;
    t = warp_sum_d(t);
    __syncthreads();
    return t;
}

// What the single sampling step of this verification draws from.
enum SampleKind { kNone = 0, kResidual = 1, kPlain = 2 };

struct Shared {
    double red[kThreads / 32];
    double scan[kThreads];
    int kind, row, qrow, result, crossing, last_support;
    double u, scale, inv_mass;
    int removed[16];
    int n_removed;
};

// value of the sampling distribution at i (before the zero-mass decision for kResidual)
__device__ __forceinline__ double sample_value(const Ctx& c, const Shared& sh, int i) {
    if (sh.kind == kResidual) {
        const double d = c.p_at(sh.row, i) - c.q_at(sh.qrow, i);
        if (sh.inv_mass < 0.0) return c.p_at(sh.row, i);  // residual_or_p fallback
        return (d > 0.0 ? d : 0.0) * sh.inv_mass;
    }
    for (int k = 0; k < sh.n_removed; ++k)
        if (sh.removed[k] == i) return 0.0;
    return c.p_at(sh.row, i) * sh.scale;
}

// Inverse-CDF sample over V with the block (all threads participate).
__device__ int block_sample(const Ctx& c, Shared& sh) {
    const int V = c.P->V;
    const int chunk = (V + kThreads - 1) / kThreads;
    const int lo = min(V, threadIdx.x * chunk), hi = min(V, lo + chunk);
    if (sh.kind == kResidual) {
        double m = 0.0;
        for (int i = lo; i < hi; ++i) {
            const double d = c.p_at(sh.row, i) - c.q_at(sh.qrow, i);
            m += d > 0.0 ? d : 0.0;
        }
        const double mass = block_sum_d(m, sh.red);
        if (threadIdx.x == 0) sh.inv_mass = mass < kZeroMass ? -1.0 : 1.0 / mass;
        __syncthreads();
    }
    double s = 0.0;
    int last = -1;
    for (int i = lo; i < hi; ++i) {
        const double v = sample_value(c, sh, i);
        if (v > 0.0) {
            s += v;
            last = i;
        }
    }
    // block inclusive scan (Hillis-Steele over kThreads doubles)
    sh.scan[threadIdx.x] = s;
    if (threadIdx.x == 0) {
        sh.crossing = kThreads;
        sh.last_support = -1;
    }
    __syncthreads();
    for (int off = 1; off < kThreads; off <<= 1) {
        const double add = threadIdx.x >= off ? sh.scan[threadIdx.x - off] : 0.0;
        __syncthreads();
        sh.scan[threadIdx.x] += add;
        __syncthreads();
    }
    const double incl = sh.scan[threadIdx.x];
    const double excl = incl - s;
    if (last >= 0) atomicMax(&sh.last_support, last);
    if (s > 0.0 && sh.u < incl) atomicMin(&sh.crossing, static_cast<int>(threadIdx.x));
    __syncthreads();
    if (static_cast<int>(threadIdx.x) == sh.crossing) {
        double acc = threadIdx.x == 0 ? 0.0 : sh.scan[threadIdx.x - 1];
        (void)excl;
        int res = last;
        for (int i = lo; i < hi; ++i) {
            const double v = sample_value(c, sh, i);
            if (v <= 0.0) continue;
            acc += v;
            if (sh.u < acc) {
                res = i;
                break;
            }
        }
        sh.result = res;
    }
    __syncthreads();
    if (sh.crossing == kThreads) return sh.last_support;  // u in the rounding slack
    return sh.result;
}

__device__ __forceinline__ double next_uniform(uint64_t seed, uint64_t& counter) {
    return u64_to_uniform(splitmix_draw(seed, ++counter));
}

__global__ void __launch_bounds__(kThreads) accept_kernel(AcceptParams P) {
    __shared__ Shared sh;
    __shared__ double red[kThreads / 32];
    __shared__ float redf[kThreads / 32];
    __shared__ int redi[kThreads / 32];
    __shared__ bool is_last;
    const int r = blockIdx.x;
    const int V = P.V;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---------------- phase A: row statistics ----------------
    if (!P.probs) {
        const float* row = P.logits + static_cast<size_t>(P.row0 + r) * V;
        if (P.greedy) {
            float best = -INFINITY;
            int bi = V;
            for (int i = threadIdx.x; i < V; i += kThreads) {
                const float v = row[i];
                if (v > best || (v == best && i < bi)) {
                    best = v;
                    bi = i;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > best || (ov == best && oi < bi)) {
                    best = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                redf[warp] = best;
                redi[warp] = bi;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                best = redf[0];
                bi = redi[0];
                for (int k = 1; k < kThreads / 32; ++k)
                    if (redf[k] > best || (redf[k] == best && redi[k] < bi)) {
                        best = redf[k];
                        bi = redi[k];
                    }
                P.row_argmax[r] = bi;
            }
        } else {
            double m = -INFINITY;
            for (int i = threadIdx.x; i < V; i += kThreads)
                m = fmax(m, static_cast<double>(row[i]) * P.inv_temp);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[warp] = m;
            __syncthreads();
            m = red[0];
            for (int k = 1; k < kThreads / 32; ++k) m = fmax(m, red[k]);
            __syncthreads();
            double s = 0.0;
            for (int i = threadIdx.x; i < V; i += kThreads)
                s += exp(static_cast<double>(row[i]) * P.inv_temp - m);
            s = block_sum_d(s, red);
            if (threadIdx.x == 0) {
                P.row_m[r] = m;
                P.row_sum[r] = s;
            }
        }
    } else if (P.greedy) {
        const double* row = P.probs + static_cast<size_t>(r) * V;
        if (threadIdx.x == 0) {  // tiny vocabularies only on this path
            int bi = 0;
            for (int i = 1; i < V; ++i)
                if (row[i] > row[bi]) bi = i;
            P.row_argmax[r] = bi;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(P.ticket, 1u);
        is_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // ---------------- phase B: sequential decisions (last CTA) ----------------
    Ctx c{&P};
    uint64_t counter = P.counter;
    if (threadIdx.x == 0) {
        sh.kind = kNone;
        sh.n_removed = 0;
        sh.scale = 1.0;
        sh.inv_mass = 1.0;
        sh.result = -1;
    }
    __syncthreads();

    __shared__ dd_verify_out out;
    __shared__ bool need_bundle;
    __shared__ double p_total;
    if (threadIdx.x == 0) {
        out = dd_verify_out{};
        out.reject_index = -1;
        out.resample = -1;
        out.seq_index = -1;
        out.fallback = -1;
        out.next_token = -1;
        need_bundle = false;
        const int L = P.L;
        if (P.mode == DD_MODE_VANILLA) {
            sh.kind = kPlain;
            sh.row = 0;
            sh.u = next_uniform(P.seed, counter);
        } else {
            int k = -1;
            for (int j = 0; j < L; ++j) {
                const int tok = P.tail[j];
                const double p = c.p_at(j, tok), q = c.q_at(j, tok);
                const double rr = next_uniform(P.seed, counter);
                if (!(rr < p / q)) {
                    k = j;
                    break;
                }
            }
            if (k >= 0) {
                sh.kind = kResidual;
                sh.row = k;
                sh.qrow = k;
                sh.u = next_uniform(P.seed, counter);
                out.reject_index = k;
                out.prefix_all_accepted = 0;
                out.sps_accepted = k;
            } else if (P.mode == DD_MODE_SPS) {
                out.sps_accepted = L;
                sh.kind = kPlain;  // bonus token from target_dists[L]
                sh.row = L;
                sh.u = next_uniform(P.seed, counter);
            } else {
                out.prefix_all_accepted = 1;
                need_bundle = true;
            }
        }
    }
    __syncthreads();

    if (need_bundle) {
        // verify_bundle on row L: point-mass tests against the running residual
        const int L = P.L;
        const int chunk = (V + kThreads - 1) / kThreads;
        const int lo = min(V, threadIdx.x * chunk), hi = min(V, lo + chunk);
        double s = 0.0;
        for (int i = lo; i < hi; ++i) s += c.p_at(L, i);
        const double tot = block_sum_d(s, red);
        if (threadIdx.x == 0) {
            p_total = tot;
            double scale = 1.0, removed_p = 0.0;
            int accepted = -1;
            for (int i = 0; i < P.s; ++i) {
                const int tok = P.firsts[i];
                bool gone = false;
                for (int k = 0; k < sh.n_removed; ++k) gone |= sh.removed[k] == tok;
                const double cur = gone ? 0.0 : c.p_at(L, tok) * scale;
                const double rr = next_uniform(P.seed, counter);
                if (rr < cur) {  // accept_test(cur[t], 1.0, r)
                    accepted = i;
                    break;
                }
                if (!gone) {
                    sh.removed[sh.n_removed++] = tok;
                    removed_p += c.p_at(L, tok);
                }
                const double mass = (p_total - removed_p) * scale;
                if (mass < kZeroMass) {  // reset to p_next (verify.cpp:77-81)
                    sh.n_removed = 0;
                    removed_p = 0.0;
                    scale = 1.0;
                } else {
                    scale = scale * (1.0 / mass);
                }
            }
            if (accepted >= 0) {
                out.bundle_accepted = 1;
                out.seq_index = accepted;
                sh.kind = kNone;
            } else {
                out.bundle_accepted = 0;
                sh.kind = kPlain;
                sh.row = L;
                sh.scale = scale;
                sh.u = next_uniform(P.seed, counter);
            }
        }
        __syncthreads();
    }

    if (sh.kind != kNone) {
        const int tok = block_sample(c, sh);
        if (threadIdx.x == 0) {
            if (P.mode == DD_MODE_VANILLA) {
                out.next_token = tok;
            } else if (P.mode == DD_MODE_SPS) {
                out.next_token = tok;
            } else if (out.reject_index >= 0) {
                out.resample = tok;
            } else {
                out.fallback = tok;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out.counter_out = counter;
        out.n_draws = static_cast<int>(counter - P.counter);
        // every field, one system-scope fence, then the sequence word the host
        // spins on (mapped pinned memory: no copy, no stream synchronisation)
        out.pad = P.seq;
        const int* src = reinterpret_cast<const int*>(&out);
        volatile int* dst = reinterpret_cast<volatile int*>(P.out);
        constexpr int kSeqWord = offsetof(dd_verify_out, pad) / sizeof(int);
        for (int i = 0; i < static_cast<int>(sizeof(dd_verify_out) / sizeof(int)); ++i)
            if (i != kSeqWord) dst[i] = src[i];
        *P.ticket = 0u;  // reusable for the next launch
        __threadfence_system();
        dst[kSeqWord] = P.seq;
    }
}

}  // namespace

cudaError_t launch_accept(const AcceptParams& p, cudaStream_t stream) {
    accept_kernel<<<p.L + 1, kThreads, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace dd

namespace dd {
void preload_accept_kernels() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, accept_kernel);
}
}  // namespace dd
