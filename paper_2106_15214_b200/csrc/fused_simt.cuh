// Kernels shared by both forms of the fused single-read pass (the tcgen05
// kernel, fused_tc_kernel.cuh, and the SIMT pair, fused_simt2.cuh):
// the fixed-order reduction of the per-CTA partials and the W update.
#pragma once

#include "fused_common.cuh"
#include "simt_kernels.cuh"

namespace bnmf {

constexpr int FS_KMAX = 64;   // largest rank of the fused schedule (fs2 SIMT pair)

// comm[0:2FK] = sum_g part[g], comm[2FK] = sum_g opart[g]  (fixed order)
// Fixed-order sum of the per-CTA partials.  With a row-split cluster
// (cl == 2) CTA g owns rows [0, split) when g is even, else [split, F); it
// only writes its own rows, so row f sums the CTAs of its owner rank.
static __global__ void fused_reduce(const double* __restrict__ part, const double* __restrict__ opart,
                             int G, int Gobj, int FK2, int K, int split, int cl,
                             double* __restrict__ comm,
                             const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < FK2) {
    const int f = (i % (FK2 / 2)) / K;
    const int r = (cl > 1 && f >= split) ? 1 : 0;
    // loads batched 8 at a time, summed in slab order
    double s = 0.0;
    int g = r;
    for (; g + 7 * cl < G; g += 8 * cl) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(g + u * cl) * FK2 + i];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; g < G; g += cl) s += part[(size_t)g * FK2 + i];
    comm[i] = s;
  } else if (i == FK2) {
    double s = 0.0;
    for (int g = 0; g < Gobj; ++g) s += opart[g];
    comm[i] = s;
  }
}

// W update for iteration p+1 and everything pass p+1 needs (one block per k):
//   W_{p+1} = W~_p * (num/max(den,floor))^gamma   (updates.py:203-220)
//   norms_{p+1}, W~_{p+1} = W_{p+1}/norms (solver.py:167-171)
//   C1 = chi1(W_{p+1}, W~_p), C2 = chi2(...) (JMM) or W_{p+1} (BMM)
struct WPair { float* w[2]; };

static __global__ void __launch_bounds__(1024) fused_update(const double* __restrict__ comm, int F, int K,
                             WPair Wt2, float* Wn, float* C1, float* C2, double* norms,
                             double* csum2,
                             int algorithm, int den_ones, Scalars sc, const RunState* st, int slot,
                             int p_override, RunState* st_fin, double* tr_obj, double* tr_sec) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  // st_fin != nullptr: trace row and stop rule of this iteration (the finish_iter launch folded
  // in; the objective sits behind the W sums in comm).  A stop leaves this slot active.
  if (st_fin && blockIdx.x == 0 && threadIdx.x == 0)
    finish_body(st_fin, slot, comm[(size_t)2 * F * K], tr_obj, tr_sec, sc.tol);
  const int par = iter_parity(st, slot, p_override);
  const float* Wcur = Wt2.w[par];    // W~_p
  float* Wnext = Wt2.w[par ^ 1];     // W~_{p+1}
  const int k = blockIdx.x;
  __shared__ double red[32];
  const double* num = comm;
  const double* den = comm + (size_t)F * K;
  double s = 0.0;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    size_t i = (size_t)f * K + k;
    double r = num[i] / fmax(den[i], sc.floor);
    float w = float(double(Wcur[i]) * apply_exponent<double>(r, sc.gamma));
    Wn[i] = w;
    s += double(w) * double(w);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    red[0] = sqrt(t);
    norms[k] = red[0];
  }
  __syncthreads();
  const double nrm = red[0];
  const float beta = float(sc.beta);
  double cs = 0.0;
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    size_t i = (size_t)f * K + k;
    float w = Wn[i];
    Wnext[i] = float(double(w) / nrm);
    float c2;
    if (algorithm == 0) {
      C1[i] = chi1<float>(w, Wcur[i], beta);
      c2 = chi2<float>(w, Wcur[i], beta);
    } else {
      C1[i] = w;
      c2 = w;
    }
    C2[i] = c2;
    cs += double(c2);
  }
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cs;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    csum2[k] = t;
  }
}

}  // namespace bnmf
