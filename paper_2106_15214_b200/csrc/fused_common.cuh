// Shared pieces of the fused single-read schedule (fp32, L = 1).
//
// Pass p (iteration p >= 1) reads V once and, per column block:
//   1. recomputes Vt_{p-1} = Wa H~_{p-1} + kappa (Wa = W~_{p-1} for JMM, the new
//      W_p for BMM) and finishes the H update of iteration p
//        H_p = H~_{p-1} * ((chi1^T Zn)/max(chi2^T Zd, floor))^gamma
//      (updates.py:223-235 / 173-181), then H~_p = H_p * norms_p;
//   2. forms Vt_p = W~_p H~_p + kappa (== W_p H_p + kappa, solver.py:304-306),
//      the objective of iterate p (core.py:89-114, cancellation-free form),
//      and the W-side sums of iteration p+1: Zn(Vt_p) H~_p^T, Zd(Vt_p) H~_p^T
//      (updates.py:203-220; chi(H~,H~) = H~ at L = 1).
// The prologue pass (before iteration 1) does step 2 only, on the raw init.
#pragma once

#include "bnmf_common.cuh"

namespace bnmf {

// Pointers of one pass; ping-pong buffers are chosen on the device from the
// parity of the iteration so that CUDA graphs can replay fixed arguments.
struct FusedArgs {
  const float* V;
  long long ldv;
  int F, N, K;
  const float* Hbuf[2];   // H~ (N x K) by iteration parity
  float* Hout[2];
  const float* Wt2[2];    // W~ (F x K) by iteration parity
  const float* Wn;        // W_{p} unnormalised (BMM's H-side factor)
  const float* C1;        // chi1(W_p, W~_{p-1}) (F x K)
  const float* C2;        // chi2(...)
  const double* norms;    // norms of W_p (K)
  const double* csum2;    // colsum(C2) (K), used when den_ones
  double* part;           // per-CTA W-side partials [G][2][F][K]
  double* opart;          // per-CTA objective partials [G]
  int algorithm;          // 0 jmm, 1 bmm
  int do_h;               // 0 = prologue (W-side + objective only)
  int den_ones;           // beta == 1: H den = colsum(C2), W den = rowsum(H~)
  int kkt;                // 1 = KKT pass (H side only, no update): sum |min(H~_p, W~_p^T (Zd - Zn))|
                          // per CTA into opart (diagnostics.py:46-59); Wa = C1 = C2 = W~_p
  long long* prof;        // optional per-CTA wait-cycle counters [G][48] (BNMF_TC_PROF=1)
  unsigned long long* tmark;  // RunState::t_begin when this launch opens a timed iteration, else null
  Scalars sc;
};

__device__ __forceinline__ int iter_parity(const RunState* st, int slot, int p_override) {
  long long p = p_override >= 0 ? p_override : st->base + slot;
  return int(p & 1);
}

// ---- fp32 elementwise forms ---------------------------------------------

template <int BC>
__device__ __forceinline__ void bases32(float x, float y, float beta, float& zn, float& zd) {
  if (BC == BC_2) { zn = x; zd = y; }
  else if (BC == BC_1) { zn = __fdiv_rn(x, y); zd = 1.f; }
  else if (BC == BC_0) { float r = __fdiv_rn(1.f, y); zn = x * r * r; zd = r; }
  else {
    float a = powf(y, beta - 2.f);
    zn = x * a; zd = a * y;
  }
}

// phi(u) = [(1+u)^b - 1 - b u] / (b (b-1)) for |u| < 0.25 by its series
// sum_{j>=2} C(b, j) u^j / (b (b-1)); coefficients c_j = prod_{i=2}^{j-1} (b-i)/ (i+1)... built
// incrementally: t_2 = 1/2, t_{j+1} = t_j * (b - j) / (j + 1).
__device__ __forceinline__ float phi_series(float u, float b) {
  float t = 0.5f, s = 0.f, up = u * u;
#pragma unroll
  for (int j = 2; j < 14; ++j) {
    s = fmaf(t, up, s);
    t = t * (b - float(j)) / float(j + 1);
    up *= u;
  }
  return s;
}

// d_beta(x | y) in fp32 without catastrophic cancellation (x ~ y).  The
// reference's literal forms (core.py:97-109) lose all digits there in fp32.
template <int BC>
__device__ __forceinline__ float divergence32(float x, float y, float beta) {
  if (BC == BC_2) { float d = x - y; return 0.5f * d * d; }
  float u = __fdiv_rn(x - y, y);  // t - 1, accurate
  if (BC == BC_1) {
    // y * (t log t - t + 1) = y * ((1+u) log1p(u) - u)
    if (x == 0.f) return y;
    if (fabsf(u) < 0.25f) {
      // (1+u)log1p(u) - u = sum_{j>=2} (-1)^j u^j / (j (j-1))
      float s = 0.f, up = u * u, sg = 1.f;
#pragma unroll
      for (int j = 2; j < 16; ++j) { s = fmaf(sg / float(j * (j - 1)), up, s); up *= u; sg = -sg; }
      return y * s;
    }
    return x * logf(x / y) - x + y;
  }
  if (BC == BC_0) {
    // t - log t - 1 = u - log1p(u)
    if (fabsf(u) < 0.25f) {
      float s = 0.f, up = u * u, sg = 1.f;
#pragma unroll
      for (int j = 2; j < 16; ++j) { s = fmaf(sg / float(j), up, s); up *= u; sg = -sg; }
      return s;
    }
    float t = x / y;
    return t - logf(t) - 1.f;
  }
  // generic: y^b * phi(u)
  float yb = powf(y, beta);
  if (fabsf(u) < 0.25f) return yb * phi_series(u, beta);
  return powf(x, beta) / (beta * (beta - 1.f)) + yb / beta - x * powf(y, beta - 1.f) / (beta - 1.f);
}

}  // namespace bnmf
