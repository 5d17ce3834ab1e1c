// Shared device-side definitions for the beta-NMF B200 library.
//
// Elementwise rules restate the reference (paths relative to
// /root/reference/pkg/src/betanmf):
//   joint bases / power pair ........ updates.py:184-200, core.py:156-173
//   chi maps ......................... updates.py:84-107
//   guarded divide + exponent ........ core.py:117-130, updates.py:118-123
//   entrywise divergence ............. core.py:89-109
//   KKT gradient core ................ diagnostics.py:46-59
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

namespace bnmf {

// beta classes with literal fast forms (updates.py:243-331); everything else
// is the generic power-pair rule.
enum BetaClass : int { BC_GEN = 0, BC_0 = 1, BC_1 = 2, BC_2 = 3 };

inline int beta_class(double beta) {
  if (beta == 0.0) return BC_0;
  if (beta == 1.0) return BC_1;
  if (beta == 2.0) return BC_2;
  return BC_GEN;
}

// Per-run scalar parameters, passed by value to every kernel.
struct Scalars {
  double beta;
  double gamma;
  double kappa;
  double floor;
  double tol;
};

// Device-resident run control (see engine.cu): iteration base for graph
// chunks, stop iteration, trace bookkeeping.
struct RunState {
  long long base;        // global iteration index of chunk slot 0 (1-based)
  long long stop_iter;   // last iteration to execute (INT64_MAX until stop)
  long long max_iter;    // max_outer_iters
  long long iters_done;  // last finished iteration
  double prev_obj;
  unsigned long long t_begin;  // globaltimer at the start of the current iter
  double elapsed;        // accumulated seconds (solver.py:302-312 timer)
  int converged;
  int pad;
  unsigned long long t_last;   // sparse path: globaltimer at the last finished iteration
};

__device__ __forceinline__ bool iter_active(const RunState* st, int slot) {
  long long it = st->base + slot;
  return it <= st->stop_iter && it <= st->max_iter;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Objective bookkeeping + stop rule of iteration base + slot (solver.py:309-319, 174-180); one
// thread.  o: the reduced objective (global, after any allreduce).
__device__ __forceinline__ void finish_body(RunState* st, int slot, double o,
                                            double* __restrict__ trace_obj,
                                            double* __restrict__ trace_sec, double tol) {
  long long it = st->base + slot;
  bool stop = false;
  if (it > 1) {
    double prev = st->prev_obj;
    if (o == prev) stop = true;
    else if (o <= 0.0) stop = false;
    else stop = (prev - o) / o <= tol;
  }
  unsigned long long t = globaltimer();
  st->elapsed += double(t - st->t_begin) * 1e-9;
  trace_obj[it - 1] = o;
  trace_sec[it - 1] = st->elapsed;
  st->prev_obj = o;
  st->iters_done = it;
#ifdef BNMF_X_NOSTOP
  stop = false;   // timing experiments with garbage numerics
#endif
  if (stop) { st->stop_iter = it; st->converged = 1; }
}

// ---------------------------------------------------------------------------
// Elementwise rules.  T is the storage/compute type (float or double).

template <typename T> __device__ __forceinline__ T dpow(T a, T b);
template <> __device__ __forceinline__ double dpow<double>(double a, double b) { return pow(a, b); }
template <> __device__ __forceinline__ float dpow<float>(float a, float b) { return powf(a, b); }
template <typename T> __device__ __forceinline__ T dsqrt(T a);
template <> __device__ __forceinline__ double dsqrt<double>(double a) { return sqrt(a); }
template <> __device__ __forceinline__ float dsqrt<float>(float a) { return sqrtf(a); }

// (Z_num, Z_den) = (x * y^(beta-2), y^(beta-1)); Z_den == 1 for beta = 1.
// Literal joint_bases / fast-path forms (updates.py:193-200, 251-258).
template <int BC, typename T>
__device__ __forceinline__ void bases(T x, T y, T beta, T& zn, T& zd) {
  if (BC == BC_2) {
    zn = x; zd = y;
  } else if (BC == BC_1) {
    zn = x / y; zd = T(1);
  } else if (BC == BC_0) {
    zn = x / (y * y); zd = T(1) / y;
  } else {
    T p = beta - T(2);
    if (p == T(1)) {            // beta = 3: power_pair p == 1
      zn = x * y; zd = y * y;
    } else {
      T a = dpow<T>(y, p);
      zn = x * a; zd = a * y;
    }
  }
}

// KKT gradient core p^(beta-2) (p - x) (diagnostics.py:51-54).
template <int BC, typename T>
__device__ __forceinline__ T grad_core(T x, T y, T beta) {
  if (BC == BC_2) return y - x;
  T e = beta - T(2);
  T pw;
  if (e == T(0)) pw = T(1);
  else if (e == T(1)) pw = y;
  else if (e == T(-1)) pw = T(1) / y;
  else if (e == T(-2)) pw = T(1) / (y * y);
  else if (e == T(0.5)) pw = dsqrt<T>(y);
  else pw = dpow<T>(y, e);
  return pw * (y - x);
}

// d_beta(x | y) in double, literal core.py:97-109 (xlogy convention for x=0).
template <int BC>
__device__ __forceinline__ double divergence(double x, double y, double beta) {
  if (BC == BC_2) { double d = x - y; return 0.5 * d * d; }
  if (BC == BC_1) { return (x != 0.0 ? x * log(x / y) : 0.0) - x + y; }
  if (BC == BC_0) { double r = x / y; return r - log(r) - 1.0; }
  return pow(x, beta) / (beta * (beta - 1.0)) + pow(y, beta) / beta
         - x * pow(y, beta - 1.0) / (beta - 1.0);
}

// chi1 / chi2 (updates.py:84-107), entrywise on (m, m_tilde).
template <typename T>
__device__ __forceinline__ T chi1(T m, T mt, T beta) {
  if (beta >= T(2)) return m;
  if (beta == T(1)) return mt;
  if (beta == T(0)) return (mt * mt) / m;
  return dpow<T>(mt, T(2) - beta) * dpow<T>(m, beta - T(1));
}
template <typename T>
__device__ __forceinline__ T chi2(T m, T mt, T beta) {
  if (beta <= T(1)) return m;
  if (beta == T(2)) return (m * m) / mt;
  return dpow<T>(m, beta) / dpow<T>(mt, beta - T(1));
}

// ratio^gamma with the exponent short-cuts of updates.py:118-123.
template <typename T>
__device__ __forceinline__ T apply_exponent(T r, T g) {
  if (g == T(1)) return r;
  if (g == T(0.5)) return dsqrt<T>(r);
  return dpow<T>(r, g);
}

}  // namespace bnmf
