// Small per-iteration kernels: fixed-order reductions of partial sums, the
// multiplicative factor update, chi maps, normalisation and the trace /
// stop-rule bookkeeping (solver.py:167-180, 292-326; updates.py:118-123).
#pragma once

#include "bnmf_common.cuh"

namespace bnmf {

// out[i] = sum_{s < S} part[s * stride + i], fixed order (deterministic).
static __global__ void reduce_segments(const double* __restrict__ part, size_t stride, int S,
                                size_t count, double* __restrict__ out,
                                const RunState* st, int slot) {
  if (st && !iter_active(st, slot)) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[(size_t)k * stride + i];
    out[i] = s;
  }
}

// Single-block fixed-order sum of `count` doubles into *out (count small).
static __global__ void sum_small(const double* __restrict__ in, int count, double* __restrict__ out,
                          const RunState* st, int slot) {
  if (st && !iter_active(st, slot)) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += in[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    *out = t;
  }
}

// chi1 / chi2 of (M, Mt) entrywise, count entries.
template <typename T>
__global__ void chi_maps(const T* __restrict__ M, const T* __restrict__ Mt, T* __restrict__ o1,
                         T* __restrict__ o2, size_t count, Scalars sc, const RunState* st,
                         int slot) {
  if (!iter_active(st, slot)) return;
  const T beta = T(sc.beta);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T m = M[i], mt = Mt[i];
    if (o1) o1[i] = chi1<T>(m, mt, beta);
    if (o2) o2[i] = chi2<T>(m, mt, beta);
  }
}

// W-side update: out[f,k] = base[f,k] * (num/max(den,floor))^gamma, where den is
// either a full F x K array or (den_ones) the row-sum K-vector broadcast.
template <typename T>
__global__ void update_w(const T* __restrict__ base, const double* __restrict__ num,
                         const double* __restrict__ den, int den_is_vec, int F, int K,
                         T* __restrict__ out, Scalars sc, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F * K; i += gridDim.x * blockDim.x) {
    int k = i % K;
    double d = den_is_vec ? den[k] : den[i];
    double r = num[i] / fmax(d, sc.floor);
    out[i] = T(double(base[i]) * apply_exponent<double>(r, sc.gamma));
  }
}

// reduce_segments + update_w in one launch (one rank: no allreduce between them), optionally
// with the chi maps of the new W against its base (the JMM H-side factors, updates.py:97-107).
// The segment sums are added in the order reduce_segments uses, so the result is bitwise the
// same as the three launches it replaces.
template <typename T>
__global__ void reduce_update_w(const double* __restrict__ part, size_t stride, int S,
                                const T* __restrict__ base, int F, int K, T* __restrict__ out,
                                T* __restrict__ c1, T* __restrict__ c2, double* __restrict__ sums,
                                Scalars sc, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int fk = F * K;
  const T beta = T(sc.beta);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < fk; i += gridDim.x * blockDim.x) {
    // the segment partials are loaded in batches of 8 + 8 (independent loads in flight), then
    // added in segment order
    double num = 0.0, den = 0.0;
    int k = 0;
    for (; k + 8 <= S; k += 8) {
      double a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = part[(size_t)(k + u) * stride + i];
        b[u] = part[(size_t)(k + u) * stride + fk + i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { num += a[u]; den += b[u]; }
    }
    for (; k < S; ++k) {
      num += part[(size_t)k * stride + i];
      den += part[(size_t)k * stride + fk + i];
    }
    sums[i] = num;
    sums[fk + i] = den;
    const double r = num / fmax(den, sc.floor);
    const T b = base[i];
    const T w = T(double(b) * apply_exponent<double>(r, sc.gamma));
    out[i] = w;
    if (c1) c1[i] = chi1<T>(w, b, beta);
    if (c2) c2[i] = chi2<T>(w, b, beta);
  }
}

// Column sums of an F x K matrix -> double K-vector, one thread per column, rows added in
// order: the order of numpy's sum over axis 0, so that the beta = 1 denominators (and the
// exact-equality stop rule that can hang on their last bit) match the reference bit for bit.
// The loads, not the adds, are the latency (F dependent round trips to L2 took 36 us at
// config 1), so one block streams the matrix through shared memory with cp.async, as many
// rows per round as fit, and thread k then adds its column from there.
constexpr int CS_THREADS = 256;
constexpr size_t CS_SMEM_MAX = 160 * 1024;

template <typename T>
__global__ void __launch_bounds__(CS_THREADS)
col_sums(const T* __restrict__ M, int F, int K, double* __restrict__ out, int rows_per_round,
         const RunState* st, int slot) {
  if (st && !iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char cs_smem[];
  T* buf = reinterpret_cast<T*>(cs_smem);
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(buf));
  double s[(128 + CS_THREADS - 1) / CS_THREADS] = {0.0};   // K <= 128: one column per thread
  for (int f0 = 0; f0 < F; f0 += rows_per_round) {
    const int rows = min(rows_per_round, F - f0);
    const int n = rows * K;
    const T* src = M + (size_t)f0 * K;
    for (int i = threadIdx.x; i < n; i += CS_THREADS) {
      if (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 8u * i), "l"(src + i)
                     : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sbase + 4u * i), "l"(src + i)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < K) {
      const int k = threadIdx.x;
      for (int r = 0; r < rows; ++r) s[0] += double(buf[r * K + k]);
    }
    __syncthreads();
  }
  if (threadIdx.x < K) out[threadIdx.x] = s[0];
}

// norms[k] = sqrt(sum_f W[f,k]^2); Wn = W / norms (solver.py:167-171).
// One block of NW_THREADS per column: fixed-order thread partition, shuffle tree per warp, the
// warp sums added in warp order.
constexpr int NW_THREADS = 128;
template <typename T>
__global__ void __launch_bounds__(NW_THREADS)
normalize_w(const T* __restrict__ W, int F, int K, T* __restrict__ Wn,
            double* __restrict__ norms, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[NW_THREADS / 32];
  int k = blockIdx.x;
  double s = 0.0;
  for (int f = threadIdx.x; f < F; f += NW_THREADS) {
    double w = double(W[(size_t)f * K + k]);
    s += w * w;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < NW_THREADS / 32; ++w) tot += red[w];
  double nrm = sqrt(tot);
  if (threadIdx.x == 0) norms[k] = nrm;
  for (int f = threadIdx.x; f < F; f += NW_THREADS)
    Wn[(size_t)f * K + k] = T(double(W[(size_t)f * K + k]) / nrm);
}

// Hn[n,k] = H[n,k] * norms[k]  (Ht layout N x K).
template <typename T>
__global__ void scale_h(const T* __restrict__ H, size_t N, int K, const double* __restrict__ norms,
                        T* __restrict__ Hn, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  size_t count = N * (size_t)K;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    int k = int(i % K);
    Hn[i] = T(double(H[i]) * norms[k]);
  }
}

// scale_h plus the chi maps of the rescaled H against itself: the W-side factors of the next
// JMM iteration at its first sub-iteration (chi(H~, H~), updates.py:217-218)
template <typename T>
__global__ void scale_h_chi(const T* __restrict__ H, size_t N, int K,
                            const double* __restrict__ norms, T* __restrict__ Hn,
                            T* __restrict__ c1, T* __restrict__ c2, Scalars sc,
                            const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const T beta = T(sc.beta);
  size_t count = N * (size_t)K;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    int k = int(i % K);
    const T h = T(double(H[i]) * norms[k]);
    Hn[i] = h;
    c1[i] = chi1<T>(h, h, beta);
    c2[i] = chi2<T>(h, h, beta);
  }
}

// Mark the start of an iteration (timer, solver.py:302).
static __global__ void begin_iter(RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  st->t_begin = globaltimer();
}

// Objective bookkeeping + stop rule (solver.py:309-319, 174-180).
// obj: reduced objective (global, after any allreduce).
static __global__ void finish_iter(RunState* st, int slot, const double* __restrict__ obj,
                            double* __restrict__ trace_obj, double* __restrict__ trace_sec,
                            double tol) {
  if (!iter_active(st, slot)) return;
  finish_body(st, slot, *obj, trace_obj, trace_sec, tol);
}

// sum_small + finish_iter in one launch (one rank: no allreduce of the objective between them)
static __global__ void finish_iter_sum(RunState* st, int slot, const double* __restrict__ in,
                                       int count, double* __restrict__ obj,
                                       double* __restrict__ trace_obj,
                                       double* __restrict__ trace_sec, double tol) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += in[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double o = 0.0;
  for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) o += red[w];
  *obj = o;
  finish_body(st, slot, o, trace_obj, trace_sec, tol);
}

// res_W = sum |min(W, gradW)| / (F K)   (diagnostics.py:57)
template <typename T>
__global__ void kkt_w_residual(const T* __restrict__ W, const double* __restrict__ grad, int F,
                               int K, const double* __restrict__ resh_sum, size_t KN,
                               double* __restrict__ trace_kkt, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < F * K; i += blockDim.x)
    s += fabs(fmin(double(W[i]), grad[i]));
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    long long it = st->base + slot;
    trace_kkt[2 * (it - 1) + 0] = t / (double(F) * K);
    trace_kkt[2 * (it - 1) + 1] = *resh_sum / double(KN);
  }
}

static __global__ void advance_base(RunState* st, int n) { st->base += n; }

// --- layout conversion helpers (upload / download) -------------------------

// dst[r * ldd + c] = T(src[r * lds + c]) + kappa   (row-major convert)
template <typename S, typename T>
__global__ void convert_rows(const S* __restrict__ src, size_t lds, T* __restrict__ dst,
                             size_t ldd, int rows, size_t cols, double kappa) {
  size_t count = (size_t)rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t r = i / cols, c = i - r * cols;
    double v = double(src[r * lds + c]);
    dst[r * ldd + c] = kappa != 0.0 ? T(v + kappa) : T(v);
  }
}

// Data statistics for the input checks of DataMatrix / default_kappa
// (core.py:176-228): per-block [min, max, sum, non-finite count] of a rows x
// cols matrix (leading dimension lds), fp64, fixed-order tree reduction.
constexpr int STATS_BLOCKS = 296;
template <typename S>
__global__ void __launch_bounds__(256) stats_partial(const S* __restrict__ src, size_t lds, int rows,
                                                     size_t cols, double* __restrict__ part) {
  double mn = INFINITY, mx = -INFINITY, sm = 0.0, nf = 0.0;
  const size_t count = (size_t)rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    // contiguous rows (lds == cols, e.g. the factor checks): no 64-bit divide
    size_t j = i;
    if (lds != cols) {
      const size_t r = i / cols;
      j = r * lds + (i - r * cols);
    }
    const double v = double(src[j]);
    if (isfinite(v)) {
      mn = fmin(mn, v);
      mx = fmax(mx, v);
      sm += v;
    } else {
      nf += 1.0;
    }
  }
  __shared__ double red[4][256];
  red[0][threadIdx.x] = mn; red[1][threadIdx.x] = mx; red[2][threadIdx.x] = sm; red[3][threadIdx.x] = nf;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] = fmin(red[0][threadIdx.x], red[0][threadIdx.x + o]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + o]);
      red[2][threadIdx.x] += red[2][threadIdx.x + o];
      red[3][threadIdx.x] += red[3][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = red[threadIdx.x][0];
}
// fold the block partials (fixed order) into acc[4]; accumulate across calls
static __global__ void stats_final(const double* __restrict__ part, int nblk, double* acc, int first) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mn = first ? INFINITY : acc[0], mx = first ? -INFINITY : acc[1];
  double sm = first ? 0.0 : acc[2], nf = first ? 0.0 : acc[3];
  double cs = 0.0;
  for (int b = 0; b < nblk; ++b) {
    mn = fmin(mn, part[4 * b]);
    mx = fmax(mx, part[4 * b + 1]);
    cs += part[4 * b + 2];
    nf += part[4 * b + 3];
  }
  acc[0] = mn; acc[1] = mx; acc[2] = sm + cs; acc[3] = nf;
}

// K x N (fp64, row-major) -> N x K (T)
template <typename T>
__global__ void transpose_in(const double* __restrict__ src, int K, size_t N, T* __restrict__ dst) {
  size_t count = N * (size_t)K;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t n = i / K; int k = int(i - n * K);
    dst[i] = T(src[(size_t)k * N + n]);
  }
}

// N x K (T) -> K x N (fp64)
template <typename T>
__global__ void transpose_out(const T* __restrict__ src, int K, size_t N, double* __restrict__ dst) {
  size_t count = N * (size_t)K;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t k = i / N, n = i - k * N;
    dst[i] = double(src[n * K + k]);
  }
}

template <typename T>
__global__ void to_double(const T* __restrict__ src, size_t count, double* __restrict__ dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = double(src[i]);
}

template <typename T>
__global__ void from_double(const double* __restrict__ src, size_t count, T* __restrict__ dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = T(src[i]);
}

}  // namespace bnmf
