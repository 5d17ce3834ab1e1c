// Sparse KL (beta = 1) path: V in CSR (plus a CSC view for the column sums),
// fp32 factors, fp64 reductions, deterministic (no float atomics).
//
// Restates the dense beta = 1 updates at the nonzeros (the reference has no
// sparse kernel: it densifies, matrixio.py:115-128):
//   W_p = W~ * ((V/Vt) H~^T) / rowsum(H~)          updates.py:301-303
//   H_p = H~ * (W^T (V/Vt)) / colsum(W_p)            updates.py:325-327
//         (JMM: W^T with W = W~ and Vt = W~H~; BMM: W = W_p, Vt = W_p H~)
//   D(V | WH) = sum_nnz [x log(x/y) - x] + (1^T W)(H 1)   core.py:101 at x=0
// Per outer iteration (solver.py:301-319); rows of V (and of W) are local to
// the rank, H~ is replicated:
//   pass A  (CSR, warp per row)      y, z = x/y at the nonzeros, W_p row update,
//                                    per-block colsum / sum-of-squares of W_p
//   reduce A (+ allreduce 2K)        DenH = colsum(W_p), norms = ||W_p[:,k]||
//   pass B1 (CSC segments, warp each) partial H numerators: columns are cut
//                                    into segments of <= SP_SEG nonzeros so
//                                    that a Zipf-heavy column spreads over
//                                    many warps
//   pass B2 (column x k)             segment partials summed in order
//   (+ allreduce N x K of the numerators when rows are sharded)
//   pass B3 (column x k)             H_p = H~ * num/DenH, H~_p = H_p * norms,
//                                    per-block rowsum of H~_p (next DenW)
//   pass C  (CSR, warp per row)      W~_p = W_p / norms
//   finish                           rowsum(H~_p), dense objective term
// The nonzero part of the objective of iterate p needs W~_p H~_p at every
// nonzero, which is the product pass A of iteration p+1 forms anyway: pass A
// accumulates it there (bit for bit the sum a separate pass would give), and
// the trace row / stop rule of iterate p run right after it.  A stop at p
// skips the rest of slot p+1, so W~_p and H~_p stay the live iterate; one
// trailing objective-only slot finishes the last iteration.
//
// Warp layout of the nonzero passes: 4 groups of 8 lanes, one nonzero per
// group, each lane holding KPL consecutive k of the (KL = K rounded up to 32)
// padded factor rows, so a factor row is one coalesced 8-lane vector load and
// the dot product needs 3 shuffles.  Factor matrices are stored row-major with
// leading dimension KL (zero padded).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"
#include "small_kernels.cuh"

namespace bnmf {

constexpr int SP_THREADS = 256;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr int SP_KMAX = 128;
constexpr int SP_SEG = 2048;   // nonzeros per column segment (pass B1)
// Columns with more than SP_HEAVY nonzeros are also cut at row-tile
// boundaries (SP_TILE rows): their segments are ordered tile by tile, so the
// W~ rows they gather stay in L2 (one 16 MB tile of W~ at K = 64) instead of
// being fetched from HBM once per nonzero.
constexpr int SP_HEAVY = 2048;
// columns with more segments than this are summed by pass B2h (a block each)
constexpr int SP_B2_HEAVY = 64;
constexpr int SP_TILE = 131072;
constexpr int SP_SEG_H = 512;  // heavy-column segments (more warps per tile)
#ifndef BNMF_SP_U
#define BNMF_SP_U 4
#endif
constexpr int SP_U = BNMF_SP_U;   // nonzeros per 8-lane group in flight

struct SpArgs {
  int F, N, K, KL;
  const long long* indptr;
  const int* indices;
  const float* vals;
  const int* rowidx;           // CSC row index
  const int* perm;             // CSC position -> CSR position
  const long long* segptr;     // [S][2] CSC range of each segment
  const int* segcol;           // [S] column of each segment
  const int* colseg;           // [N + 1] each column's run in seglist
  const int* seglist;          // [S] segment ids of each column, in row order
  int S;
  const int* hcols;            // columns with > SP_B2_HEAVY segments (pass B2h)
  int NH;
  float* z;                    // per nonzero (CSR order)
  float* Wt;                   // W~ (F x KL)
  float* Wp;                   // W_p (F x KL)
  float* Ht;                   // H~ (N x KL)
  float* Hn;                   // H~_p (N x KL)
  float* part;                 // segment partials (S x KL)
  float* num;                  // H numerators (N x KL)
  const double* denw;          // rowsum(H~) (K)
  const double* denh;          // colsum(W_p) (K)
  const double* norms;         // ||W_p[:,k]|| (K)
  double* pa;                  // pass A partials [blocks][2K]: colsum, sumsq
  double* pb;                  // pass B3 partials [blocks][K]: rowsum(H~_p)
  double* pc;                  // pass C partials [blocks]
  int algorithm;
  Scalars sc;
};

template <int KPL>
__device__ __forceinline__ void ld_row(const float* p, float* v) {
#pragma unroll
  for (int i = 0; i < KPL; i += 4) {
    const float4 t = *reinterpret_cast<const float4*>(p + i);
    v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
  }
}
template <int KPL>
__device__ __forceinline__ void st_row(float* p, const float* v) {
#pragma unroll
  for (int i = 0; i < KPL; i += 4)
    *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}
// sum over the 8 lanes of a group (every lane of the group gets the total)
__device__ __forceinline__ float group_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  return v;
}

// iterate base+slot-1 is finished in slot `slot` (lagged objective)
__device__ __forceinline__ bool prev_live(const RunState* st, int slot) {
  const long long it = st->base + slot - 1;
  return it >= 1 && it <= st->stop_iter && it <= st->max_iter;
}

// ---- pass A: rows --------------------------------------------------------
template <int KPL>
__global__ void __launch_bounds__(SP_THREADS, 3) sp_pass_a(SpArgs a, const RunState* st, int slot) {
  const bool upd = iter_active(st, slot);   // W update of this iteration
  const bool objp = prev_live(st, slot);    // objective of the previous iterate
  if (!upd && !objp) return;
  // per-group running objective sums live in shared memory (registers are
  // what bounds the rows in flight)
  __shared__ double red[SP_THREADS / 8];
  if ((threadIdx.x & 7) == 0) red[threadIdx.x >> 3] = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, sl = lane & 7, k0 = sl * KPL;
  const int KL = a.KL;
  // 1 / max(rowsum H~, floor) per k in shared memory (not 8 fp64 registers per
  // thread: pass A is latency bound on the H~ gathers, and registers set how
  // many rows are in flight); the W_p column statistics are a separate pass
  __shared__ double s_rinv[SP_KMAX];
  for (int k = threadIdx.x; k < KL; k += blockDim.x)
    s_rinv[k] = k < a.K ? 1.0 / fmax(a.denw[k], a.sc.floor) : 0.0;
  __syncthreads();
  for (int f = blockIdx.x * SP_WARPS + warp; f < a.F; f += gridDim.x * SP_WARPS) {
    float w[KPL], num[KPL];
    ld_row<KPL>(a.Wt + size_t(f) * KL + k0, w);
#pragma unroll
    for (int i = 0; i < KPL; ++i) num[i] = 0.f;
    float rowacc = 0.f;
    const long long j0 = a.indptr[f], j1 = a.indptr[f + 1];
    for (long long jj = j0; jj < j1; jj += 4 * SP_U) {
      // SP_U nonzeros per group in flight: indices first, then the row gathers
      int n[SP_U];
      float x[SP_U], h[SP_U][KPL];
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        const long long j = jj + 4 * u + grp;
        n[u] = j < j1 ? a.indices[j] : 0;
        x[u] = j < j1 ? a.vals[j] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SP_U; ++u) ld_row<KPL>(a.Ht + size_t(n[u]) * KL + k0, h[u]);
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        const long long j = jj + 4 * u + grp;
        const bool ok = j < j1;
        float p = 0.f;
#pragma unroll
        for (int i = 0; i < KPL; ++i) p = fmaf(w[i], h[u][i], p);
        const float y = group_sum(p);
        const float zz = ok ? x[u] / y : 0.f;
        // x log(x / y) - x at the nonzero (core.py:101), iterate p-1
        if (objp && x[u] != 0.f) rowacc += x[u] * logf(zz) - x[u];
        if (upd && ok && sl == 0) a.z[j] = zz;
#pragma unroll
        for (int i = 0; i < KPL; ++i) num[i] = fmaf(zz, h[u][i], num[i]);
      }
    }
    if (objp && sl == 0) red[threadIdx.x >> 3] += double(rowacc);
#pragma unroll
    for (int i = 0; i < KPL; ++i) {   // groups 0..3 in a fixed tree
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 8);
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 16);
    }
    if (upd && grp == 0) {
      float wn[KPL];
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int k = k0 + i;
        wn[i] = 0.f;
        if (k < a.K) {
          const double r = double(num[i]) * s_rinv[k];
          wn[i] = float(double(w[i]) * apply_exponent<double>(r, a.sc.gamma));
        }
      }
      st_row<KPL>(a.Wp + size_t(f) * KL + k0, wn);
    }
  }
  if (objp) {   // per-block partial in a fixed order
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < SP_THREADS / 8; ++i) t += red[i];
      a.pc[blockIdx.x] = t;
    }
  }
}

// W_p column statistics: per-block fp64 partials of colsum and sum of squares
// over a fixed row assignment (block b: rows b*RP + r, stepping gridDim*RP),
// reduced in a fixed order -> deterministic
__global__ void __launch_bounds__(SP_THREADS) sp_colstats(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int KL = a.KL, RP = SP_THREADS / KL;
  const int k = threadIdx.x % KL, r = threadIdx.x / KL;
  double cs = 0.0, sq = 0.0;
  if (k < a.K && r < RP) {
    // 4 rows' loads in flight per step, added in row order
    const int stride = gridDim.x * RP;
    int f = blockIdx.x * RP + r;
    for (; f + 3 * stride < a.F; f += 4 * stride) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = a.Wp[size_t(f + u * stride) * KL + k];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double w = double(v[u]);
        cs += w;
        sq += w * w;
      }
    }
    for (; f < a.F; f += stride) {
      const double w = double(a.Wp[size_t(f) * KL + k]);
      cs += w;
      sq += w * w;
    }
  }
  __shared__ double red[2][SP_THREADS];
  red[0][threadIdx.x] = cs;
  red[1][threadIdx.x] = sq;
  __syncthreads();
  if (threadIdx.x < a.K) {
    double s0 = 0.0, s1 = 0.0;
    for (int rr = 0; rr < RP; ++rr) {
      s0 += red[0][rr * KL + threadIdx.x];
      s1 += red[1][rr * KL + threadIdx.x];
    }
    a.pa[size_t(blockIdx.x) * 2 * a.K + threadIdx.x] = s0;
    a.pa[size_t(blockIdx.x) * 2 * a.K + a.K + threadIdx.x] = s1;
  }
}

// ---- pass B1: column segments -> partial H numerators ----------------------
template <int KPL>
__global__ void __launch_bounds__(SP_THREADS) sp_pass_b1(SpArgs a, const RunState* st, int slot,
                                                          int s_begin, int s_end) {
  if (!iter_active(st, slot)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, sl = lane & 7, k0 = sl * KPL;
  const int KL = a.KL;
  const bool bmm = a.algorithm == BNMF_BMM;
  const float* W = bmm ? a.Wp : a.Wt;
  for (int s = s_begin + blockIdx.x * SP_WARPS + warp; s < s_end; s += gridDim.x * SP_WARPS) {
    const long long j0 = a.segptr[2 * size_t(s)], j1 = a.segptr[2 * size_t(s) + 1];
    float num[KPL], h[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) num[i] = 0.f;
    if (bmm) ld_row<KPL>(a.Ht + size_t(a.segcol[s]) * KL + k0, h);
    for (long long jj = j0; jj < j1; jj += 4 * SP_U) {
      int f[SP_U];
      float zx[SP_U], w[SP_U][KPL];
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        const long long j = jj + 4 * u + grp;
        const bool ok = j < j1;
        f[u] = ok ? a.rowidx[j] : 0;
        const int pj = ok ? a.perm[j] : 0;
        // JMM: the anchor's Z from pass A; BMM: the value (Z recomputed below)
        zx[u] = ok ? (bmm ? a.vals[pj] : a.z[pj]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SP_U; ++u) ld_row<KPL>(W + size_t(f[u]) * KL + k0, w[u]);
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        float zz = zx[u];
        if (bmm) {   // block update: Vt2 = W_p H~ at this nonzero (updates.py:173-181)
          float p = 0.f;
#pragma unroll
          for (int i = 0; i < KPL; ++i) p = fmaf(w[u][i], h[i], p);
          const float y = group_sum(p);
          zz = zx[u] != 0.f ? zx[u] / y : 0.f;
        }
#pragma unroll
        for (int i = 0; i < KPL; ++i) num[i] = fmaf(zz, w[u][i], num[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 8);
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 16);
    }
    if (grp == 0) st_row<KPL>(a.part + size_t(s) * KL + k0, num);
  }
}

// ---- pass B2: segment partials of each column, in order -------------------
__global__ void sp_pass_b2(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const size_t total = size_t(a.N) * a.KL;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total;
       t += size_t(gridDim.x) * blockDim.x) {
    const int n = int(t / a.KL), k = int(t - size_t(n) * a.KL);
    const int s0 = a.colseg[n], s1 = a.colseg[n + 1];
    if (s1 - s0 > SP_B2_HEAVY) continue;   // pass B2h
    float v = a.part[size_t(a.seglist[s0]) * a.KL + k];
    if (s1 - s0 > 1) {
      // same left-to-right order as a plain loop (bitwise identical), but the
      // segment ids and partials of 8 segments are loaded before any is added:
      // a Zipf-heavy column has thousands of segments, and a dependent
      // id -> partial -> add chain per segment made this pass latency bound
      double acc = double(v);
      int s = s0 + 1;
      for (; s + 8 <= s1; s += 8) {
        int id[8];
        float pv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) id[i] = a.seglist[s + i];
#pragma unroll
        for (int i = 0; i < 8; ++i) pv[i] = a.part[size_t(id[i]) * a.KL + k];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += double(pv[i]);
      }
      for (; s < s1; ++s) acc += double(a.part[size_t(a.seglist[s]) * a.KL + k]);
      v = float(acc);
    }
    a.num[t] = v;
  }
}

// ---- pass B2h: the Zipf-heavy columns, one block each ----------------------
// thread (k, p): p-th contiguous run of the column's segments after the first,
// summed in order; the runs are then added to the first segment in p order
// (a fixed order, so deterministic)
__global__ void __launch_bounds__(1024) sp_pass_b2h(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[1024];
  const int KL = a.KL, P = blockDim.x / KL;
  const int k = threadIdx.x % KL, p = threadIdx.x / KL;
  const int n = a.hcols[blockIdx.x];
  const int s0 = a.colseg[n], s1 = a.colseg[n + 1];
  const int L = s1 - s0 - 1, per = (L + P - 1) / P;
  double acc = 0.0;
  if (p < P) {
    int s = s0 + 1 + p * per;
    const int e = min(s1, s + per);
    for (; s + 8 <= e; s += 8) {
      int id[8];
      float pv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) id[i] = a.seglist[s + i];
#pragma unroll
      for (int i = 0; i < 8; ++i) pv[i] = a.part[size_t(id[i]) * KL + k];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += double(pv[i]);
    }
    for (; s < e; ++s) acc += double(a.part[size_t(a.seglist[s]) * KL + k]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (p == 0) {
    double t = double(a.part[size_t(a.seglist[s0]) * KL + k]);
    for (int q = 0; q < P; ++q) t += red[q * KL + k];
    a.num[size_t(n) * KL + k] = float(t);
  }
}

// ---- pass B3: H update, normalisation, rowsum partials ----------------------
// block = (SP_THREADS / KL) columns x KL k; grid-stride over column groups
__global__ void __launch_bounds__(SP_THREADS) sp_pass_b3(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int KL = a.KL, cpb = SP_THREADS / KL;
  const int k = threadIdx.x % KL, c = threadIdx.x / KL;
  __shared__ double red[SP_THREADS];
  double rs = 0.0;
  if (c < cpb && k < a.K) {
    const double dinv = 1.0 / fmax(a.denh[k], a.sc.floor), nk = a.norms[k];
    for (int n = blockIdx.x * cpb + c; n < a.N; n += gridDim.x * cpb) {
      const size_t t = size_t(n) * KL + k;
      const double r = double(a.num[t]) * dinv;
      const double hp = double(a.Ht[t]) * apply_exponent<double>(r, a.sc.gamma);
      const float hn = float(hp * nk);
      a.Hn[t] = hn;
      rs += double(hn);
    }
  }
  red[threadIdx.x] = rs;
  __syncthreads();
  if (threadIdx.x < a.K) {
    double s = 0.0;
    for (int cc = 0; cc < cpb; ++cc) s += red[cc * KL + threadIdx.x];
    a.pb[size_t(blockIdx.x) * a.K + threadIdx.x] = s;
  }
}

// ---- pass C: normalise W ------------------------------------------------
// W~_p = W_p / norms, float4 per thread, rows grid-strided (no index divides)
__global__ void __launch_bounds__(SP_THREADS) sp_pass_c(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int KL4 = a.KL >> 2, rpb = SP_THREADS / KL4;
  const int k4 = threadIdx.x % KL4, r = threadIdx.x / KL4;
  if (r >= rpb) return;
  double ninv[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = 4 * k4 + i;
    ninv[i] = k < a.K ? 1.0 / a.norms[k] : 0.0;
  }
  const bool pad[4] = {4 * k4 >= a.K, 4 * k4 + 1 >= a.K, 4 * k4 + 2 >= a.K, 4 * k4 + 3 >= a.K};
  for (size_t f = blockIdx.x * size_t(rpb) + r; f < size_t(a.F); f += size_t(gridDim.x) * rpb) {
    const float4 w = *reinterpret_cast<const float4*>(a.Wp + f * a.KL + 4 * k4);
    float4 o;
    o.x = pad[0] ? 0.f : float(double(w.x) * ninv[0]);
    o.y = pad[1] ? 0.f : float(double(w.y) * ninv[1]);
    o.z = pad[2] ? 0.f : float(double(w.z) * ninv[2]);
    o.w = pad[3] ? 0.f : float(double(w.w) * ninv[3]);
    *reinterpret_cast<float4*>(a.Wt + f * a.KL + 4 * k4) = o;
  }
}


// ---- KKT residuals of the finished iterate (diagnostics.py:46-59 at beta = 1) -----------
// grad_core = 1 - V / (W~ H~) (all entries; 1 where V = 0), so
//   grad_W = rowsum(H~) - (V / Vt) H~^T      rows:    the SDDMM of pass A on (W~_p, H~_p)
//   grad_H = colsum(W~) - W~^T (V / Vt)      columns: pass B1/B2 in its joint form
// Untimed like the reference's (the loop timer is moved past them).
template <int KPL>
__global__ void __launch_bounds__(SP_THREADS, 3) sp_kkt_a(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[SP_THREADS / 8];
  __shared__ double s_den[SP_KMAX];
  if ((threadIdx.x & 7) == 0) red[threadIdx.x >> 3] = 0.0;
  for (int k = threadIdx.x; k < a.KL; k += blockDim.x) s_den[k] = k < a.K ? a.denw[k] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane >> 3, sl = lane & 7, k0 = sl * KPL;
  const int KL = a.KL;
  for (int f = blockIdx.x * SP_WARPS + warp; f < a.F; f += gridDim.x * SP_WARPS) {
    float w[KPL], num[KPL];
    ld_row<KPL>(a.Wt + size_t(f) * KL + k0, w);
#pragma unroll
    for (int i = 0; i < KPL; ++i) num[i] = 0.f;
    const long long j0 = a.indptr[f], j1 = a.indptr[f + 1];
    for (long long jj = j0; jj < j1; jj += 4 * SP_U) {
      int n[SP_U];
      float x[SP_U], h[SP_U][KPL];
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        const long long j = jj + 4 * u + grp;
        n[u] = j < j1 ? a.indices[j] : 0;
        x[u] = j < j1 ? a.vals[j] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SP_U; ++u) ld_row<KPL>(a.Ht + size_t(n[u]) * KL + k0, h[u]);
#pragma unroll
      for (int u = 0; u < SP_U; ++u) {
        const long long j = jj + 4 * u + grp;
        const bool ok = j < j1;
        float p = 0.f;
#pragma unroll
        for (int i = 0; i < KPL; ++i) p = fmaf(w[i], h[u][i], p);
        const float y = group_sum(p);
        const float zz = ok ? x[u] / y : 0.f;
        if (ok && sl == 0) a.z[j] = zz;
#pragma unroll
        for (int i = 0; i < KPL; ++i) num[i] = fmaf(zz, h[u][i], num[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 8);
      num[i] += __shfl_xor_sync(0xffffffffu, num[i], 16);
    }
    {
      // the row's 8 lanes of group 0 hold its KL entries; fixed shuffle tree, lane 0 adds
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < KPL; ++i)
        if (k0 + i < a.K) t += fabs(fmin(double(w[i]), s_den[k0 + i] - double(num[i])));
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      if (lane == 0) red[threadIdx.x >> 3] += t;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < SP_THREADS / 8; ++i) t += red[i];
    a.pc[blockIdx.x] = t;
  }
}

// sum_nk |min(H~[n,k], colsum(W~)[k] - num[n,k])| per block (same thread map as pass B3)
__global__ void __launch_bounds__(SP_THREADS) sp_kkt_h(SpArgs a, const double* comm_a,
                                                       const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int KL = a.KL, cpb = SP_THREADS / KL;
  const int k = threadIdx.x % KL, c = threadIdx.x / KL;
  __shared__ double red[SP_THREADS];
  double rs = 0.0;
  if (c < cpb && k < a.K) {
    const double cs = comm_a[k] / a.norms[k];   // colsum(W_p) / ||W_p[:, k]|| = colsum(W~_p)
    for (int n = blockIdx.x * cpb + c; n < a.N; n += gridDim.x * cpb) {
      const size_t t = size_t(n) * KL + k;
      rs += fabs(fmin(double(a.Ht[t]), cs - double(a.num[t])));
    }
  }
  red[threadIdx.x] = rs;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < SP_THREADS; ++i) s += red[i];
    a.pb[blockIdx.x] = s;
  }
}
__global__ void sp_kkt_sum(const double* pc, int GC, const double* pb, int GB, double* out2,
                           RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  double s = 0.0;
  for (int g = 0; g < GC; ++g) s += pc[g];
  out2[0] = s;
  s = 0.0;
  for (int g = 0; g < GB; ++g) s += pb[g];
  out2[1] = s;
}
__global__ void sp_kkt_finish(const double* in2, double fk, double kn, double* tr_kkt,
                              RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const long long it = st->base + slot;
  tr_kkt[2 * (it - 1) + 0] = in2[0] / fk;
  tr_kkt[2 * (it - 1) + 1] = in2[1] / kn;
  // the loop timer does not see the KKT passes (solver.py:312-314)
  st->t_last += globaltimer() - st->t_begin;
}
__global__ void sp_kkt_begin(RunState* st, int slot) {
  if (iter_active(st, slot)) st->t_begin = globaltimer();
}

// fixed-order reduction of the pass-A partials -> comm[0:2K] (colsum, sumsq)
__global__ void sp_reduce_a(const double* pa, int G, int K, double* comm, const RunState* st,
                            int slot) {
  if (!iter_active(st, slot)) return;
  // block i sums output i: thread t takes partials t, t + 256, ... in order,
  // then a fixed shared-memory tree (deterministic)
  __shared__ double red[256];
  const int i = blockIdx.x;
  double s = 0.0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) s += pa[size_t(g) * 2 * K + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) comm[i] = red[0];
}
// DenH = colsum(W_p), norms = sqrt(sum_f W_p^2)  (after the allreduce)
__global__ void sp_post_a(const double* comm, int K, double* denh, double* norms,
                          const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    denh[k] = comm[k];
    norms[k] = sqrt(comm[K + k]);
  }
}
// rowsum(H~_p) -> denw (next iteration); global dense part of the objective of
// iterate p, sum_k colsum(W~_p) rowsum(H~_p) -> comm_obj[1]
__global__ void sp_finish(const double* pb, int GB, int K, const double* comm_a,
                          const double* norms, double* denw, double* comm_obj, const RunState* st,
                          int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double part[SP_KMAX];
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double rs = 0.0;
    int g = 0;
    for (; g + 7 < GB; g += 8) {   // 8 loads in flight, added in order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = pb[size_t(g + u) * K + k];
#pragma unroll
      for (int u = 0; u < 8; ++u) rs += v[u];
    }
    for (; g < GB; ++g) rs += pb[size_t(g) * K + k];
    denw[k] = rs;
    part[k] = (comm_a[k] / norms[k]) * rs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double dense = 0.0;
    for (int k = 0; k < K; ++k) dense += part[k];
    comm_obj[1] = dense;
  }
}
// local nonzero part of the objective of iterate base+slot-1 (pass A partials)
// -> comm_obj[0]
__global__ void sp_obj_prev(const double* pc, int GC, double* comm_obj, const RunState* st,
                            int slot) {
  if (!prev_live(st, slot)) return;
  double s = 0.0;
  int g = 0;
  for (; g + 7 < GC; g += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = pc[g + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; g < GC; ++g) s += pc[g];
  comm_obj[0] = s;
}
__global__ void sp_total_obj(double* comm_obj, const RunState* st, int slot) {
  if (!prev_live(st, slot)) return;
  comm_obj[2] = comm_obj[0] + comm_obj[1];
}
__global__ void sp_begin(RunState* st, int slot) {
  if (st->base + slot == 1) st->t_last = globaltimer();
}
// trace row + stop rule of iterate base+slot-1 (finish_iter, solver.py:309-319,
// 174-180); the timer accumulates from the previous finish
__global__ void sp_finish_prev(RunState* st, int slot, const double* __restrict__ obj,
                               double* __restrict__ trace_obj, double* __restrict__ trace_sec,
                               double tol) {
  if (!prev_live(st, slot)) return;
  const long long it = st->base + slot - 1;
  const double o = *obj;
  bool stop = false;
  if (it > 1) {
    const double prev = st->prev_obj;
    if (o == prev) stop = true;
    else if (o <= 0.0) stop = false;
    else stop = (prev - o) / o <= tol;
  }
  const unsigned long long t = globaltimer();
  st->elapsed += double(t - st->t_last) * 1e-9;
  st->t_last = t;
  trace_obj[it - 1] = o;
  trace_sec[it - 1] = st->elapsed;
  st->prev_obj = o;
  st->iters_done = it;
#ifdef BNMF_X_NOSTOP
  stop = false;
#endif
  if (stop) { st->stop_iter = it; st->converged = 1; }
}
// rowsum(H~) of the initial iterate: per-block partials, then a fixed-order sum
__global__ void sp_rowsum_part(const float* Ht, int N, int KL, int K, double* pb) {
  const int cpb = SP_THREADS / KL;
  const int k = threadIdx.x % KL, c = threadIdx.x / KL;
  __shared__ double red[SP_THREADS];
  double rs = 0.0;
  if (c < cpb && k < K)
    for (int n = blockIdx.x * cpb + c; n < N; n += gridDim.x * cpb) rs += double(Ht[size_t(n) * KL + k]);
  red[threadIdx.x] = rs;
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int cc = 0; cc < cpb; ++cc) s += red[cc * KL + threadIdx.x];
    pb[size_t(blockIdx.x) * K + threadIdx.x] = s;
  }
}
__global__ void sp_rowsum_final(const double* pb, int GB, int K, double* denw) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < GB; ++g) s += pb[size_t(g) * K + k];
    denw[k] = s;
  }
}
// K-strided fp64 rows <-> KL-padded fp32 rows
__global__ void sp_pad_in(const double* __restrict__ src, size_t rows, int K, int KL,
                          float* __restrict__ dst) {
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < rows * KL;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t r = t / KL;
    const int k = int(t - r * KL);
    dst[t] = k < K ? float(src[r * K + k]) : 0.f;
  }
}
// H (K x N, row-major fp64) -> H~ (N x KL fp32)
__global__ void sp_transpose_in(const double* __restrict__ src, size_t N, int K, int KL,
                                float* __restrict__ dst) {
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < N * KL;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t n = t / KL;
    const int k = int(t - n * KL);
    dst[t] = k < K ? float(src[size_t(k) * N + n]) : 0.f;
  }
}
__global__ void sp_pad_out(const float* __restrict__ src, size_t rows, int K, int KL,
                           double* __restrict__ dst) {
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < rows * K;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t r = t / K;
    const int k = int(t - r * K);
    dst[t] = double(src[r * KL + k]);
  }
}
__global__ void sp_transpose_out(const float* __restrict__ src, size_t N, int K, int KL,
                                 double* __restrict__ dst) {
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < N * K;
       t += size_t(gridDim.x) * blockDim.x) {
    const int k = int(t / N);
    const size_t n = t - size_t(k) * N;
    dst[t] = double(src[n * KL + k]);
  }
}

#define SCK(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      return fail(BNMF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                               \
  } while (0)

struct SparseEngine : EngineBase {
  int F = 0, N = 0, K = 0, KL = 32, S = 0;
  long long nnz = 0;
  long long* indptr = nullptr;
  int* indices = nullptr;
  float* vals = nullptr;
  int* rowidx = nullptr;
  int* perm = nullptr;
  long long* segptr = nullptr;
  int* segcol = nullptr;
  int* colseg = nullptr;
  int* seglist = nullptr;
  int* hcols = nullptr;
  int NH = 0;
  std::vector<int> tstart;   // [ntile + 2] B1 launch ranges of segments
  float *z = nullptr, *Wt = nullptr, *Wp = nullptr, *Ht = nullptr, *Hn = nullptr;
  float *part = nullptr, *num = nullptr;
  double *denw = nullptr, *denh = nullptr, *norms = nullptr, *pa = nullptr, *pb = nullptr,
         *pc = nullptr, *comm = nullptr;
  double *tr_obj = nullptr, *tr_sec = nullptr, *tr_kkt = nullptr;
  int64_t tr_cap = 0;
  RunState* st = nullptr;
  RunState* st_host = nullptr;
  int GA = 1, GB1 = 1, GB3 = 1, GS = 1, nsm = 148;
  bnmf_params p{};
  Scalars sc{};
  bool begun = false;
  cudaGraphExec_t gexec = nullptr;
  int gchunk = 0;
  int launches = 0;

  SparseEngine(int dev, cudaStream_t s) {
    device = dev; dtype = BNMF_FP32; stream = s;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  ~SparseEngine() override {
    if (gexec) cudaGraphExecDestroy(gexec);
    void* ptrs[] = {indptr, indices, vals, rowidx, perm, segptr, segcol, colseg, seglist, hcols, z, Wt, Wp, Ht,
                    Hn, part, num, denw, denh, norms, pa, pb, pc, comm, tr_obj, tr_sec, tr_kkt, st};
    for (void* q : ptrs) if (q) cudaFree(q);
    if (st_host) cudaFreeHost(st_host);
    if (comm_nccl) ncclCommDestroy(comm_nccl);
    if (stream) cudaStreamDestroy(stream);
  }

  int set_dense(const void*, int, int, int64_t, int64_t, int64_t, double) override {
    return fail(BNMF_E_STATE, "context holds a sparse matrix");
  }

  template <typename Tp>
  int upload(Tp** dst, const void* src, size_t count, int on_dev) {
    if (*dst) SCK(cudaFree(*dst));
    *dst = nullptr;
    SCK(cudaMalloc(dst, std::max<size_t>(count, 1) * sizeof(Tp)));
    if (count)
      SCK(cudaMemcpyAsync(*dst, src, count * sizeof(Tp),
                          on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    return 0;
  }

  int set_csr(const long long* ip, const int* ix, const float* v, const long long* cp,
              const int* ri, const int* pm, int64_t F_, int64_t N_, int64_t nnz_, int on_dev) {
    SCK(cudaSetDevice(device));
    if (F_ < 1 || N_ < 1 || nnz_ < 0 || F_ > INT_MAX || N_ > INT_MAX)
      return fail(BNMF_E_ARG, "bad sparse shape");
    F = int(F_); N = int(N_); nnz = nnz_;
    int rc;
    if ((rc = upload(&indptr, ip, size_t(F) + 1, on_dev))) return rc;
    if ((rc = upload(&indices, ix, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&vals, v, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&rowidx, ri, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&perm, pm, size_t(nnz), on_dev))) return rc;
    // column segments (every column gets >= 1): light columns are cut every
    // SP_SEG nonzeros; heavy ones also at row-tile boundaries, and their
    // segments come first, tile by tile (W~ row locality in pass B1)
    std::vector<long long> hcp(size_t(N) + 1);
    std::vector<int> hri;
    const int* rip = ri;
    if (on_dev) {
      hri.resize(size_t(nnz));
      SCK(cudaMemcpyAsync(hcp.data(), cp, hcp.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                          stream));
      if (nnz) SCK(cudaMemcpyAsync(hri.data(), ri, size_t(nnz) * sizeof(int), cudaMemcpyDeviceToHost,
                                   stream));
      SCK(cudaStreamSynchronize(stream));
      rip = hri.data();
    } else {
      std::memcpy(hcp.data(), cp, hcp.size() * sizeof(long long));
    }
    const int ntile = (F + SP_TILE - 1) / SP_TILE;
    struct Seg { long long a0, a1; int col, tile; };
    std::vector<Seg> heavy, light;
    for (int n = 0; n < N; ++n) {
      const long long a0 = hcp[n], a1 = hcp[n + 1];
      if (a1 - a0 > SP_HEAVY) {
        long long s = a0;
        for (int t = 0; t < ntile && s < a1; ++t) {
          const int rend = int(std::min<long long>(F, (long long)(t + 1) * SP_TILE));
          const long long e = std::lower_bound(rip + s, rip + a1, rend) - rip;
          for (long long q = s; q < e; q += SP_SEG_H) heavy.push_back({q, std::min(e, q + SP_SEG_H), n, t});
          s = e;
        }
      } else {
        long long q = a0;
        do {
          light.push_back({q, std::min(a1, q + SP_SEG), n, 0});
          q += SP_SEG;
        } while (q < a1);
      }
    }
    std::stable_sort(heavy.begin(), heavy.end(),
                     [](const Seg& x, const Seg& y) { return x.tile < y.tile; });
    std::vector<Seg> all;
    all.reserve(heavy.size() + light.size());
    all.insert(all.end(), heavy.begin(), heavy.end());
    all.insert(all.end(), light.begin(), light.end());
    S = int(all.size());
    // B1 launch ranges: the heavy segments of each row tile, then all light ones
    tstart.assign(size_t(ntile) + 2, 0);
    for (const Seg& g : heavy) ++tstart[g.tile + 1];
    for (int t = 0; t < ntile; ++t) tstart[t + 1] += tstart[t];
    tstart[ntile + 1] = S;
    std::vector<int> scol(S), cs(size_t(N) + 1, 0), sl(S);
    for (int i = 0; i < S; ++i) { scol[i] = all[i].col; ++cs[all[i].col + 1]; }
    for (int n = 0; n < N; ++n) cs[n + 1] += cs[n];
    {
      // per column, its segments in increasing row order (= increasing a0)
      std::vector<int> fill(cs.begin(), cs.end() - 1);
      std::vector<int> order(S);
      for (int i = 0; i < S; ++i) order[i] = i;
      std::sort(order.begin(), order.end(), [&](int x, int y) {
        return all[x].col != all[y].col ? all[x].col < all[y].col : all[x].a0 < all[y].a0;
      });
      for (int i = 0; i < S; ++i) sl[fill[all[order[i]].col]++] = order[i];
    }
    // [begin, end) of each segment (no longer contiguous in CSC order)
    std::vector<long long> spe(2 * size_t(S));
    for (int i = 0; i < S; ++i) { spe[2 * size_t(i)] = all[i].a0; spe[2 * size_t(i) + 1] = all[i].a1; }
    if ((rc = upload(&segptr, spe.data(), spe.size(), 0))) return rc;
    if ((rc = upload(&segcol, scol.data(), scol.size(), 0))) return rc;
    if ((rc = upload(&colseg, cs.data(), cs.size(), 0))) return rc;
    if ((rc = upload(&seglist, sl.data(), sl.size(), 0))) return rc;
    {
      std::vector<int> hc;
      for (int n = 0; n < N; ++n)
        if (cs[n + 1] - cs[n] > SP_B2_HEAVY) hc.push_back(n);
      NH = int(hc.size());
      if ((rc = upload(&hcols, hc.data(), hc.size(), 0))) return rc;
    }
    if (z) SCK(cudaFree(z));
    z = nullptr;
    SCK(cudaMalloc(&z, std::max<size_t>(nnz, 1) * sizeof(float)));
    if (!st) {
      SCK(cudaMalloc(&st, sizeof(RunState)));
      SCK(cudaMallocHost(&st_host, sizeof(RunState)));
    }
    SCK(cudaStreamSynchronize(stream));   // host vectors above are the copy sources
    K = 0;
    begun = false;
    return 0;
  }

  int set_factors(const double* w, const double* h, int64_t K_, int on_dev) override {
    if (!indptr) return fail(BNMF_E_STATE, "set_csr must precede set_factors");
    if (K_ < 1 || K_ > SP_KMAX) return fail(BNMF_E_UNSUPPORTED, "sparse path supports rank 1..128");
    SCK(cudaSetDevice(device));
    if (K != K_) {
      float** fp[] = {&Wt, &Wp, &Ht, &Hn, &part, &num};
      for (float** q : fp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      double** dp[] = {&denw, &denh, &norms, &pa, &pb, &pc, &comm};
      for (double** q : dp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      K = int(K_);
      KL = (K + 31) / 32 * 32;
      if (KL == 96) KL = 128;   // KPL in {4, 8, 16}
      SCK(cudaMalloc(&Wt, size_t(F) * KL * sizeof(float)));
      SCK(cudaMalloc(&Wp, size_t(F) * KL * sizeof(float)));
      SCK(cudaMalloc(&Ht, size_t(N) * KL * sizeof(float)));
      SCK(cudaMalloc(&Hn, size_t(N) * KL * sizeof(float)));
      SCK(cudaMalloc(&part, size_t(S) * KL * sizeof(float)));
      SCK(cudaMalloc(&num, size_t(N) * KL * sizeof(float)));
      SCK(cudaMemset(Hn, 0, size_t(N) * KL * sizeof(float)));
      SCK(cudaMemset(Wp, 0, size_t(F) * KL * sizeof(float)));
      GA = std::max(1, std::min((F + SP_WARPS - 1) / SP_WARPS, nsm * 8));
      GB1 = std::max(1, std::min((S + SP_WARPS - 1) / SP_WARPS, nsm * 8));
      const int cpb = SP_THREADS / KL;
      GB3 = std::max(1, std::min((N + cpb - 1) / cpb, nsm * 4));
      SCK(cudaMalloc(&denw, K * sizeof(double)));
      SCK(cudaMalloc(&denh, K * sizeof(double)));
      SCK(cudaMalloc(&norms, K * sizeof(double)));
      GS = std::max(1, std::min((F + SP_THREADS / KL - 1) / (SP_THREADS / KL), nsm * 4));
      SCK(cudaMalloc(&pa, size_t(GS) * 2 * K * sizeof(double)));
      SCK(cudaMalloc(&pb, size_t(GB3) * K * sizeof(double)));
      SCK(cudaMalloc(&pc, size_t(GA) * sizeof(double)));
      SCK(cudaMalloc(&comm, (2 * K + 8) * sizeof(double)));
    }
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    double* stg;
    SCK(cudaMalloc(&stg, std::max(fk, nk) * sizeof(double)));
    SCK(cudaMemcpyAsync(stg, w, fk * sizeof(double),
                        on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    sp_pad_in<<<nsm * 8, 256, 0, stream>>>(stg, size_t(F), K, KL, Wt);
    SCK(cudaMemcpyAsync(stg, h, nk * sizeof(double),
                        on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    sp_transpose_in<<<nsm * 8, 256, 0, stream>>>(stg, size_t(N), K, KL, Ht);
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(stream));
    SCK(cudaFree(stg));
    begun = false;
    return 0;
  }

  SpArgs args() {
    SpArgs a;
    a.F = F; a.N = N; a.K = K; a.KL = KL;
    a.indptr = indptr; a.indices = indices; a.vals = vals;
    a.rowidx = rowidx; a.perm = perm;
    a.segptr = segptr; a.segcol = segcol; a.colseg = colseg; a.seglist = seglist; a.S = S;
    a.hcols = hcols; a.NH = NH;
    a.z = z;
    a.Wt = Wt; a.Wp = Wp; a.Ht = Ht; a.Hn = Hn; a.part = part; a.num = num;
    a.denw = denw; a.denh = denh; a.norms = norms;
    a.pa = pa; a.pb = pb; a.pc = pc;
    a.algorithm = p.algorithm; a.sc = sc;
    return a;
  }

  int begin(const bnmf_params* pp, int64_t max_iters) override {
    if (!Wt) return fail(BNMF_E_STATE, "factors must be set before begin");
    if (pp->beta != 1.0) return fail(BNMF_E_UNSUPPORTED, "sparse path implements beta = 1 (KL)");
    if (pp->kappa != 0.0) return fail(BNMF_E_UNSUPPORTED, "sparse path needs kappa = 0");
    if (pp->sub_iters != 1 || pp->sub_iters_w > 1 || pp->sub_iters_h > 1)
      return fail(BNMF_E_UNSUPPORTED, "sparse path implements one sub-iteration");
    SCK(cudaSetDevice(device));
    p = *pp;
    sc.beta = p.beta; sc.gamma = p.gamma; sc.kappa = 0.0; sc.floor = p.floor; sc.tol = p.tol;
    active_schedule = BNMF_SCHED_REFERENCE;
    if (tr_cap < max_iters) {
      double** dp[] = {&tr_obj, &tr_sec, &tr_kkt};
      for (double** q : dp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      SCK(cudaMalloc(&tr_obj, size_t(max_iters) * sizeof(double)));
      SCK(cudaMalloc(&tr_sec, size_t(max_iters) * sizeof(double)));
      SCK(cudaMalloc(&tr_kkt, size_t(max_iters) * 2 * sizeof(double)));
      tr_cap = max_iters;
    }
    SCK(cudaMemsetAsync(tr_kkt, 0xff, size_t(max_iters) * 2 * sizeof(double), stream));
    RunState h{};
    h.base = 1;
    h.stop_iter = LLONG_MAX;
    h.max_iter = max_iters;
    *st_host = h;
    SCK(cudaMemcpyAsync(st, st_host, sizeof(RunState), cudaMemcpyHostToDevice, stream));
    enqueued = 0;
    sp_rowsum_part<<<GB3, SP_THREADS, 0, stream>>>(Ht, N, KL, K, pb);
    sp_rowsum_final<<<1, 128, 0, stream>>>(pb, GB3, K, denw);
    SCK(cudaGetLastError());
    if (gexec) { SCK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    SCK(cudaStreamSynchronize(stream));
    begun = true;
    return 0;
  }

  int allreduce(void* buf, size_t count, ncclDataType_t t) {
    if (nranks > 1) {
      ncclResult_t r = ncclAllReduce(buf, buf, count, t, ncclSum, comm_nccl, stream);
      if (r != ncclSuccess) return fail(BNMF_E_NCCL, ncclGetErrorString(r));
      launches += 1;
    }
    return 0;
  }

  template <int KPL>
  void launch_rows_a(const SpArgs& a, int slot) {
    sp_pass_a<KPL><<<GA, SP_THREADS, 0, stream>>>(a, st, slot);
  }
  template <int KPL>
  void launch_b1(const SpArgs& a, int slot) {
    // one launch per row tile (every warp gathers W~ rows of the same tile,
    // which stay in L2), then the light columns
    for (size_t t = 0; t + 1 < tstart.size(); ++t) {
      const int s0 = tstart[t], s1 = tstart[t + 1];
      if (s1 <= s0) continue;
      const int g = std::max(1, std::min((s1 - s0 + SP_WARPS - 1) / SP_WARPS, GB1));
      sp_pass_b1<KPL><<<g, SP_THREADS, 0, stream>>>(a, st, slot, s0, s1);
      ++launches;
    }
  }

  void dispatch(int which, const SpArgs& a, int slot) {
    const int kpl = KL / 8;
    if (which == 0) {
      if (kpl == 4) launch_rows_a<4>(a, slot);
      else if (kpl == 8) launch_rows_a<8>(a, slot);
      else launch_rows_a<16>(a, slot);
    } else if (which == 1) {
      if (kpl == 4) launch_b1<4>(a, slot);
      else if (kpl == 8) launch_b1<8>(a, slot);
      else launch_b1<16>(a, slot);
    } else {
      sp_pass_c<<<nsm * 8, SP_THREADS, 0, stream>>>(a, st, slot);
    }
  }

  // KKT residuals of iterate base+slot: W~_p = Wt (pass C done), H~_p = Hn (before the swap),
  // rowsum(H~_p) = denw (sp_finish done), colsum(W~_p) = comm[k] / norms[k]
  int enqueue_kkt(const SpArgs& a, int slot) {
    SpArgs k = a;
    k.Ht = Hn;
    k.algorithm = BNMF_JMM;   // pass B1 in its joint form: W~^T Z with the Z written below
    sp_kkt_begin<<<1, 1, 0, stream>>>(st, slot);
    const int kpl = KL / 8;
    if (kpl == 4) sp_kkt_a<4><<<GA, SP_THREADS, 0, stream>>>(k, st, slot);
    else if (kpl == 8) sp_kkt_a<8><<<GA, SP_THREADS, 0, stream>>>(k, st, slot);
    else sp_kkt_a<16><<<GA, SP_THREADS, 0, stream>>>(k, st, slot);
    dispatch(1, k, slot);
    sp_pass_b2<<<nsm * 8, 256, 0, stream>>>(k, st, slot);
    if (NH > 0) {
      sp_pass_b2h<<<NH, 1024, 0, stream>>>(k, st, slot);
      ++launches;
    }
    SCK(cudaGetLastError());
    launches += 3;
    if (int rc = allreduce(num, size_t(N) * KL, ncclFloat)) return rc;
    sp_kkt_h<<<GB3, SP_THREADS, 0, stream>>>(k, comm, st, slot);
    double* k2 = comm + 2 * K + 4;
    sp_kkt_sum<<<1, 1, 0, stream>>>(pc, GA, pb, GB3, k2, st, slot);
    SCK(cudaGetLastError());
    launches += 2;
    if (int rc = allreduce(k2, 1, ncclDouble)) return rc;   // rows (res_W) are sharded
    const double fg = double(nranks > 1 ? n_global : F);
    sp_kkt_finish<<<1, 1, 0, stream>>>(k2, fg * K, double(K) * N, tr_kkt, st, slot);
    SCK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  int enqueue_iteration(int slot) {
    SpArgs a = args();
    double* cobj = comm + 2 * K;
    sp_begin<<<1, 1, 0, stream>>>(st, slot);
    dispatch(0, a, slot);   // W update of this iteration + objective of the previous iterate
    sp_obj_prev<<<1, 1, 0, stream>>>(pc, GA, cobj, st, slot);
    SCK(cudaGetLastError());
    launches += 3;
    if (int rc = allreduce(cobj, 1, ncclDouble)) return rc;   // nonzero part only
    sp_total_obj<<<1, 1, 0, stream>>>(cobj, st, slot);
    sp_finish_prev<<<1, 1, 0, stream>>>(st, slot, cobj + 2, tr_obj, tr_sec, sc.tol);
    sp_colstats<<<GS, SP_THREADS, 0, stream>>>(a, st, slot);
    sp_reduce_a<<<2 * K, 256, 0, stream>>>(pa, GS, K, comm, st, slot);
    SCK(cudaGetLastError());
    launches += 4;
    if (int rc = allreduce(comm, 2 * size_t(K), ncclDouble)) return rc;
    sp_post_a<<<1, 128, 0, stream>>>(comm, K, denh, norms, st, slot);
    dispatch(1, a, slot);
    sp_pass_b2<<<nsm * 8, 256, 0, stream>>>(a, st, slot);
    if (NH > 0) {
      sp_pass_b2h<<<NH, 1024, 0, stream>>>(a, st, slot);
      ++launches;
    }
    SCK(cudaGetLastError());
    launches += 3;
    // rows are sharded: every rank holds a partial H numerator of its rows
    if (int rc = allreduce(num, size_t(N) * KL, ncclFloat)) return rc;
    sp_pass_b3<<<GB3, SP_THREADS, 0, stream>>>(a, st, slot);
    dispatch(2, a, slot);
    sp_finish<<<1, 128, 0, stream>>>(pb, GB3, K, comm, norms, denw, cobj, st, slot);
    SCK(cudaGetLastError());
    launches += 3;
    if (p.compute_kkt) {
      if (int rc = enqueue_kkt(a, slot)) return rc;
    }
    // H~_p becomes the next iterate
    std::swap(Ht, Hn);
    SCK(cudaGetLastError());
    launches += 2;
    return 0;
  }

  int capture(int chunk) {
    if (gexec && gchunk == chunk) return 0;
    if (gexec) { SCK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    if (chunk % 2) return fail(BNMF_E_STATE, "graph chunk must be even (H~ ping-pong)");
    cudaGraph_t g;
    SCK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    int l0 = launches, rc = 0;
    for (int j = 0; j < chunk && rc == 0; ++j) rc = enqueue_iteration(j);
    if (rc == 0) advance_base<<<1, 1, 0, stream>>>(st, chunk);
    cudaError_t ec = cudaStreamEndCapture(stream, &g);
    if (rc) return rc;
    if (ec != cudaSuccess) return fail(BNMF_E_CUDA, cudaGetErrorString(ec));
    launches_per_iter = (launches - l0) / chunk;
    SCK(cudaGraphInstantiate(&gexec, g, 0));
    SCK(cudaGraphDestroy(g));
    gchunk = chunk;
    return 0;
  }

  int prepare(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    SCK(cudaSetDevice(device));
    return n >= 16 ? capture(16) : 0;
  }

  // Inactive iterations (after the stop) skip every kernel, but the host-side
  // H~ ping-pong still swaps; the live iterate is tracked by parity of the
  // number of enqueued iterations, so the step count is kept even around a
  // graph launch and an inactive trailing iteration swaps back harmlessly:
  // the last ACTIVE iteration wrote Hn before the swap, and get_factors reads
  // the buffer that holds iterate iters_done (see live_h()).
  int64_t enqueued = 0;

  int step(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    SCK(cudaSetDevice(device));
    const int chunk = 16;
    for (int64_t i = 0; i < n / chunk; ++i) {
      if (int rc = capture(chunk)) return rc;
      SCK(cudaGraphLaunch(gexec, stream));
      enqueued += chunk;
    }
    for (int64_t i = 0; i < n % chunk; ++i) {
      int l0 = launches;
      if (int rc = enqueue_iteration(0)) return rc;
      launches_per_iter = launches - l0;
      advance_base<<<1, 1, 0, stream>>>(st, 1);
      SCK(cudaGetLastError());
      enqueued += 1;
      if (gexec) {   // the captured graph baked in the pointer parity
        SCK(cudaGraphExecDestroy(gexec));
        gexec = nullptr;
      }
    }
    return 0;
  }

  int sync(int64_t* done, int* conv) override {
    SCK(cudaSetDevice(device));
    SCK(cudaMemcpyAsync(st_host, st, sizeof(RunState), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    if (done) *done = st_host->iters_done;
    if (conv) *conv = st_host->converged;
    return 0;
  }

  int read_trace(double* obj, double* sec, double* kkt, int64_t n) override {
    if (n > tr_cap) return fail(BNMF_E_ARG, "trace request exceeds max_iters");
    if (obj) SCK(cudaMemcpyAsync(obj, tr_obj, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (sec) SCK(cudaMemcpyAsync(sec, tr_sec, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (kkt) SCK(cudaMemcpyAsync(kkt, tr_kkt, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    return 0;
  }

  int get_factors(double* w, double* h) override {
    SCK(cudaSetDevice(device));
    int64_t done = 0;
    if (int rc = sync(&done, nullptr)) return rc;
    // iterate `done` lives in Ht if the (done .. enqueued) inactive tail had an
    // even number of swaps, else in Hn
    const float* Hlive = ((enqueued - done) % 2 == 0) ? Ht : Hn;
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    double* stg;
    SCK(cudaMalloc(&stg, std::max(fk, nk) * sizeof(double)));
    sp_pad_out<<<nsm * 8, 256, 0, stream>>>(Wt, size_t(F), K, KL, stg);
    SCK(cudaMemcpyAsync(w, stg, fk * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    sp_transpose_out<<<nsm * 8, 256, 0, stream>>>(Hlive, size_t(N), K, KL, stg);
    SCK(cudaMemcpyAsync(h, stg, nk * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    SCK(cudaFree(stg));
    return 0;
  }

  int init_comm(int r, int nr, const void* id, int64_t ng) override {
    (void)ng;
    rank = r; nranks = nr;
    if (nr > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      ncclResult_t rr = ncclCommInitRank(&comm_nccl, nr, uid, r);
      if (rr != ncclSuccess) return fail(BNMF_E_NCCL, ncclGetErrorString(rr));
    }
    return 0;
  }
  int set_profiling(int) override { return 0; }
  int pass_time(float* ms, int* n) override { *ms = 0.f; *n = 0; return 0; }
};

EngineBase* make_sparse_engine(int device, cudaStream_t stream) {
  return new SparseEngine(device, stream);
}

int sparse_set_csr(EngineBase* e, const long long* ip, const int* ix, const float* v,
                   const long long* cp, const int* ri, const int* pm, int64_t F, int64_t N,
                   int64_t nnz, int on_dev) {
  return static_cast<SparseEngine*>(e)->set_csr(ip, ix, v, cp, ri, pm, F, N, nnz, on_dev);
}

}  // namespace bnmf
