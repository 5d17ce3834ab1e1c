// SIMT kernels of the reference-order schedule (any dtype, any beta, any
// sub-iteration count).  These follow the reference loop literally:
//   W-side pass  : updates.py:203-220 (jmm) / 157-170 (bmm)
//   H-side pass  : updates.py:223-235 (jmm) / 173-181 (bmm)
//   objective    : solver.py:304-309 + core.py:89-114
//   KKT          : diagnostics.py:46-59
// V is F x ldv row-major; W is F x K row-major; H is stored transposed
// ("Ht", N x K row-major, k contiguous per column n).  All reductions are
// fixed-order (no float atomics): results are bitwise reproducible.
//
// fp64 (T = double) forms every product on the FP64 tensor path: the 32 x 32 model tile
// W H^T and the skinny side products are chains of mma.sync.m8n8k4.f64 (SASS: DMMA) on
// 8 x 8 sub-tiles, accumulators in the D fragments; fp32 keeps the scalar FMA form.
#pragma once

#include <cooperative_groups.h>
#include <type_traits>

#include "bnmf_common.cuh"

namespace bnmf {

// D (8 x 8) += A (8 x 4, row) * B (4 x 8, col) in fp64.  Fragments of lane L (g = L / 4,
// t = L % 4): a = A[g][t], b = B[t][g], d[0..1] = D[g][2 t + {0, 1}].
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int ST_TF = 32;       // rows of F per tile
constexpr int ST_NC = 32;       // columns of N per tile
constexpr int ST_THREADS = 256;
constexpr int ST_KCH = 64;      // k handled per accumulation sweep (8 per thread)
constexpr int ST_KMAX = 128;    // largest rank of the SIMT path

enum PassMode : int { PM_UPDATE = 0, PM_KKT = 1 };

__host__ __device__ inline int kstride(int K) { return (K & 1) ? K : K + 1; }

// Cooperative copy of `rows` rows of K values (global row stride K) into a
// shared buffer with row stride ks; rows past `valid` are zero-filled.
template <typename T>
__device__ __forceinline__ void load_rows(T* dst, const T* __restrict__ src, int rows,
                                          int valid, int K, int ks) {
  // (r, k) of element i advance with i by (blockDim / K, blockDim % K): two divisions per call
  // instead of one per element
  const int dr = blockDim.x / K, dk = blockDim.x - dr * K;
  int r = threadIdx.x / K, k = threadIdx.x - r * K;
  for (int i = threadIdx.x; i < rows * K; i += blockDim.x) {
    dst[r * ks + k] = r < valid ? src[i] : T(0);
    r += dr;
    k += dk;
    if (k >= K) { k -= K; ++r; }
  }
}

// The same copy with cp.async (8-byte elements): the caller commits the group and waits for it
// one tile later, so the L2 round trip of a tile's rows runs under the previous tile's work.
__device__ __forceinline__ void load_rows_async(double* dst, const double* __restrict__ src,
                                                int rows, int valid, int K, int ks) {
  const int dr = blockDim.x / K, dk = blockDim.x - dr * K;
  int r = threadIdx.x / K, k = threadIdx.x - r * K;
  const unsigned d0 = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  for (int i = threadIdx.x; i < rows * K; i += blockDim.x) {
    if (r < valid)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d0 + 8u * (r * ks + k)),
                   "l"(src + i)
                   : "memory");
    else
      dst[r * ks + k] = 0.0;
    r += dr;
    k += dk;
    if (k >= K) { k -= K; ++r; }
  }
}

// Z tile for rows [f0, f0+TF) x cols [n0, n0+NC): y = W[f,:] . H[:,n] + kappa,
// then (zn, zd) by the beta rule (or the KKT gradient core in zn).  Entries
// outside the matrix are 0 so they never contribute.
template <int BC, int MODE, typename T>
__device__ __forceinline__ void z_tile(const T* __restrict__ V, size_t ldv, int F, int N,
                                       int f0, int n0, const T* Ws, const T* Hs, int K,
                                       int ks, T kappa, T beta, T* Zn, T* Zd) {
  if constexpr (std::is_same<T, double>::value) {
    // warp w: f sub-tile r = w & 3, n sub-tiles 2 (w >> 2) + {0, 1}; lane (g, t) ends up with
    // y at rows 8 r + g, columns 8 c + 2 t + {0, 1}
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = w & 3, cp = w >> 2, g = lane >> 2, t = lane & 3;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    // the V values of the thread's four elements are requested before the product chain, so
    // that their latency runs under it
    T xv[2][2];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int f = 8 * r + g, n = 8 * (2 * cp + c) + 2 * t + e;
        xv[c][e] = (f0 + f < F && n0 + n < N) ? V[(size_t)(f0 + f) * ldv + (n0 + n)] : T(0);
      }
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int k = k0 + t;
      const double a = k < K ? Ws[(8 * r + g) * ks + k] : 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double b = k < K ? Hs[(8 * (2 * cp + c) + g) * ks + k] : 0.0;
        dmma884(acc[c], a, b);
      }
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int f = 8 * r + g, n = 8 * (2 * cp + c) + 2 * t + e;
        T zn = T(0), zd = T(0);
        if (f0 + f < F && n0 + n < N) {
          const T y = acc[c][e] + kappa;
          const T x = xv[c][e];
          if (MODE == PM_KKT) {
            zn = grad_core<BC, T>(x, y, beta);
          } else {
            bases<BC, T>(x, y, beta, zn, zd);
          }
        }
        Zn[f * (ST_NC + 1) + n] = zn;
        Zd[f * (ST_NC + 1) + n] = zd;
      }
    return;
  }
  for (int e = threadIdx.x; e < ST_TF * ST_NC; e += blockDim.x) {
    int f = e / ST_NC, n = e - f * ST_NC;
    T zn = T(0), zd = T(0);
    if (f0 + f < F && n0 + n < N) {
      const T* wr = Ws + f * ks;
      const T* hr = Hs + n * ks;
      T y = T(0);
      for (int k = 0; k < K; ++k) y = fma(wr[k], hr[k], y);
      y += kappa;
      T x = V[(size_t)(f0 + f) * ldv + (n0 + n)];
      if (MODE == PM_KKT) {
        zn = grad_core<BC, T>(x, y, beta);
      } else {
        bases<BC, T>(x, y, beta, zn, zd);
      }
    }
    Zn[f * (ST_NC + 1) + n] = zn;
    Zd[f * (ST_NC + 1) + n] = zd;
  }
}

// ---------------------------------------------------------------------------
// W-side partial sums over a column segment:
//   num[f,k] = sum_n Zn[f,n] C1[n,k],  den[f,k] = sum_n Zd[f,n] C2[n,k]
// part layout: [seg][2][F][K] (double).  Grid (ceil(F/TF), S).
template <int BC, int MODE, typename T>
__global__ void __launch_bounds__(ST_THREADS)
wside_partials(const T* __restrict__ V, size_t ldv, int F, int N, int K,
               const T* __restrict__ Wp, const T* __restrict__ Hp,
               const T* __restrict__ C1, const T* __restrict__ C2,
               int seg_cols, Scalars sc, double* __restrict__ part, int nbuf,
               const RunState* st, int slot, T* __restrict__ zgn, T* __restrict__ zgd,
               size_t ldz) {
  if (!iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ks = kstride(K);
  // nbuf (1 or 2) copies of the column stage [Hs | C1s | C2s]; two when they fit (fp64 path)
  T* Ws = reinterpret_cast<T*>(smem_raw);
  T* Hs = Ws + ST_TF * ks;
  T* C1s = Hs + ST_NC * ks;
  T* C2s = C1s + ST_NC * ks;
  T* Zn = Hs + nbuf * 3 * ST_NC * ks;
  T* Zd = Zn + ST_TF * (ST_NC + 1);

  const int f0 = blockIdx.x * ST_TF;
  const int seg = blockIdx.y;
  const int nbeg = seg * seg_cols;
  const int nend = min(N, nbeg + seg_cols);
  const T kappa = T(sc.kappa), beta = T(sc.beta);

  load_rows(Ws, Wp + (size_t)f0 * K, ST_TF, F - f0, K, ks);

  if constexpr (std::is_same<T, double>::value) {
    // DMMA accumulation: warp w owns rows 8 r + [0, 8) (r = w & 3) and the k sub-tiles
    // kc = (w >> 2) + 2 j; the sums over the whole segment stay in the D fragments
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = w & 3, kp = w >> 2, g = lane >> 2, t = lane & 3;
    constexpr int NJ = ST_KMAX / 16;
    double dn[NJ][2], dd[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) { dn[j][0] = dn[j][1] = 0.0; dd[j][0] = dd[j][1] = 0.0; }
    // beta = 1: Z_den is all ones, so den[f, k] = sum_n C2[n, k] is the same for every row of the
    // tile: thread k adds the staged C2 rows in column order instead of a second DMMA chain per
    // row (a third of the pass's DMMA work)
    constexpr bool ONES = (BC == BC_1) && (MODE == PM_UPDATE);
    __shared__ double s_seg[ST_KMAX];
    double segs = 0.0;
    const int bstride = 3 * ST_NC * ks;   // doubles between the two column stages
    auto stage = [&](int n0, int b) {
      const int valid = min(ST_NC, nend - n0);
      load_rows_async(Hs + b * bstride, Hp + (size_t)n0 * K, ST_NC, valid, K, ks);
      load_rows_async(C1s + b * bstride, C1 + (size_t)n0 * K, ST_NC, valid, K, ks);
      if (MODE != PM_KKT) load_rows_async(C2s + b * bstride, C2 + (size_t)n0 * K, ST_NC, valid, K, ks);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (nbuf == 2 && nbeg < nend) stage(nbeg, 0);
    int it = 0;
    for (int n0 = nbeg; n0 < nend; n0 += ST_NC, ++it) {
      const int b = nbuf == 2 ? (it & 1) : 0;
      __syncthreads();   // the previous step's products have read the other stage and Zn / Zd
      if (nbuf == 2) {
        const bool more = n0 + ST_NC < nend;
        if (more) stage(n0 + ST_NC, b ^ 1);
        if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
      } else {
        stage(n0, 0);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* Hb = Hs + b * bstride;
      const double* C1b = C1s + b * bstride;
      const double* C2b = C2s + b * bstride;
      z_tile<BC, MODE, T>(V, ldv, F, nend, f0, n0, Ws, Hb, K, ks, kappa, beta, Zn, Zd);
      if (ONES && threadIdx.x < K) {
        const int vn = min(ST_NC, nend - n0);
        for (int r2 = 0; r2 < vn; ++r2) segs += C2b[r2 * ks + threadIdx.x];
      }
      __syncthreads();
      // JMM: the H-side pass of this outer iteration uses the same anchor, hence the same Z
      // (updates.py:184-200); it reads the tiles back instead of forming W~H~ and Z again
      if (zgn) {
        for (int e = threadIdx.x; e < ST_TF * ST_NC; e += ST_THREADS) {
          const int f = e / ST_NC, n = e - f * ST_NC;
          if (f0 + f < F && n0 + n < nend) {
            zgn[(size_t)(f0 + f) * ldz + n0 + n] = Zn[f * (ST_NC + 1) + n];
            if (zgd) zgd[(size_t)(f0 + f) * ldz + n0 + n] = Zd[f * (ST_NC + 1) + n];
          }
        }
      }
#pragma unroll 2
      for (int n4 = 0; n4 < ST_NC / 4; ++n4) {
        const double an = Zn[(8 * r + g) * (ST_NC + 1) + 4 * n4 + t];
        const double ad = Zd[(8 * r + g) * (ST_NC + 1) + 4 * n4 + t];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int kk = 8 * (kp + 2 * j) + g;
          if (8 * (kp + 2 * j) < K) {
            const double b1 = kk < K ? C1b[(4 * n4 + t) * ks + kk] : 0.0;
            dmma884(dn[j], an, b1);
            if (MODE != PM_KKT && !ONES) {
              const double b2 = kk < K ? C2b[(4 * n4 + t) * ks + kk] : 0.0;
              dmma884(dd[j], ad, b2);
            }
          }
        }
      }
    }
    if (ONES) {
      if (threadIdx.x < K) s_seg[threadIdx.x] = segs;
      __syncthreads();
    }
    const int f = f0 + 8 * r + g;
    if (f < F) {
      double* pn = part + ((size_t)seg * 2 + 0) * F * K + (size_t)f * K;
      double* pd = part + ((size_t)seg * 2 + 1) * F * K + (size_t)f * K;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 8 * (kp + 2 * j) + 2 * t + e;
          if (k < K) { pn[k] = dn[j][e]; pd[k] = ONES ? s_seg[k] : dd[j][e]; }
        }
    }
    return;
  }

  const int fl = threadIdx.x & 31;   // row within the tile
  const int kg = threadIdx.x >> 5;   // k group (warp-uniform)
  const int nkc = (K + ST_KCH - 1) / ST_KCH;
  double accn[ST_KMAX / 8], accd[ST_KMAX / 8];
#pragma unroll
  for (int j = 0; j < ST_KMAX / 8; ++j) { accn[j] = 0.0; accd[j] = 0.0; }

  for (int n0 = nbeg; n0 < nend; n0 += ST_NC) {
    __syncthreads();
    int valid = min(ST_NC, nend - n0);
    load_rows(Hs, Hp + (size_t)n0 * K, ST_NC, valid, K, ks);
    load_rows(C1s, C1 + (size_t)n0 * K, ST_NC, valid, K, ks);
    if (MODE != PM_KKT) load_rows(C2s, C2 + (size_t)n0 * K, ST_NC, valid, K, ks);
    __syncthreads();
    z_tile<BC, MODE, T>(V, ldv, F, nend, f0, n0, Ws, Hs, K, ks, kappa, beta, Zn, Zd);
    __syncthreads();
    const T* zr = Zn + fl * (ST_NC + 1);
    const T* zdr = Zd + fl * (ST_NC + 1);
#pragma unroll
    for (int j = 0; j < ST_KMAX / 8; ++j) {
      int k = kg + 8 * j;
      if (j < nkc * 8 && k < K) {
        T sn = T(0), sd = T(0);
        for (int n = 0; n < ST_NC; ++n) {
          sn = fma(zr[n], C1s[n * ks + k], sn);
          if (MODE != PM_KKT) sd = fma(zdr[n], C2s[n * ks + k], sd);
        }
        accn[j] += double(sn);
        accd[j] += double(sd);
      }
    }
  }
  if (f0 + fl < F) {
    double* pn = part + ((size_t)seg * 2 + 0) * F * K + (size_t)(f0 + fl) * K;
    double* pd = part + ((size_t)seg * 2 + 1) * F * K + (size_t)(f0 + fl) * K;
#pragma unroll
    for (int j = 0; j < ST_KMAX / 8; ++j) {
      int k = kg + 8 * j;
      if (k < K) { pn[k] = accn[j]; pd[k] = accd[j]; }
    }
  }
}

// ---------------------------------------------------------------------------
// H-side pass over a block of NC columns and all F rows.
//   PM_UPDATE: Hout[n,k] = Hbase[n,k] * (num/max(den,floor))^gamma with
//              num[k,n] = sum_f C1w[f,k] Zn[f,n], den likewise with C2w/Zd;
//              den_ones (beta=1): den[k,n] = colsum(C2w)[k] (updates.py:133-137)
//   PM_KKT   : grad[k,n] = sum_f Wp[f,k] g[f,n]; writes the per-block sum of
//              |min(Hp[n,k], grad[k,n])| to part[block] (diagnostics.py:56-58)
template <int BC, int MODE, typename T>
__global__ void __launch_bounds__(ST_THREADS)
hside_pass(const T* __restrict__ V, size_t ldv, int F, int N, int K,
           const T* __restrict__ Wp, const T* __restrict__ Hp,
           const T* __restrict__ C1w, const T* __restrict__ C2w,
           const T* __restrict__ Hbase, T* __restrict__ Hout,
           const double* __restrict__ colsum_c2, int den_ones, Scalars sc,
           double* __restrict__ part, int nbuf, const RunState* st, int slot,
           const T* __restrict__ zgn, const T* __restrict__ zgd, size_t ldz) {
  if (!iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ks = kstride(K);
  // nbuf (1 or 2) copies of the row stage [Ws | C1s | C2s]; two when they fit (fp64 path)
  T* Hs = reinterpret_cast<T*>(smem_raw);
  T* Ws = Hs + ST_NC * ks;
  T* C1s = Ws + ST_TF * ks;
  T* C2s = C1s + ST_TF * ks;
  T* Zn = Ws + nbuf * 3 * ST_TF * ks;
  T* Zd = Zn + ST_TF * (ST_NC + 1);
  __shared__ double red[ST_THREADS / 32];

  // fp64 with few column blocks: the F rows of a block are split over a cluster of CS CTAs
  // (launch attribute; 1 otherwise), rank 0 adds the partial sums over DSMEM and updates
  cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
  const int CS = int(cl.num_blocks()), cr = int(cl.block_rank());
  const int hb = blockIdx.x / CS;
  const int n0 = hb * ST_NC;
  const int valid_n = min(ST_NC, N - n0);
  const T kappa = T(sc.kappa), beta = T(sc.beta);
  load_rows(Hs, Hp + (size_t)n0 * K, ST_NC, valid_n, K, ks);

  if constexpr (std::is_same<T, double>::value) {
    // DMMA accumulation: D rows = k (sub-tiles kc = (w >> 2) + 2 j), D columns = n
    // (sub-tile c = w & 3); lane (g, t) ends up with (k = 8 kc + g, n = 8 c + 2 t + {0, 1})
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = w & 3, kp = w >> 2, g = lane >> 2, t = lane & 3;
    constexpr int NJ = ST_KMAX / 16;
    double dn[NJ][2], dd[NJ][2];
#pragma unroll
    for (int j = 0; j < NJ; ++j) { dn[j][0] = dn[j][1] = 0.0; dd[j][0] = dd[j][1] = 0.0; }
    const bool use_den = (MODE != PM_KKT) && !den_ones;
    // beta = 1 denominators: colsum(C2w), accumulated here from the staged C2 rows (thread k
    // adds rows 0, 1, ... in order, numpy's order, like the separate col_sums launch it replaces)
    const bool fold_cs = (MODE != PM_KKT) && den_ones;
    __shared__ double s_cs[ST_KMAX];
    double cs = 0.0;
    const int bstride = 3 * ST_TF * ks;   // doubles between the two row stages
    // rows of tile f0 into stage b, one cp.async group
    // Z of the W-side pass of the same outer iteration (JMM, same anchor) read back from global
    // memory instead of the model tile + Z rule; the W~ rows are then not needed
    const bool zread = (MODE != PM_KKT) && zgn != nullptr;
    // numerator-only case (beta = 1) with room in the unused W~ slot of the stage: the Z tile is
    // prefetched with the stage's cp.async group, one tile ahead like the factor rows
    const bool zpre = zread && !use_den && ks >= ST_NC + 1;
    auto stage = [&](int f0, int b) {
      const int valid_f = min(ST_TF, F - f0);
      if (!zread) load_rows_async(Ws + b * bstride, Wp + (size_t)f0 * K, ST_TF, valid_f, K, ks);
      if (zpre) {
        double* zt = Ws + b * bstride;
        const unsigned z0 = static_cast<unsigned>(__cvta_generic_to_shared(zt));
        for (int e = threadIdx.x; e < ST_TF * ST_NC; e += ST_THREADS) {
          const int f = e / ST_NC, n = e - f * ST_NC;
          if (f0 + f < F && n0 + n < N)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                             z0 + 8u * (f * (ST_NC + 1) + n)),
                         "l"(zgn + (size_t)(f0 + f) * ldz + n0 + n)
                         : "memory");
          else
            zt[f * (ST_NC + 1) + n] = 0.0;
        }
      }
      if (MODE != PM_KKT) {
        load_rows_async(C1s + b * bstride, C1w + (size_t)f0 * K, ST_TF, valid_f, K, ks);
        if (use_den || fold_cs)
          load_rows_async(C2s + b * bstride, C2w + (size_t)f0 * K, ST_TF, valid_f, K, ks);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ntile = (F + ST_TF - 1) / ST_TF, per = (ntile + CS - 1) / CS;
    const int fbeg = min(F, cr * per * ST_TF), fend = min(F, (cr + 1) * per * ST_TF);
    if (nbuf == 2 && fbeg < fend) stage(fbeg, 0);
    int it = 0;
    for (int f0 = fbeg; f0 < fend; f0 += ST_TF, ++it) {
      const int b = nbuf == 2 ? (it & 1) : 0;
      __syncthreads();   // the previous tile's products have read the other stage and Zn / Zd
      if (nbuf == 2) {
        const bool more = f0 + ST_TF < fend;
        if (more) stage(f0 + ST_TF, b ^ 1);
        if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
      } else {
        stage(f0, 0);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* Wb = Ws + b * bstride;
      const double* C1b = C1s + b * bstride;
      const double* C2b = C2s + b * bstride;
      if (zpre) {
        // the tile arrived with the stage
      } else if (zread) {
        for (int e = threadIdx.x; e < ST_TF * ST_NC; e += ST_THREADS) {
          const int f = e / ST_NC, n = e - f * ST_NC;
          const bool ok = f0 + f < F && n0 + n < N;
          Zn[f * (ST_NC + 1) + n] = ok ? zgn[(size_t)(f0 + f) * ldz + n0 + n] : 0.0;
          if (use_den) Zd[f * (ST_NC + 1) + n] = ok ? zgd[(size_t)(f0 + f) * ldz + n0 + n] : 0.0;
        }
      } else {
        z_tile<BC, MODE, T>(V, ldv, F, N, f0, n0, Wb, Hs, K, ks, kappa, beta, Zn, Zd);
      }
      if (fold_cs && threadIdx.x < K) {
        const int vf = min(ST_TF, F - f0);
        for (int r = 0; r < vf; ++r) cs += C2b[r * ks + threadIdx.x];
      }
      __syncthreads();
      const T* A1 = (MODE == PM_KKT) ? Wb : C1b;
      const double* Znp = zpre ? Wb : Zn;
#pragma unroll 2
      for (int f4 = 0; f4 < ST_TF / 4; ++f4) {
        const double bn = Znp[(4 * f4 + t) * (ST_NC + 1) + 8 * c + g];
        const double bd = Zd[(4 * f4 + t) * (ST_NC + 1) + 8 * c + g];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int kk = 8 * (kp + 2 * j) + g;
          if (8 * (kp + 2 * j) < K) {
            const double a1 = kk < K ? A1[(4 * f4 + t) * ks + kk] : 0.0;
            dmma884(dn[j], a1, bn);
            if (use_den) {
              const double a2 = kk < K ? C2b[(4 * f4 + t) * ks + kk] : 0.0;
              dmma884(dd[j], a2, bd);
            }
          }
        }
      }
    }
    if (CS > 1) {
      // partial sums of this CTA's rows -> shared memory (the row stages are free now), one
      // column per thread; rank 0 adds the peers' in rank order
      __syncthreads();
      double* P = reinterpret_cast<double*>(Ws);
      const int NJA = (K + 15) / 16;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (j < NJA) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            P[((0 * NJA + j) * 2 + e) * ST_THREADS + threadIdx.x] = dn[j][e];
            P[((1 * NJA + j) * 2 + e) * ST_THREADS + threadIdx.x] = dd[j][e];
          }
        }
      if (fold_cs && threadIdx.x < K) s_cs[threadIdx.x] = cs;
      cl.sync();
      if (cr == 0) {
        for (int r = 1; r < CS; ++r) {
          const double* Pr = cl.map_shared_rank(P, r);
#pragma unroll
          for (int j = 0; j < NJ; ++j)
            if (j < NJA) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                dn[j][e] += Pr[((0 * NJA + j) * 2 + e) * ST_THREADS + threadIdx.x];
                dd[j][e] += Pr[((1 * NJA + j) * 2 + e) * ST_THREADS + threadIdx.x];
              }
            }
          if (fold_cs && threadIdx.x < K) cs += cl.map_shared_rank(s_cs, r)[threadIdx.x];
        }
      }
      cl.sync();   // the peers' shared memory stays valid until rank 0 has read it
      if (cr != 0) return;
    }
    if (MODE == PM_KKT) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = 8 * (kp + 2 * j) + g, n = 8 * c + 2 * t + e;
          if (k < K && n < valid_n) s += fabs(fmin(double(Hs[n * ks + k]), dn[j][e]));
        }
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (lane == 0) red[w] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tt = 0.0;
        for (int ww = 0; ww < ST_THREADS / 32; ++ww) tt += red[ww];
        part[hb] = tt;
      }
      return;
    }
    if (fold_cs) {
      if (threadIdx.x < K) s_cs[threadIdx.x] = cs;
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 8 * (kp + 2 * j) + g, n = 8 * c + 2 * t + e;
        if (k < K && n < valid_n) {
          const double den = den_ones ? s_cs[k] : dd[j][e];
          const double rr = dn[j][e] / fmax(den, sc.floor);
          const double b = double(Hbase[(size_t)(n0 + n) * K + k]);
          Hout[(size_t)(n0 + n) * K + k] = T(b * apply_exponent<double>(rr, sc.gamma));
        }
      }
    return;
  }

  const int nl = threadIdx.x & 31;
  const int kg = threadIdx.x >> 5;
  double accn[ST_KMAX / 8], accd[ST_KMAX / 8];
#pragma unroll
  for (int j = 0; j < ST_KMAX / 8; ++j) { accn[j] = 0.0; accd[j] = 0.0; }
  const bool use_den = (MODE != PM_KKT) && !den_ones;

  for (int f0 = 0; f0 < F; f0 += ST_TF) {
    __syncthreads();
    int valid_f = min(ST_TF, F - f0);
    load_rows(Ws, Wp + (size_t)f0 * K, ST_TF, valid_f, K, ks);
    if (MODE != PM_KKT) {
      load_rows(C1s, C1w + (size_t)f0 * K, ST_TF, valid_f, K, ks);
      if (use_den) load_rows(C2s, C2w + (size_t)f0 * K, ST_TF, valid_f, K, ks);
    }
    __syncthreads();
    z_tile<BC, MODE, T>(V, ldv, F, N, f0, n0, Ws, Hs, K, ks, kappa, beta, Zn, Zd);
    __syncthreads();
    const T* A1 = (MODE == PM_KKT) ? Ws : C1s;
#pragma unroll
    for (int j = 0; j < ST_KMAX / 8; ++j) {
      int k = kg + 8 * j;
      if (k < K) {
        T sn = T(0), sd = T(0);
        for (int f = 0; f < ST_TF; ++f) {
          sn = fma(A1[f * ks + k], Zn[f * (ST_NC + 1) + nl], sn);
          if (use_den) sd = fma(C2s[f * ks + k], Zd[f * (ST_NC + 1) + nl], sd);
        }
        accn[j] += double(sn);
        accd[j] += double(sd);
      }
    }
  }

  if (MODE == PM_KKT) {
    double s = 0.0;
    if (nl < valid_n) {
#pragma unroll
      for (int j = 0; j < ST_KMAX / 8; ++j) {
        int k = kg + 8 * j;
        if (k < K) s += fabs(fmin(double(Hs[nl * ks + k]), accn[j]));
      }
    }
    // fixed-order block reduction
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < ST_THREADS / 32; ++w) t += red[w];
      part[hb] = t;
    }
    return;
  }
  if (nl < valid_n) {
    const double fl = sc.floor;
    const double g = sc.gamma;
#pragma unroll
    for (int j = 0; j < ST_KMAX / 8; ++j) {
      int k = kg + 8 * j;
      if (k < K) {
        double den = den_ones ? colsum_c2[k] : accd[j];
        double r = accn[j] / fmax(den, fl);
        double b = double(Hbase[(size_t)(n0 + nl) * K + k]);
        Hout[(size_t)(n0 + nl) * K + k] = T(b * apply_exponent<double>(r, g));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Objective partials: sum over tiles of d_beta(V | W H + kappa) in double.
// Grid (ceil(F/TF), S); part[blockIdx.y * gridDim.x + blockIdx.x].
template <int BC, typename T>
__global__ void __launch_bounds__(ST_THREADS)
objective_partials(const T* __restrict__ V, size_t ldv, int F, int N, int K,
                   const T* __restrict__ W, const T* __restrict__ Ht, int seg_cols,
                   Scalars sc, double* __restrict__ part, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int ks = kstride(K);
  T* Ws = reinterpret_cast<T*>(smem_raw);
  T* Hs = Ws + ST_TF * ks;
  __shared__ double red[ST_THREADS / 32];
  const int f0 = blockIdx.x * ST_TF;
  const int nbeg = blockIdx.y * seg_cols;
  const int nend = min(N, nbeg + seg_cols);
  const T kappa = T(sc.kappa);
  load_rows(Ws, W + (size_t)f0 * K, ST_TF, F - f0, K, ks);
  double s = 0.0;
  if constexpr (std::is_same<T, double>::value) {
    // fp64: the H~ rows of the next 32 columns arrive (cp.async, second stage) while this step
    // forms its model tile; the V values are requested before the product chain
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = w & 3, cp = w >> 2, g = lane >> 2, t = lane & 3;
    const int bstride = ST_NC * ks;
    auto stage = [&](int n0, int b) {
      load_rows_async(Hs + b * bstride, Ht + (size_t)n0 * K, ST_NC, min(ST_NC, nend - n0), K, ks);
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (nbeg < nend) stage(nbeg, 0);
    int it = 0;
    for (int n0 = nbeg; n0 < nend; n0 += ST_NC, ++it) {
      const int b = it & 1;
      __syncthreads();   // the previous step has read the other stage
      const bool more = n0 + ST_NC < nend;
      if (more) stage(n0 + ST_NC, b ^ 1);
      if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      double xv[2][2];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int f = 8 * r + g, n = 8 * (2 * cp + c) + 2 * t + e;
          xv[c][e] = (f0 + f < F && n0 + n < nend) ? double(V[(size_t)(f0 + f) * ldv + n0 + n]) : 0.0;
        }
      __syncthreads();
      const double* Hb = Hs + b * bstride;
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int k = k0 + t;
        const double a = k < K ? Ws[(8 * r + g) * ks + k] : 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double bb = k < K ? Hb[(8 * (2 * cp + c) + g) * ks + k] : 0.0;
          dmma884(acc[c], a, bb);
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int f = 8 * r + g, n = 8 * (2 * cp + c) + 2 * t + e;
          if (f0 + f < F && n0 + n < nend)
            s += divergence<BC>(xv[c][e], acc[c][e] + double(kappa), sc.beta);
        }
    }
  }
  for (int n0 = nbeg; n0 < nend && !std::is_same<T, double>::value; n0 += ST_NC) {
    __syncthreads();
    load_rows(Hs, Ht + (size_t)n0 * K, ST_NC, min(ST_NC, nend - n0), K, ks);
    __syncthreads();
    for (int e = threadIdx.x; e < ST_TF * ST_NC; e += blockDim.x) {
      int f = e / ST_NC, n = e - f * ST_NC;
      if (f0 + f < F && n0 + n < nend) {
        T y = T(0);
        for (int k = 0; k < K; ++k) y = fma(Ws[f * ks + k], Hs[n * ks + k], y);
        y += kappa;
        double x = double(V[(size_t)(f0 + f) * ldv + n0 + n]);
        s += divergence<BC>(x, double(y), sc.beta);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < ST_THREADS / 32; ++w) t += red[w];
    part[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

}  // namespace bnmf
