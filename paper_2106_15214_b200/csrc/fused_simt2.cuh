// Register-tiled SIMT form of the fused pass (fp32, any F, K <= 64), used for
// the shapes outside the tcgen05 kernel's limits (configs 2 and 3: F > 256,
// K > 16).  Same contract as fused_pass_tc / fused_common.cuh, split in two
// kernels so that each keeps its accumulators in registers:
//
//   fs2::hpass  one CTA per 32-column block, all F rows in 64-row chunks:
//               Vt_{p-1} = Wa H~_{p-1} + kappa, Z by the beta rule, and the
//               H-side sums chi1^T Zn / chi2^T Zd -> H_p, H~_p = H_p norms_p
//               (updates.py:223-235 / 173-181, solver.py:167-171);
//   fs2::wpass  grid (64-row chunk, column segment): Vt_p = W~_p H~_p + kappa,
//               the objective of iterate p (solver.py:304-309) and the W-side
//               sums Zn H~_p^T, Zd H~_p^T of iteration p+1 (updates.py:203-220),
//               held in fp64 registers over the whole segment and written
//               once to the segment's slab part[seg][2][F][K].
//
// V is read twice per iteration; at configs 2 and 3 it is L2-resident
// (34 / 67 MB < 126 MB), so the second read is served by L2.  Every thread
// owns a 4-row x 2-column tile of Vt (columns tn and tn+16, so the 16-byte
// loads of the H rows are bank-conflict free with a row stride = 4 mod 8).
// Per chunk/step the sums are fp32 and are folded into fp64 registers; all
// orders are fixed, so results are bitwise reproducible.
#pragma once

#include "fused_common.cuh"
#include "simt_kernels.cuh"

namespace bnmf {
namespace fs2 {

constexpr int THREADS = 256;
constexpr int TF = 64;        // rows per chunk
constexpr int NC = 32;        // columns per block / step
constexpr int TFP = TF + 4;   // row stride of the transposed Z tile
constexpr int VS = NC + 4;    // row stride of the staged V tile (conflict-free reads)

__host__ __device__ inline int kr4(int K) { return (K + 3) & ~3; }
// row stride of the row-major factor tiles: >= K rounded to 4, = 4 (mod 8)
__host__ __device__ inline int krs(int K) { int r = kr4(K); return (r & 7) == 4 ? r : r + 4; }
__host__ __device__ inline int kj_of(int K) { return K <= 32 ? 1 : 2; }

__host__ inline size_t h_smem(int K) {
  const int rs = krs(K), ks = 32 * kj_of(K);
  // Hp [NC][rs] (+32 slack); two stage buffers {Ws [TF][rs], C1s/C2s [TF][ks],
  // Vs [TF][VS]}; Zn/Zd [TF][NC], which the group sums Red [4][2][ks][NC] alias
  const size_t buf = size_t(TF) * rs + 2 * size_t(TF) * ks + size_t(TF) * VS;
  const size_t z = 2 * size_t(TF) * NC, red = size_t(8) * ks * NC;
  return sizeof(float) * (size_t(NC) * rs + 32 + 2 * buf + (z > red ? z : red));
}
__host__ inline size_t w_smem(int K) {
  const int rs = krs(K);
  // Ws [TF][rs]; two stage buffers {Hs [NC][rs] (+64 slack), Vs [TF][VS]};
  // ZnT/ZdT [NC][TFP]
  return sizeof(float) * (size_t(TF) * rs + 2 * (size_t(NC) * rs + 64 + size_t(TF) * VS) +
                          2 * size_t(NC) * TFP);
}

// ---- elementwise forms of the SIMT pair ------------------------------------
// One reciprocal per element (rcp.approx + one Newton step, within an ulp of
// 1/y) shared by the bases and the objective; the series of the
// cancellation-free objective forms (fused_common.cuh) in Horner form.  The
// log of the far branch (|t - 1| >= 1/4, so |log t| >= 0.22) is MUFU.LG2
// based (__logf: absolute error ~2^-21 near 1, relative ~2 ulp elsewhere),
// i.e. <= ~1e-5 relative on such an element.
__device__ __forceinline__ float rcp_nr(float y) {
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(y));
  return fmaf(r, fmaf(-y, r, 1.f), r);
}
// u - log1p(u) = sum_{j=2..15} (-1)^j u^j / j
__device__ __forceinline__ float ser0(float u) {
  float p = -1.f / 15.f;
#pragma unroll
  for (int j = 14; j >= 2; --j) p = fmaf(p, u, ((j & 1) ? -1.f : 1.f) / float(j));
  return u * u * p;
}
// (1+u) log1p(u) - u = sum_{j=2..15} (-1)^j u^j / (j (j-1))
__device__ __forceinline__ float ser1(float u) {
  float p = -1.f / 210.f;
#pragma unroll
  for (int j = 14; j >= 2; --j) p = fmaf(p, u, ((j & 1) ? -1.f : 1.f) / float(j * (j - 1)));
  return u * u * p;
}
// (Zn, Zd) by the beta rule (updates.py:184-200)
template <int BC>
__device__ __forceinline__ void zbases(float x, float y, float beta, float& zn, float& zd) {
  if (BC == BC_2) { zn = x; zd = y; }
  else if (BC == BC_1) { zn = x * rcp_nr(y); zd = 1.f; }
  else if (BC == BC_0) { const float r = rcp_nr(y); zn = x * r * r; zd = r; }
  else bases32<BC>(x, y, beta, zn, zd);
}
// d_beta(x | y) (core.py:89-114, cancellation-free) plus the bases
template <int BC>
__device__ __forceinline__ float zdiv(float x, float y, float beta, float& zn, float& zd) {
  if (BC == BC_2) { zn = x; zd = y; const float d = x - y; return 0.5f * d * d; }
  if (BC == BC_1) {
    const float r = rcp_nr(y), q = x * r;
    zn = q; zd = 1.f;
    if (x == 0.f) return y;
    const float u = (x - y) * r;
    if (fabsf(u) < 0.25f) return y * ser1(u);
    return x * __logf(q) - x + y;
  }
  if (BC == BC_0) {
    const float r = rcp_nr(y);
    zn = x * r * r; zd = r;
    const float u = (x - y) * r;
    if (fabsf(u) < 0.25f) return ser0(u);
    const float t = x * r;
    return t - __logf(t) - 1.f;
  }
  bases32<BC>(x, y, beta, zn, zd);
  return divergence32<BC>(x, y, beta);
}

// y[i][j] = sum_k Ws[r_i][k] * Hs[c_j][k], rows r_i = 4 tf + i, columns
// c_0 = tn, c_1 = tn + 16; k in ascending order
__device__ __forceinline__ void vt_tile(const float* Ws, const float* Hs, int rs, int kr, int tf,
                                        int tn, float (&y)[4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) { y[i][0] = 0.f; y[i][1] = 0.f; }
  const float* h0p = Hs + tn * rs;
  const float* h1p = Hs + (tn + 16) * rs;
  const float* wp = Ws + (tf * 4) * rs;
#pragma unroll 2
  for (int k = 0; k < kr; k += 4) {
    const float4 h0 = *reinterpret_cast<const float4*>(h0p + k);
    const float4 h1 = *reinterpret_cast<const float4*>(h1p + k);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 w = *reinterpret_cast<const float4*>(wp + i * rs + k);
      y[i][0] = fmaf(w.x, h0.x, y[i][0]); y[i][1] = fmaf(w.x, h1.x, y[i][1]);
      y[i][0] = fmaf(w.y, h0.y, y[i][0]); y[i][1] = fmaf(w.y, h1.y, y[i][1]);
      y[i][0] = fmaf(w.z, h0.z, y[i][0]); y[i][1] = fmaf(w.z, h1.z, y[i][1]);
      y[i][0] = fmaf(w.w, h0.w, y[i][0]); y[i][1] = fmaf(w.w, h1.w, y[i][1]);
    }
  }
}

__device__ __forceinline__ void cp4(float* dst, const float* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void cp16(float* dst, const float* src, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes)
               : "memory");
}

// 16-byte row copies of a K-wide row-major block (K % 4 == 0, K <= 64): lane l
// copies chunk l % q (q = K / 4) of row l / q of each group of 32 / q rows,
// so the loop has no runtime division.  Rows past `valid` are zero-filled;
// columns >= K are left untouched (they only feed unused accumulators).
struct RowMap {
  int rr, c, rpw;
  bool on;
};
__device__ __forceinline__ RowMap row_map(int K) {
  const int q = K >> 2, lane = threadIdx.x & 31;
  RowMap m;
  m.rpw = 32 / q;
  m.rr = lane / q;
  m.c = (lane - m.rr * q) * 4;
  m.on = m.rr < m.rpw;
  return m;
}
__device__ __forceinline__ void rows_async16(float* dst, const float* __restrict__ src, int rows,
                                             int valid, int K, int rs, const RowMap& m) {
  if (!m.on) return;
  for (int r = (threadIdx.x >> 5) * m.rpw + m.rr; r < rows; r += (THREADS / 32) * m.rpw)
    cp16(dst + r * rs + m.c, r < valid ? src + (size_t)r * K + m.c : src, r < valid ? 16 : 0);
}

// async form of load_tile (zero fill through the cp.async source size)
__device__ __forceinline__ void tile_async(float* dst, const float* __restrict__ src, int rows,
                                           int valid, int K, int rs, int width) {
  for (int i = threadIdx.x; i < rows * width; i += THREADS) {
    const int r = i / width, k = i - r * width;
    const bool ok = r < valid && k < K;
    cp4(dst + r * rs + k, ok ? src + (size_t)r * K + k : src, ok);
  }
}

// V tile [TF rows x NC columns] at v (row stride ldv) -> dst (row stride VS),
// 16-byte copies (ldv and the column offset are multiples of 4), partial /
// zero fill past vf rows and vn columns
__device__ __forceinline__ void vtile_async(float* dst, const float* __restrict__ v, long long ldv,
                                            int vf, int vn) {
  for (int i = threadIdx.x; i < TF * (NC / 4); i += THREADS) {
    const int r = i / (NC / 4), c = (i - r * (NC / 4)) * 4;
    const int cols = r < vf ? max(0, min(4, vn - c)) : 0;
    cp16(dst + r * VS + c, cols > 0 ? v + (size_t)r * ldv + c : v, cols * 4);
  }
}

// rows [0, rows) of a row-major K-wide global block -> smem row stride rs,
// zero-filled to width `width` and past `valid` rows
__device__ __forceinline__ void load_tile(float* dst, const float* __restrict__ src, int rows,
                                          int valid, int K, int rs, int width) {
  for (int i = threadIdx.x; i < rows * width; i += THREADS) {
    const int r = i / width, k = i - r * width;
    dst[r * rs + k] = (r < valid && k < K) ? src[(size_t)r * K + k] : 0.f;
  }
}

template <int BC, int KJ>
__global__ void __launch_bounds__(THREADS)
hpass(FusedArgs a, const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  // the H pass opens a timed iteration: the start of its timer (begin_iter folded in)
  if (a.tmark && blockIdx.x == 0 && threadIdx.x == 0) *a.tmark = globaltimer();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int KS = 32 * KJ;
  constexpr bool DEN = BC != BC_1;   // beta = 1: den = colsum(C2) (updates.py:133-137)
  const int K = a.K, F = a.F, N = a.N, rs = krs(K), kr = kr4(K);
  float* Hp = reinterpret_cast<float*>(smem_raw);   // [NC][rs]
  float* B0 = Hp + NC * rs + 32;                    // 2 x {Ws, C1s, C2s, Vs}
  const int bsz = TF * rs + 2 * TF * KS + TF * VS;
  float* Zn = B0 + 2 * bsz;                         // [TF][NC]
  float* Zd = Zn + TF * NC;
  const int par = iter_parity(st, slot, p_override);
  // KKT pass (a.kkt): the same sums on the finished iterate (W~_p, H~_p) with W~_p as both
  // chi maps give W~^T Zn and W~^T Zd; the block reports sum |min(H~_p, den - num)|
  // (diagnostics.py:55-58) instead of updating H
  const int kkt = a.kkt;
  const float* Hprev = kkt ? a.Hbuf[par] : a.Hbuf[par ^ 1];
  float* Hnew = a.Hout[par];
  const float* Wa = kkt ? a.Wt2[par] : (a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn);
  const float* C1g = kkt ? a.Wt2[par] : a.C1;
  const float* C2g = kkt ? a.Wt2[par] : a.C2;
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  const int tid = threadIdx.x, tn = tid & 15, tf = tid >> 4;
  const int n0 = blockIdx.x * NC;
  const int valid_n = min(NC, N - n0);

  load_tile(Hp, Hprev + (size_t)n0 * K, NC, valid_n, K, rs, kr);

  // per chunk: 4 row groups of 16 rows x (4 k x 4 n tiles); the group sums
  // meet in Red (aliasing the chunk's tiles) and are folded into fp64 in a
  // fixed order.  Thread tid owns the (k, n) outputs e = tid + 256 m.
  constexpr int NOUT = KS * NC / THREADS;
  float* Red = Zn;                                  // [4][2][KS][NC] after the sums
  // K <= 32: only ceil(K/4) k-quads per group are live, so whole warps of
  // the 4 x 8 x nk4 layout sit the sums out instead of computing padding
  const int nk4 = KJ == 1 ? (K + 3) >> 2 : 8;
  const bool hact = tid < 32 * nk4;
  const int fg = tid / (8 * nk4), t = tid - fg * 8 * nk4;
  const int k4 = (t >> 3) * 4, n4 = (t & 7) * 4;
  double accn[NOUT], accd[NOUT];
#pragma unroll
  for (int m = 0; m < NOUT; ++m) { accn[m] = 0.0; accd[m] = 0.0; }

  const bool k16 = (K & 3) == 0;
  const RowMap rmap = row_map(k16 ? K : 4);
  // stage chunk f0 into buffer b: Wa rows, chi maps, V tile (one cp.async group)
  auto stage = [&](int f0, int b) {
    const int vf = min(TF, F - f0);
    float* ws = B0 + b * bsz;
    float* c1 = ws + TF * rs;
    if (k16) {
      rows_async16(ws, Wa + (size_t)f0 * K, TF, vf, K, rs, rmap);
      rows_async16(c1, C1g + (size_t)f0 * K, TF, vf, K, KS, rmap);
      if (DEN) rows_async16(c1 + TF * KS, C2g + (size_t)f0 * K, TF, vf, K, KS, rmap);
    } else {
      tile_async(ws, Wa + (size_t)f0 * K, TF, vf, K, rs, kr);
      tile_async(c1, C1g + (size_t)f0 * K, TF, vf, K, KS, KS);
      if (DEN) tile_async(c1 + TF * KS, C2g + (size_t)f0 * K, TF, vf, K, KS, KS);
    }
    vtile_async(c1 + 2 * TF * KS, a.V + (size_t)f0 * a.ldv + n0, a.ldv, vf, valid_n);
    cp_commit();
  };
  stage(0, 0);

  int buf = 0;
  for (int f0 = 0; f0 < F; f0 += TF, buf ^= 1) {
    const int vf = min(TF, F - f0);
    cp_wait_all();
    __syncthreads();                       // chunk f0 visible; buffer buf^1 free
    if (f0 + TF < F) stage(f0 + TF, buf ^ 1);
    const float* Ws = B0 + buf * bsz;
    const float* C1s = Ws + TF * rs;
    const float* C2s = C1s + TF * KS;
    const float* Vs = C2s + TF * KS;
    float x[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) x[i][j] = Vs[(tf * 4 + i) * VS + tn + 16 * j];
    float y[4][2];
    vt_tile(Ws, Hp, rs, kr, tf, tn, y);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int f = tf * 4 + i, n = tn + 16 * j;
        float zn = 0.f, zd = 0.f;
        if (f < vf && n < valid_n) zbases<BC>(x[i][j], y[i][j] + kappa, beta, zn, zd);
        Zn[f * NC + n] = zn;
        if (DEN) Zd[f * NC + n] = zd;
      }
    __syncthreads();
    // group sums: S[k][n] = sum_{f in group} C1[f][k] Zn[f][n]  (and C2 / Zd)
    float sn[KJ][4][4], sd[KJ][4][4];
#pragma unroll
    for (int j = 0; j < KJ; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) { sn[j][u][v] = 0.f; sd[j][u][v] = 0.f; }
    const int fe = hact ? min(16, vf - fg * 16) : 0;
#pragma unroll 2
    for (int ff = 0; ff < fe; ++ff) {
      const int f = fg * 16 + ff;
      const float4 z4 = *reinterpret_cast<const float4*>(Zn + f * NC + n4);
      const float z[4] = {z4.x, z4.y, z4.z, z4.w};
      float d[4] = {0.f, 0.f, 0.f, 0.f};
      if (DEN) {
        const float4 d4 = *reinterpret_cast<const float4*>(Zd + f * NC + n4);
        d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
      }
#pragma unroll
      for (int j = 0; j < KJ; ++j) {
        const float4 c4 = *reinterpret_cast<const float4*>(C1s + f * KS + k4 + 32 * j);
        const float c[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) sn[j][u][v] = fmaf(c[u], z[v], sn[j][u][v]);
        if (DEN) {
          const float4 e4 = *reinterpret_cast<const float4*>(C2s + f * KS + k4 + 32 * j);
          const float e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) sd[j][u][v] = fmaf(e[u], d[v], sd[j][u][v]);
        }
      }
    }
    __syncthreads();   // Zn/Zd dead: Red aliases them
    float* rn = Red + (size_t)fg * 2 * KS * NC;
    float* rd = rn + KS * NC;
#pragma unroll
    for (int j = 0; j < KJ && hact; ++j)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k4 + 32 * j + u;
        *reinterpret_cast<float4*>(rn + k * NC + n4) =
            make_float4(sn[j][u][0], sn[j][u][1], sn[j][u][2], sn[j][u][3]);
        if (DEN)
          *reinterpret_cast<float4*>(rd + k * NC + n4) =
              make_float4(sd[j][u][0], sd[j][u][1], sd[j][u][2], sd[j][u][3]);
      }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < NOUT; ++m) {
      const int e = tid + THREADS * m;
      float tn_ = 0.f, td_ = 0.f;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        tn_ += Red[(size_t)g * 2 * KS * NC + e];
        if (DEN) td_ += Red[(size_t)g * 2 * KS * NC + KS * NC + e];
      }
      accn[m] += double(tn_);
      if (DEN) accd[m] += double(td_);
    }
  }
  if (kkt) {
    // res_H partial of this column block (a.csum2 = colsum(W~_p) when beta = 1)
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < NOUT; ++m) {
      const int e = tid + THREADS * m, k = e / NC, n = e - k * NC;
      if (k < K && n < valid_n) {
        const double den = DEN ? accd[m] : a.csum2[k];
        t += fabs(fmin(double(Hp[n * rs + k]), den - accn[m]));
      }
    }
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    __syncthreads();
    double* redd = reinterpret_cast<double*>(Red);
    if ((tid & 31) == 0) redd[tid >> 5] = t;
    __syncthreads();
    if (tid == 0) {
      double tt = 0.0;
      for (int w = 0; w < THREADS / 32; ++w) tt += redd[w];
      a.opart[blockIdx.x] = tt;
    }
    return;
  }
  // H_p = H~_{p-1} * ratio^gamma ; H~_p = H_p * norms_p
#pragma unroll
  for (int m = 0; m < NOUT; ++m) {
    const int e = tid + THREADS * m, k = e / NC, n = e - k * NC;
    if (k < K && n < valid_n) {
      const double den = DEN ? accd[m] : a.csum2[k];
      const double r = accn[m] / fmax(den, a.sc.floor);
      const double h = double(Hp[n * rs + k]) * apply_exponent<double>(r, a.sc.gamma);
      Hnew[(size_t)(n0 + n) * K + k] = float(h * a.norms[k]);
    }
  }
}

template <int BC, int KJ>
__global__ void __launch_bounds__(THREADS)
wpass(FusedArgs a, const RunState* st, int slot, int p_override, int seg_cols) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, F = a.F, N = a.N, rs = krs(K), kr = kr4(K);
  float* Ws = reinterpret_cast<float*>(smem_raw);   // [TF][rs]
  float* B0 = Ws + TF * rs;                         // 2 x {Hs [NC][rs] (+64), Vs [TF][VS]}
  const int bsz = NC * rs + 64 + TF * VS;
  float* ZnT = B0 + 2 * bsz;                        // [NC][TFP]
  float* ZdT = ZnT + NC * TFP;
  __shared__ double red[THREADS / 32];

  const int par = iter_parity(st, slot, p_override);
  const float* Wt = a.Wt2[par];                             // W~_p
  const float* Hc = a.do_h ? a.Hout[par] : a.Hbuf[par];     // H~_p
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  const int tid = threadIdx.x, tn = tid & 15, tf = tid >> 4;
  // W-sum tile: 4 rows x k pair; K <= 32: ceil(K/2) live pairs, the other
  // warps sit the sums out
  const int kp2 = KJ == 1 ? (K + 1) >> 1 : 16;
  const bool cact = tid < 16 * kp2;
  const int cf = (tid / kp2) * 4, ck = (tid % kp2) * 2;
  const int f0 = blockIdx.x * TF, vf = min(TF, F - f0);
  const int nbeg = blockIdx.y * seg_cols, nend = min(N, nbeg + seg_cols);

  const bool k16 = (K & 3) == 0;
  const RowMap rmap = row_map(k16 ? K : 4);
  // stage step n0 into buffer b: H~_p rows and the V tile (one cp.async group)
  auto stage = [&](int n0, int b) {
    const int vn = min(NC, nend - n0);
    float* hs = B0 + b * bsz;
    if (k16) rows_async16(hs, Hc + (size_t)n0 * K, NC, vn, K, rs, rmap);
    else tile_async(hs, Hc + (size_t)n0 * K, NC, vn, K, rs, kr);
    vtile_async(hs + NC * rs + 64, a.V + (size_t)f0 * a.ldv + n0, a.ldv, vf, vn);
    cp_commit();
  };
  tile_async(Ws, Wt + (size_t)f0 * K, TF, vf, K, rs, kr);
  if (nbeg < nend) stage(nbeg, 0);

  double pn[KJ][4][2], pd[KJ][4][2];
#pragma unroll
  for (int j = 0; j < KJ; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) { pn[j][i][0] = pn[j][i][1] = 0.0; pd[j][i][0] = pd[j][i][1] = 0.0; }
  double obj = 0.0;

  int buf = 0;
  for (int n0 = nbeg; n0 < nend; n0 += NC, buf ^= 1) {
    const int valid_n = min(NC, nend - n0);
    cp_wait_all();
    __syncthreads();                       // step n0 visible; buffer buf^1 and Z free
    if (n0 + NC < nend) stage(n0 + NC, buf ^ 1);
    const float* Hs = B0 + buf * bsz;
    const float* Vs = Hs + NC * rs + 64;
    float x[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) x[i][j] = Vs[(tf * 4 + i) * VS + tn + 16 * j];
    float y[4][2];
    vt_tile(Ws, Hs, rs, kr, tf, tn, y);
    float zn[4][2], zd[4][2], ob = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        zn[i][j] = 0.f; zd[i][j] = 0.f;
        const int f = tf * 4 + i, n = tn + 16 * j;
        if (f < vf && n < valid_n) {
          ob += zdiv<BC>(x[i][j], y[i][j] + kappa, beta, zn[i][j], zd[i][j]);
        }
      }
    obj += double(ob);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int n = tn + 16 * j;
      *reinterpret_cast<float4*>(ZnT + n * TFP + tf * 4) =
          make_float4(zn[0][j], zn[1][j], zn[2][j], zn[3][j]);
      *reinterpret_cast<float4*>(ZdT + n * TFP + tf * 4) =
          make_float4(zd[0][j], zd[1][j], zd[2][j], zd[3][j]);
    }
    __syncthreads();
    // P[f][k] += sum_n Zn[f][n] H~[n][k]  (and Zd)
    float sn[KJ][4][2], sd[KJ][4][2];
#pragma unroll
    for (int j = 0; j < KJ; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) { sn[j][i][0] = sn[j][i][1] = 0.f; sd[j][i][0] = sd[j][i][1] = 0.f; }
    const int ne = cact ? valid_n : 0;
#pragma unroll 4
    for (int n = 0; n < ne; ++n) {
      const float4 z = *reinterpret_cast<const float4*>(ZnT + n * TFP + cf);
      const float4 d = *reinterpret_cast<const float4*>(ZdT + n * TFP + cf);
      const float zz[4] = {z.x, z.y, z.z, z.w}, dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int j = 0; j < KJ; ++j) {
        const float2 h = *reinterpret_cast<const float2*>(Hs + n * rs + ck + 32 * j);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sn[j][i][0] = fmaf(zz[i], h.x, sn[j][i][0]); sn[j][i][1] = fmaf(zz[i], h.y, sn[j][i][1]);
          sd[j][i][0] = fmaf(dd[i], h.x, sd[j][i][0]); sd[j][i][1] = fmaf(dd[i], h.y, sd[j][i][1]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          pn[j][i][v] += double(sn[j][i][v]);
          pd[j][i][v] += double(sd[j][i][v]);
        }
  }
  cp_wait_all();
  // this segment's slab: rows [f0, f0+vf) of part[seg][2][F][K]
  double* slab = a.part + (size_t)blockIdx.y * 2 * F * K;
#pragma unroll
  for (int j = 0; j < KJ; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int f = cf + i, k = ck + 32 * j + v;
        if (cact && f < vf && k < K) {
          const size_t idx = (size_t)(f0 + f) * K + k;
          slab[idx] = pn[j][i][v];
          slab[(size_t)F * K + idx] = pd[j][i][v];
        }
      }
  for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
  if ((tid & 31) == 0) red[tid >> 5] = obj;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < THREADS / 32; ++w) t += red[w];
    a.opart[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

}  // namespace fs2
}  // namespace bnmf
