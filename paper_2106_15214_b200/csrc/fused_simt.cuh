// SIMT implementation of the fused single-read pass (fp32, any F, K <= 64).
// It is the correctness twin of the tcgen05 pass (fused_tc.cu) and the pass
// used when that kernel's shape limits are not met.  One CTA walks column
// blocks of 32 columns x all F rows (persistent, grid-stride); per block it
// finishes the H update and produces the W-side partial sums, accumulated in
// a per-CTA fp64 slab (fixed order => deterministic).
#pragma once

#include "fused_common.cuh"
#include "simt_kernels.cuh"

namespace bnmf {

constexpr int FS_KMAX = 64;

template <int BC>
__global__ void __launch_bounds__(ST_THREADS)
fused_pass_simt(FusedArgs a, const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, F = a.F, N = a.N;
  const int ks = kstride(K);
  float* Hp = reinterpret_cast<float*>(smem_raw);   // H~_{p-1} block  [NC][ks]
  float* Hn = Hp + ST_NC * ks;                      // H~_p block      [NC][ks]
  float* Ws = Hn + ST_NC * ks;                      // W rows          [TF][ks]
  float* C1s = Ws + ST_TF * ks;
  float* C2s = C1s + ST_TF * ks;
  float* Zn = C2s + ST_TF * ks;                     // [TF][NC+1]
  float* Zd = Zn + ST_TF * (ST_NC + 1);
  __shared__ double red[ST_THREADS / 32];

  const int par = iter_parity(st, slot, p_override);
  const float* Hprev = a.do_h ? a.Hbuf[par ^ 1] : a.Hbuf[par];
  float* Hnew = a.Hout[par];
  const float* Wt = a.Wt2[par];                                 // W~_p
  const float* Wa = a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn;   // H-side factor
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  const int tl = threadIdx.x & 31, kg = threadIdx.x >> 5;
  double* mypart = a.part + (size_t)blockIdx.x * 2 * F * K;
  double obj = 0.0;

  // zero this CTA's partial slab
  for (int i = threadIdx.x; i < 2 * F * K; i += blockDim.x) mypart[i] = 0.0;

  const int nblocks = (N + ST_NC - 1) / ST_NC;
  for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const int n0 = b * ST_NC;
    const int valid_n = min(ST_NC, N - n0);
    __syncthreads();
    load_rows(Hp, Hprev + (size_t)n0 * K, ST_NC, valid_n, K, ks);
    if (a.do_h) {
      // ---- H-side: finish H_p for this block --------------------------------
      double accn[FS_KMAX / 8], accd[FS_KMAX / 8];
#pragma unroll
      for (int j = 0; j < FS_KMAX / 8; ++j) { accn[j] = 0.0; accd[j] = 0.0; }
      for (int f0 = 0; f0 < F; f0 += ST_TF) {
        __syncthreads();
        int vf = min(ST_TF, F - f0);
        load_rows(Ws, Wa + (size_t)f0 * K, ST_TF, vf, K, ks);
        load_rows(C1s, a.C1 + (size_t)f0 * K, ST_TF, vf, K, ks);
        if (!a.den_ones) load_rows(C2s, a.C2 + (size_t)f0 * K, ST_TF, vf, K, ks);
        __syncthreads();
        for (int e = threadIdx.x; e < ST_TF * ST_NC; e += blockDim.x) {
          int f = e / ST_NC, n = e - f * ST_NC;
          float zn = 0.f, zd = 0.f;
          if (f0 + f < F && n < valid_n) {
            float y = 0.f;
            for (int k = 0; k < K; ++k) y = fmaf(Ws[f * ks + k], Hp[n * ks + k], y);
            y += kappa;
            bases32<BC>(a.V[(size_t)(f0 + f) * a.ldv + n0 + n], y, beta, zn, zd);
          }
          Zn[f * (ST_NC + 1) + n] = zn;
          Zd[f * (ST_NC + 1) + n] = zd;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < FS_KMAX / 8; ++j) {
          int k = kg + 8 * j;
          if (k < K) {
            float sn = 0.f, sd = 0.f;
            for (int f = 0; f < ST_TF; ++f) {
              sn = fmaf(C1s[f * ks + k], Zn[f * (ST_NC + 1) + tl], sn);
              if (!a.den_ones) sd = fmaf(C2s[f * ks + k], Zd[f * (ST_NC + 1) + tl], sd);
            }
            accn[j] += double(sn);
            accd[j] += double(sd);
          }
        }
      }
      // H_p = H~_{p-1} * ratio^gamma ;  H~_p = H_p * norms
      if (tl < valid_n) {
#pragma unroll
        for (int j = 0; j < FS_KMAX / 8; ++j) {
          int k = kg + 8 * j;
          if (k < K) {
            double den = a.den_ones ? a.csum2[k] : accd[j];
            double r = accn[j] / fmax(den, a.sc.floor);
            double h = double(Hp[tl * ks + k]) * apply_exponent<double>(r, a.sc.gamma);
            float hn = float(h * a.norms[k]);
            Hn[tl * ks + k] = hn;
            Hnew[(size_t)(n0 + tl) * K + k] = hn;
          }
        }
      } else {
        for (int j = 0; j < FS_KMAX / 8; ++j) {
          int k = kg + 8 * j;
          if (k < K) Hn[tl * ks + k] = 0.f;
        }
      }
    } else {
      __syncthreads();
      for (int i = threadIdx.x; i < ST_NC * ks; i += blockDim.x) Hn[i] = Hp[i];
    }
    // ---- W-side + objective with Vt_p = W~_p H~_p + kappa -----------------
    for (int f0 = 0; f0 < F; f0 += ST_TF) {
      __syncthreads();
      load_rows(Ws, Wt + (size_t)f0 * K, ST_TF, min(ST_TF, F - f0), K, ks);
      __syncthreads();
      for (int e = threadIdx.x; e < ST_TF * ST_NC; e += blockDim.x) {
        int f = e / ST_NC, n = e - f * ST_NC;
        float zn = 0.f, zd = 0.f;
        if (f0 + f < F && n < valid_n) {
          float y = 0.f;
          for (int k = 0; k < K; ++k) y = fmaf(Ws[f * ks + k], Hn[n * ks + k], y);
          y += kappa;
          float x = a.V[(size_t)(f0 + f) * a.ldv + n0 + n];
          obj += double(divergence32<BC>(x, y, beta));
          bases32<BC>(x, y, beta, zn, zd);
        }
        Zn[f * (ST_NC + 1) + n] = zn;
        Zd[f * (ST_NC + 1) + n] = zd;
      }
      __syncthreads();
      if (f0 + tl < F) {
        for (int j = 0; j < FS_KMAX / 8; ++j) {
          int k = kg + 8 * j;
          if (k < K) {
            float sn = 0.f, sd = 0.f;
            for (int n = 0; n < ST_NC; ++n) {
              sn = fmaf(Zn[tl * (ST_NC + 1) + n], Hn[n * ks + k], sn);
              sd = fmaf(Zd[tl * (ST_NC + 1) + n], Hn[n * ks + k], sd);
            }
            size_t idx = (size_t)(f0 + tl) * K + k;
            mypart[idx] += double(sn);
            mypart[(size_t)F * K + idx] += double(sd);
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = obj;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < ST_THREADS / 32; ++w) t += red[w];
    a.opart[blockIdx.x] = t;
  }
}

// comm[0:2FK] = sum_g part[g], comm[2FK] = sum_g opart[g]  (fixed order)
// Fixed-order sum of the per-CTA partials.  With a row-split cluster
// (cl == 2) CTA g owns rows [0, split) when g is even, else [split, F); it
// only writes its own rows, so row f sums the CTAs of its owner rank.
static __global__ void fused_reduce(const double* __restrict__ part, const double* __restrict__ opart,
                             int G, int FK2, int K, int split, int cl, double* __restrict__ comm,
                             const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < FK2) {
    const int f = (i % (FK2 / 2)) / K;
    const int r = (cl > 1 && f >= split) ? 1 : 0;
    double s = 0.0;
    for (int g = r; g < G; g += cl) s += part[(size_t)g * FK2 + i];
    comm[i] = s;
  } else if (i == FK2) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += opart[g];
    comm[i] = s;
  }
}

// W update for iteration p+1 and everything pass p+1 needs (one block per k):
//   W_{p+1} = W~_p * (num/max(den,floor))^gamma   (updates.py:203-220)
//   norms_{p+1}, W~_{p+1} = W_{p+1}/norms (solver.py:167-171)
//   C1 = chi1(W_{p+1}, W~_p), C2 = chi2(...) (JMM) or W_{p+1} (BMM)
struct WPair { float* w[2]; };

static __global__ void fused_update(const double* __restrict__ comm, int F, int K,
                             WPair Wt2, float* Wn, float* C1, float* C2, double* norms,
                             double* csum2,
                             int algorithm, int den_ones, Scalars sc, const RunState* st, int slot,
                             int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
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
