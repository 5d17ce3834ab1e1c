// tcgen05 implementation of the fused single-read pass (fp32, rank K <= 16,
// F <= 256).  Same contract as the SIMT pair fs2::hpass + fs2::wpass (fused_common.cuh).
//
// Rows of V are split over a cluster of CL CTAs (CL = 2 when F > 128): CTA r
// owns rows [row0, row0 + FTr) and every column block of its cluster, so
// all of its V rows of a block (<= 128 x 128 fp32) stay resident in SMEM for
// both phases and V is read from HBM exactly once per pass.
//
// Warp roles (18 warps, one CTA per SM):
//   warp 0      TMA producer: V stages [32 rows x 132 cols] (528 B padded rows,
//               conflict-free in both phases) into a 7-stage ring
//   warp 1      MMA issuer (warp-uniform loop, one elected lane issues) + TMEM owner
//   warps 2..17 epilogue: TMEM -> registers, the beta-dependent terms,
//               Z back to TMEM as the A operand of the side products, the
//               H update, the objective, fp64 folding of the W sums
//
// Per column block (n0 .. n0+127), items in epilogue order:
//   H(j)   j < SH      D[n x 32 f] = H~_{p-1} Wa[j]^T  (3xTF32, A from TMEM)
//                      Z = Zn, Zd of (V, D + kappa) -> TMEM
//                      AccH[n x k] += Z * [chi_hi | chi_lo]     (A from TMEM)
//   U                  AccH of the cluster combined over DSMEM (st.async),
//                      H~_p = H~_{p-1} (num/den)^gamma norms -> SMEM + HBM
//   W(u)   u < 4       D[f x 32 n] = W~_p H~_p[u]^T; objective;
//                      AccW[f x k] += Z * [H~_hi | H~_lo]
// The first H item of block b+1 is processed before U(b) so that the AccH
// drain and the DSMEM exchange overlap epilogue work.
//
// Numerics: every product is 3xTF32 (hi*hi + hi*lo + lo*hi).  The side
// products issue Z_hi * [B_hi | B_lo] as one N = 32 MMA (the two halves of
// the accumulator are summed at readout) plus Z_lo * B_hi (N = 16).  All
// reductions have a fixed order (bitwise reproducible).
#pragma once

#include <cuda.h>

#include "fused_common.cuh"
#include "tc_primitives.cuh"

namespace bnmf {
namespace ftc {

using namespace bnmf::tc;

constexpr int BN = 128;            // columns per block
constexpr int KP = 16;             // padded rank
constexpr int FR = 128;            // rows per CTA (max)
constexpr int SW = BN / 32;        // W items per block
constexpr int NEPI = 16;           // epilogue warps (4 per TMEM lane quadrant)
constexpr int NTHREADS = 32 * (2 + NEPI);
constexpr int FOLD = 8;            // blocks accumulated in TMEM before the fp64 fold
constexpr int VROW = 132;          // padded SMEM row of a V stage (floats)
constexpr uint32_t VROWB = VROW * 4;
constexpr uint32_t STAGE_BYTES = 32 * VROWB;
constexpr int NSTAGE = 7;

// TMEM columns (512 allocated)
constexpr uint32_t TM_D = 0;       // Vt tiles, 2 x 32
constexpr uint32_t TM_Z = 64;      // Z, 2 x 128: k-step s -> Zn hi, Zn lo, Zd hi, Zd lo at 32s + 8i
constexpr uint32_t TM_ACCH = 320;  // num [hi part 16 | lo part 16], den at +32
constexpr uint32_t TM_ACCW = 384;  // same layout
constexpr uint32_t TM_HP = 448;    // H~_{p-1} rows of the block: hi 16 | lo 16
constexpr uint32_t TM_WT = 480;    // W~_p rows of this CTA: hi 16 | lo 16

// SMEM layout (bytes from the 1024-aligned base)
constexpr uint32_t OFF_STAGE = 0;
constexpr uint32_t OFF_WA = OFF_STAGE + NSTAGE * STAGE_BYTES;   // [128 f x 16] hi, lo (core tiles)
constexpr uint32_t OFF_C1 = OFF_WA + 2 * FR * KP * 4;           // [32 (k hi, k lo) x 128 f]
constexpr uint32_t OFF_C2 = OFF_C1 + 2 * FR * KP * 4;
constexpr uint32_t OFF_HN = OFF_C2 + 2 * FR * KP * 4;           // [128 n x 16] hi, lo
// H~_p transposed (B of the W-side products, K-major over n): rows k (hi) and 16 + k (lo),
// core matrices of 8 k x 4 n.  The 4-column chunks sit 144 B apart (not 128) so that a warp
// storing one k of 32 consecutive columns hits 32 different banks.
constexpr uint32_t HNT_LBO = 144;
constexpr uint32_t HNT_SBO = (BN / 4) * HNT_LBO;                // 8-row (k) group stride
constexpr uint32_t OFF_HNT = OFF_HN + 2 * BN * KP * 4;
constexpr uint32_t OFF_XCH = OFF_HNT + 4 * HNT_SBO;             // peer's AccH partial
constexpr uint32_t OFF_BAR = OFF_XCH + BN * 2 * KP * 4;
constexpr uint32_t SMEM_BYTES = OFF_BAR + 512 + 1024;           // + alignment slack
constexpr uint32_t HILO = FR * KP * 4;                          // hi -> lo offset (8 KB)
static_assert(SMEM_BYTES <= 232448, "fused_pass_tc: shared memory over the 227 KB limit");

// beta class of the fused TC epilogue (adds the beta = 1.5 fast form)
enum { FBC_GEN = 0, FBC_0 = 1, FBC_1 = 2, FBC_2 = 3, FBC_15 = 4 };

// element (k, c) of a K-major [R rows x 128] tile whose K dimension is c:
// 8-row groups at SBO = 4096 B, 4-wide chunks of c at LBO = 128 B
__host__ __device__ __forceinline__ uint32_t coreT_off(int k, int c) {
  return uint32_t((k >> 3) * 4096 + (c >> 2) * 128 + (k & 7) * 16 + (c & 3) * 4);
}
// element (k, n) of the transposed H~_p tile (k < 32: hi rows 0..15, lo rows 16..31)
__host__ __device__ __forceinline__ uint32_t hnt_off(int k, int n) {
  return uint32_t((k >> 3) * HNT_SBO + (n >> 2) * HNT_LBO + (k & 7) * 16 + (n & 3) * 4);
}

template <int FBC>
__device__ __forceinline__ void zpair(float x, float y, float beta, float& zn, float& zd) {
  if (FBC == FBC_15) {
    const float r = rsqrt_fast(y);
    zn = x * r;
    zd = y * r;
  } else if (FBC == FBC_2) {
    zn = x; zd = y;
  } else if (FBC == FBC_1) {
    zn = __fdividef(x, y); zd = 1.f;
  } else if (FBC == FBC_0) {
    const float r = __fdividef(1.f, y);
    zn = x * r * r; zd = r;
  } else {
    bases32<BC_GEN>(x, y, beta, zn, zd);
  }
}

template <int FBC>
__device__ __forceinline__ float dterm(float x, float y, float zd, float beta) {
  if (FBC == FBC_15) {
    const float sx = sqrt_fast(x);
    const float dq = sx - zd;
    return 0.6666666666666666f * dq * dq * fmaf(2.f, sx, zd);
  } else if (FBC == FBC_2) {
    return divergence32<BC_2>(x, y, beta);
  } else if (FBC == FBC_1) {
    return divergence32<BC_1>(x, y, beta);
  } else if (FBC == FBC_0) {
    return divergence32<BC_0>(x, y, beta);
  }
  return divergence32<BC_GEN>(x, y, beta);
}

// acc += d(x|y), except beta = 1.5: acc += (3/2) d(x|y) (the caller applies 2/3 once)
template <int FBC>
__device__ __forceinline__ void dacc(float x, float y, float zd, float beta, float& acc) {
  if (FBC == FBC_15) {
    // d_{3/2}(x|y) = (2/3) (sqrt x - sqrt y)^2 (2 sqrt x + sqrt y); zd = sqrt y
    const float sx = sqrt_fast(x);
    const float dq = sx - zd;
    acc = fmaf(dq * dq, fmaf(2.f, sx, zd), acc);
  } else {
    acc += dterm<FBC>(x, y, zd, beta);
  }
}

// Z and the objective term of one element from ONE reciprocal (W items of the item-team
// kernels).  beta = 0 and beta = 1 need u = (x - y) / y for their cancellation-free objective
// forms; divergence32 gets it from an IEEE division and a 14-term series, which made the W items
// of these classes ~10x the H items.  Here u = (x - y) rcp(y) with the reciprocal Z needs anyway,
// an 8-term Horner series for |u| < 1/8 (truncation < 2^-24 of the term) and the MUFU log beyond.
// series coefficients of phi(u) = [(1 + u)^b - 1 - b u] / (b (b - 1)) = sum_{j >= 2} t_j u^j,
// t_2 = 1/2, t_{j+1} = t_j (b - j) / (j + 1): computed once per thread (generic beta)
constexpr int PHI_TERMS = 12;
__device__ __forceinline__ void phi_coeffs(float b, float* pc) {
  float t = 0.5f;
#pragma unroll
  for (int j = 2; j < 2 + PHI_TERMS; ++j) {
    pc[j - 2] = t;
    t = t * (b - float(j)) / float(j + 1);
  }
}

template <int FBC>
__device__ __forceinline__ void z_and_obj(float x, float y, float zd_in, float beta, float& zn,
                                          float& zd, float& acc, const float* pc = nullptr) {
  (void)zd_in;
  if (FBC == FBC_0) {
    const float r = rcp_fast(y);
    zd = r;
    zn = x * r * r;
    const float u = (x - y) * r;
    float d;
    if (fabsf(u) < 0.125f) {
      // u - log1p(u) = u^2 (1/2 - u/3 + u^2/4 - ...)
      float p = -0.1111111111f;
      p = fmaf(p, u, 0.125f);
      p = fmaf(p, u, -0.1428571429f);
      p = fmaf(p, u, 0.1666666667f);
      p = fmaf(p, u, -0.2f);
      p = fmaf(p, u, 0.25f);
      p = fmaf(p, u, -0.3333333333f);
      p = fmaf(p, u, 0.5f);
      d = p * u * u;
    } else {
      const float t = x * r;
      d = t - __logf(t) - 1.f;
    }
    acc += d;
  } else if (FBC == FBC_1) {
    const float r = rcp_fast(y);
    zn = x * r;
    zd = 1.f;
    const float u = (x - y) * r;
    float d;
    if (fabsf(u) < 0.125f) {
      // (1 + u) log1p(u) - u = u^2 (1/2 - u/6 + u^2/12 - u^3/20 + ...), coefficient 1 / (j (j - 1))
      float p = 0.0138888889f;            // 1 / 72
      p = fmaf(p, u, -0.0178571429f);     // 1 / 56
      p = fmaf(p, u, 0.0238095238f);      // 1 / 42
      p = fmaf(p, u, -0.0333333333f);     // 1 / 30
      p = fmaf(p, u, 0.05f);              // 1 / 20
      p = fmaf(p, u, -0.0833333333f);     // 1 / 12
      p = fmaf(p, u, 0.1666666667f);      // 1 / 6
      p = fmaf(p, u, -0.5f);
      d = -p * u * u * y;
    } else if (x == 0.f) {
      d = y;
    } else {
      d = x * __logf(x * r) - x + y;
    }
    acc += d;
  } else if (FBC == FBC_GEN && pc != nullptr) {
    // one powf: a = y^(beta-2) gives Z, y^(beta-1) = a y and y^beta = a y^2; the objective is
    // y^beta phi(u) by its series (Horner, coefficients in pc) for |u| < 1/4, the three-term
    // form (one more powf) beyond
    const float a = powf(y, beta - 2.f);
    zn = x * a;
    zd = a * y;
    const float u = (x - y) * rcp_fast(y), yb = zd * y;
    float d;
    if (fabsf(u) < 0.25f) {
      float p = pc[PHI_TERMS - 1];
#pragma unroll
      for (int j = PHI_TERMS - 2; j >= 0; --j) p = fmaf(p, u, pc[j]);
      d = yb * p * u * u;
    } else {
      d = powf(x, beta) / (beta * (beta - 1.f)) + yb / beta - x * zd / (beta - 1.f);
    }
    acc += d;
  } else {
    zpair<FBC>(x, y, beta, zn, zd);
    dacc<FBC>(x, y, zd, beta, acc);
  }
}

// KKT gradient core y^(beta-2) (y - x) (diagnostics.py:51-54), formed per element so that the
// side products accumulate the gradient itself instead of two sums that cancel
template <int FBC>
__device__ __forceinline__ float gcore32(float x, float y, float beta) {
  const float d = y - x;
  if (FBC == FBC_2) return d;
  if (FBC == FBC_15) return d * rsqrt_fast(y);
  const float r = rcp_fast(y);
  if (FBC == FBC_1) return d * r;
  if (FBC == FBC_0) return d * r * r;
  return d * powf(y, beta - 2.f);
}

// Z for 8 elements; beta = 1.5 forms two lanes per instruction (FMUL2)
template <int FBC>
__device__ __forceinline__ void zpair8(const float* x, const float* y, float beta, float* zn,
                                       float* zd) {
#ifndef BNMF_NO_F2
  if (FBC == FBC_15) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      const uint64_t r = f2pack(rsqrt_fast(y[i]), rsqrt_fast(y[i + 1]));
      f2unpack(f2mul(f2pack(x[i], x[i + 1]), r), zn[i], zn[i + 1]);
      f2unpack(f2mul(f2pack(y[i], y[i + 1]), r), zd[i], zd[i + 1]);
    }
    return;
  }
#endif
#pragma unroll
  for (int i = 0; i < 8; ++i) zpair<FBC>(x[i], y[i], beta, zn[i], zd[i]);
}

// Z of one k-step (this thread's 8 columns) as TMEM A operands:
// [Zn hi | Zn lo | Zd hi | Zd lo], 8 columns each, one 32-column store
__device__ __forceinline__ void store_z(uint32_t taddr, const float* zn, const float* zd) {
#ifdef BNMF_Z1
  float a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = to_tf32(zn[i]); b[i] = to_tf32(zd[i]); }
  tmem_st8(taddr, a);
  tmem_st8(taddr + 16, b);
  return;
#endif
  float z[32];
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    z[i] = tf32_trunc(zn[i]);
    z[i + 1] = tf32_trunc(zn[i + 1]);
    z[16 + i] = tf32_trunc(zd[i]);
    z[17 + i] = tf32_trunc(zd[i + 1]);
#ifdef BNMF_NO_F2
    z[8 + i] = zn[i] - z[i];
    z[9 + i] = zn[i + 1] - z[i + 1];
    z[24 + i] = zd[i] - z[16 + i];
    z[25 + i] = zd[i + 1] - z[17 + i];
#else
    // the lo parts two at a time (FADD2)
    f2unpack(f2sub(f2pack(zn[i], zn[i + 1]), f2pack(z[i], z[i + 1])), z[8 + i], z[9 + i]);
    f2unpack(f2sub(f2pack(zd[i], zd[i + 1]), f2pack(z[16 + i], z[17 + i])), z[24 + i], z[25 + i]);
#endif
  }
  tmem_st32(taddr, z);
}

// smem descriptor arithmetic: the start-address field is addr >> 4 in the low
// 14 bits, so desc(addr + off) == desc(addr) + (off >> 4) for smem < 256 KB.
__device__ __forceinline__ uint64_t dplus(uint64_t d, uint32_t off) { return d + (off >> 4); }

// D = A * B^T over K = 16 in 3xTF32: (hi,hi) + (hi,lo) + (lo,hi), 2 k-steps
// each; A (M x 16, hi/lo) in TMEM columns a_hi / a_lo, B K-major core tiles.
__device__ __forceinline__ void issue_vt(uint32_t dcol, uint32_t a_hi, uint32_t a_lo,
                                         uint64_t b_hi, uint64_t b_lo, uint32_t idesc) {
  mma_ts(dcol, a_hi, b_hi, idesc, 0u);
  mma_ts(dcol, a_hi + 8, dplus(b_hi, 256), idesc, 1u);
  mma_ts(dcol, a_hi, b_lo, idesc, 1u);
  mma_ts(dcol, a_hi + 8, dplus(b_lo, 256), idesc, 1u);
  mma_ts(dcol, a_lo, b_hi, idesc, 1u);
  mma_ts(dcol, a_lo + 8, dplus(b_hi, 256), idesc, 1u);
}

// acc[:, 0:32] (+)= Z_hi * [B_hi | B_lo], acc[:, 0:16] += Z_lo * B_hi over a
// 32-wide K slab: Z hi/lo of k-step s at TMEM columns z + 32 s (+8 for lo),
// B (32 x K, K-major) from descriptor b, 256 B per k-step.
template <uint32_t KSTRIDE>
__device__ __forceinline__ void issue_side(uint32_t acc, uint32_t z, uint64_t b, uint32_t id32,
                                           uint32_t id16, bool fresh) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    mma_ts(acc, z + 32 * s, dplus(b, KSTRIDE * s), id32, (fresh && s == 0) ? 0u : 1u);
#ifndef BNMF_Z1
    mma_ts(acc, z + 32 * s + 8, dplus(b, KSTRIDE * s), id16, 1u);
#endif
  }
}

template <int FBC, bool KAPPA>
__global__ void __launch_bounds__(NTHREADS, 1)
fused_pass_tc(FusedArgs a, const __grid_constant__ CUtensorMap mapV, int CL, int F0,
              const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  // first kernel of an iteration: the start of its timer (begin_iter folded in, solver.py:302)
  if (a.tmark && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.tmark = globaltimer();
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* bar_full = bars;          // [NSTAGE] TMA -> epilogue
  uint64_t* bar_empty = bars + 8;     // [NSTAGE] epilogue -> TMA
  uint64_t* bar_dfull = bars + 16;    // [2] Vt tile ready
  uint64_t* bar_zfull = bars + 18;    // [2] Z written
  uint64_t* bar_hp = bars + 22;       // H~_{p-1} of the next block in TMEM
  uint64_t* bar_hn = bars + 23;       // H~_p of the block in SMEM (both layouts)
  uint64_t* bar_acch = bars + 24;     // AccH of the block complete
  uint64_t* bar_accfree = bars + 25;  // AccH read out
  uint64_t* bar_accw = bars + 26;     // AccW of a fold complete
  uint64_t* bar_accwfree = bars + 27; // AccW read out
  uint64_t* bar_wdone = bars + 28;    // W-side MMAs of a block retired
  uint64_t* bar_xfull = bars + 29;    // peer's AccH partial landed (tx)
  uint64_t* bar_xempty = bars + 30;   // peer consumed my partial (remote arrivals)
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 40);
  __shared__ double s_red[NEPI];
  // optional wait-cycle counters (build with BNMF_TC_PROF=1; one thread per role records)
#ifdef BNMF_TC_PROF
  long long* prof = a.prof ? a.prof + size_t(blockIdx.x) * 48 : nullptr;
  __shared__ unsigned long long pcs[48];
  for (int i = threadIdx.x; i < 48; i += blockDim.x) pcs[i] = 0;
  __syncthreads();
  const bool rec = prof && (threadIdx.x & 31) == 0 && (threadIdx.x < 96);
  const int pbase = (threadIdx.x >> 5) * 12;
  auto pwait = [&](uint64_t* bar, uint32_t parity, int cat) {
    if (rec) {
      const long long t0 = clock64();
      mbar_wait(bar, parity);
      atomicAdd(&pcs[pbase + cat], (unsigned long long)(clock64() - t0));
    } else {
      mbar_wait(bar, parity);
    }
  };
  auto pwait_cl = pwait;
  const long long t_start = clock64();
  // event timeline of CTA 0 (lane 0 of warps 0..2): clock << 16 | ev << 10 | pos
  long long* trace_buf = (a.prof && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && threadIdx.x < 96)
                             ? a.prof + size_t(gridDim.x) * 48 + (threadIdx.x >> 5) * 4096
                             : nullptr;
  int trace_n = 0;
  auto trace = [&](int ev, int pos) {
    if (trace_buf && trace_n < 4095)
      trace_buf[trace_n++] = (clock64() << 16) | (long long)(ev << 10) | (pos & 1023);
  };
#define BNMF_TRACE(ev, pos) trace(ev, pos)
#define BNMF_PROF_T0(v) const long long v = clock64()
#define BNMF_PROF_ADD(i, v) if (rec) atomicAdd(&pcs[pbase + (i)], (unsigned long long)(clock64() - (v)))
#else
  auto pwait = [&](uint64_t* bar, uint32_t parity, int) { mbar_wait(bar, parity); };
  auto pwait_cl = [&](uint64_t* bar, uint32_t parity, int) { mbar_wait(bar, parity); };
#define BNMF_PROF_T0(v)
#define BNMF_PROF_ADD(i, v)
#define BNMF_TRACE(ev, pos)
#endif

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = a.F, N = a.N, K = a.K;
  const uint32_t rank = CL > 1 ? cluster_ctarank() : 0u;
  const int row0 = rank ? F0 : 0;
  const int FTr = rank ? F - F0 : (F < F0 ? F : F0);
  const int SH = max(2, (FTr + 31) / 32);
  const int npairs = gridDim.x / CL, pi = blockIdx.x / CL;
  const int nblocks = (N + BN - 1) / BN;
  const int nb = pi < nblocks ? (nblocks - 1 - pi) / npairs + 1 : 0;
  const int par = iter_parity(st, slot, p_override);
  const float* Hprev = a.do_h ? a.Hbuf[par ^ 1] : a.Hbuf[par];
  float* Hnew = a.Hout[par];
  const float* Wt = a.Wt2[par];
  const float* Wa = a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn;
  const int do_h = a.do_h;
  const int den_ones = a.den_ones;
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);

  // item sequence of this CTA (the MMA warp and the epilogue walk it in the
  // same order): block bi lists its own H items (all of them for bi == 0,
  // else 2..SH-1), then H(bi+1, 0) [U1(bi)] H(bi+1, 1) [U2(bi)], then
  // W(bi, 0..SW-1).  U1 reads AccH and sends it to the peer CTA, U2 finishes
  // the H update; the H items between them hide the AccH drain and the
  // exchange.
  auto col0 = [&](int blk) { return (pi + blk * npairs) * BN; };
  auto stage_of = [&](int blk, int j, uint32_t& ph) {
    const int cnt = blk * SH + j;
    ph = uint32_t(cnt / NSTAGE) & 1u;
    return cnt % NSTAGE;
  };

  // ---- setup: barriers, TMEM, constant operands ---------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], NEPI);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_dfull[b], 1);
      mbar_init(&bar_zfull[b], NEPI);
    }
    mbar_init(bar_hp, NEPI);
    mbar_init(bar_hn, NEPI);
    mbar_init(bar_acch, 1);
    mbar_init(bar_accfree, NEPI);
    mbar_init(bar_accw, 1);
    mbar_init(bar_accwfree, NEPI);
    mbar_init(bar_wdone, 1);
    mbar_init(bar_xfull, 1);
    mbar_init(bar_xempty, NEPI);
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch(&mapV);
  if (warp == 1) tmem_alloc<512>(s_tmem);
  if (warp >= 2) {
    // Wa (B of the H-side Vt product): [f x k] core tiles, hi then lo.
    // chi1/chi2 (B of the H-side products): K-major over f, rows k (hi) and 16+k (lo).
    for (int i = threadIdx.x - 64; i < FR * KP; i += NEPI * 32) {
      const int fl = i / KP, k = i - fl * KP;
      const bool ok = fl < FTr && k < K;
      const size_t gi = size_t(row0 + fl) * K + k;
      float v, hi;
      v = ok ? Wa[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + OFF_WA + core_off(fl, k), hi);
      sts_f32(sb + OFF_WA + HILO + core_off(fl, k), v - hi);
      v = ok ? a.C1[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + OFF_C1 + coreT_off(k, fl), hi);
      sts_f32(sb + OFF_C1 + coreT_off(k + 16, fl), v - hi);
      v = ok ? a.C2[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + OFF_C2 + coreT_off(k, fl), hi);
      sts_f32(sb + OFF_C2 + coreT_off(k + 16, fl), v - hi);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();   // peer barriers initialised before any remote op
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

  if (warp == 0) {
    // ======================= TMA producer ===================================
    if (lane == 0) {
#ifndef BNMF_L2PF
#define BNMF_L2PF 1
#endif
      // V rows of block bi + BNMF_L2PF are prefetched into L2 when the stage
      // loads of block bi are issued: a stage refill (issued when the W items
      // of the block two back release their slots) then hits L2 instead of
      // waiting a full DRAM latency
      for (int bi = 0; bi < BNMF_L2PF && bi < nb; ++bi)
        for (int j = 0; j < SH; ++j) tma_prefetch_l2_2d(&mapV, col0(bi), row0 + 32 * j);
      for (int bi = 0; bi < nb; ++bi) {
        const int n0 = col0(bi);
        for (int j = 0; j < SH; ++j) {
          uint32_t ph;
          const int s = stage_of(bi, j, ph);
          if (BNMF_L2PF > 0 && bi + BNMF_L2PF < nb)
            tma_prefetch_l2_2d(&mapV, col0(bi + BNMF_L2PF), row0 + 32 * j);
          pwait(&bar_empty[s], ph ^ 1, 0);
          mbar_expect_tx(&bar_full[s], STAGE_BYTES);
          tma_load_2d(smem + OFF_STAGE + s * STAGE_BYTES, &mapV, &bar_full[s], n0, row0 + 32 * j);
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (warp-uniform) ======================
    // Straight-line per block, Vt tile of the next item issued before the
    // side products of the current one: D(c) follows side(c-2), so its commit
    // (dfull) also tells the epilogue that Z buffer c & 1 is free, and
    // zfull(c - 2) (waited before side(c - 2)) told us Vt buffer c & 1 was read.
    const uint32_t id32 = idesc_tf32(128, 32, 0, 0);
    const uint32_t id16 = idesc_tf32(128, 16, 0, 0);
    const uint64_t d_wa = sdesc(sb + OFF_WA, 128, 512);
    const uint64_t d_hn = sdesc(sb + OFF_HN, 128, 512);
    const uint64_t d_c1 = sdesc(sb + OFF_C1, 128, 4096);
    const uint64_t d_c2 = sdesc(sb + OFF_C2, 128, 4096);
    const uint64_t d_hnt = sdesc(sb + OFF_HNT, HNT_LBO, HNT_SBO);
    int nd = 0, ns = 0, w0_issued = -1;
    auto d_h = [&](int blk, int j) {
      if (j == 0) {
        pwait(bar_hp, blk & 1, 2);
        tc_fence_after();
      }
      BNMF_TRACE(1, nd);
      if (elect_one()) {
        issue_vt(tmem + TM_D + 32 * (nd & 1), tmem + TM_HP, tmem + TM_HP + 16,
                 dplus(d_wa, j * 2048), dplus(d_wa, j * 2048 + HILO), id32);
        mma_commit(&bar_dfull[nd & 1]);
      }
      __syncwarp();
      BNMF_TRACE(2, nd);
      ++nd;
    };
    auto d_w = [&](int blk, int u) {
      if (u == 0) {
        BNMF_TRACE(6, nd);
        pwait(bar_hn, blk & 1, 1);
        BNMF_TRACE(7, nd);
        tc_fence_after();
        w0_issued = blk;
      }
      BNMF_TRACE(1, nd);
      if (elect_one()) {
        issue_vt(tmem + TM_D + 32 * (nd & 1), tmem + TM_WT, tmem + TM_WT + 16,
                 dplus(d_hn, u * 2048), dplus(d_hn, u * 2048 + HILO), id32);
        mma_commit(&bar_dfull[nd & 1]);
      }
      __syncwarp();
      BNMF_TRACE(2, nd);
      ++nd;
    };
    auto s_h = [&](int blk, int j) {
      BNMF_TRACE(3, ns);
      pwait(&bar_zfull[ns & 1], (ns >> 1) & 1, 3);
      BNMF_TRACE(4, ns);
      if (j == 0 && blk > 0) pwait(bar_accfree, (blk - 1) & 1, 4);
      tc_fence_after();
      const uint32_t zb = tmem + TM_Z + 128 * (ns & 1);
      if (elect_one()) {
        issue_side<256>(tmem + TM_ACCH, zb, dplus(d_c1, j * 1024), id32, id16, j == 0);
        if (!den_ones)
          issue_side<256>(tmem + TM_ACCH + 32, zb + 16, dplus(d_c2, j * 1024), id32, id16, j == 0);
        if (j == SH - 1) mma_commit(bar_acch);
      }
      __syncwarp();
      BNMF_TRACE(5, ns);
      ++ns;
    };
    auto s_w = [&](int blk, int u) {
      BNMF_TRACE(3, ns);
      const bool fresh = (blk % FOLD) == 0 && u == 0;
      const bool fold_end = (blk % FOLD) == FOLD - 1 || blk == nb - 1;
      const uint32_t zb = tmem + TM_Z + 128 * (ns & 1);
      pwait(&bar_zfull[ns & 1], (ns >> 1) & 1, 3);
      BNMF_TRACE(4, ns);
      if (fresh && blk > 0) pwait(bar_accwfree, ((blk / FOLD) - 1) & 1, 5);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t bh = dplus(d_hnt, u * 8 * HNT_LBO);
        issue_side<2 * HNT_LBO>(tmem + TM_ACCW, zb, bh, id32, id16, fresh);
        issue_side<2 * HNT_LBO>(tmem + TM_ACCW + 32, zb + 16, bh, id32, id16, fresh);
        if (u == SW - 1) {
          mma_commit(bar_wdone);
          if (fold_end) mma_commit(bar_accw);
        }
      }
      __syncwarp();
      BNMF_TRACE(5, ns);
      ++ns;
    };

    if (nb > 0) {
      if (do_h) d_h(0, 0);
      else d_w(0, 0);
    }
    for (int bi = 0; bi < nb; ++bi) {
      const bool nxt = bi + 1 < nb;
      if (do_h) {
        for (int j = bi == 0 ? 0 : 2; j < SH; ++j) {
          if (j + 1 < SH) d_h(bi, j + 1);
          else if (nxt) d_h(bi + 1, 0);
          s_h(bi, j);
        }
        if (nxt) {
          d_h(bi + 1, 1);
          s_h(bi + 1, 0);
          d_w(bi, 0);   // U2(bi) needs the side products of H(bi, SH-1): issued above
          s_h(bi + 1, 1);
        } else if (w0_issued != bi) {
          d_w(bi, 0);
        }
      }
      for (int u = 0; u + 1 < SW; ++u) {
        d_w(bi, u + 1);
        s_w(bi, u);
      }
      // last W item: the next Vt tile is the first item of block bi + 1
      if (!nxt) {
        s_w(bi, SW - 1);
      } else if (do_h && SH > 2) {
        d_h(bi + 1, 2);
        s_w(bi, SW - 1);
      } else if (do_h && bi + 2 < nb) {
        d_h(bi + 2, 0);
        s_w(bi, SW - 1);
      } else {
        // next is W(bi + 1, 0), whose U2 waits for the W side products of bi
        s_w(bi, SW - 1);
        d_w(bi + 1, 0);
      }
    }
  } else {
    // ======================= epilogue =======================================
    const int e = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant
    const int g = e >> 2;            // 8-column slice of an item / 4-wide k group
    const int row = 32 * q + lane;   // TMEM lane: n (H items, U) or f - row0 (W items)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    double obj = 0.0;
    int nfold = 0;
    double* mypart = a.part + size_t(blockIdx.x) * 2 * F * K;
    // H-update constants in fp32 (FP64 throughput is low on this part; the
    // update ratio is formed and stored in fp32 anyway)
    float nrm[4], cs2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 4 * g + i;
      nrm[i] = (do_h && k < K) ? float(a.norms[k]) : 0.f;
      cs2[i] = (do_h && den_ones && k < K) ? float(a.csum2[k]) : 1.f;
    }
    const float gam = float(a.sc.gamma);
    const float floor_f = fmaxf(float(a.sc.floor), 1.17549435e-38f);
    // H~_{p-1} rows of blocks u, u+1, u+2 (u = next block to finish its H update)
    float h0[4], h1[4], h2[4];
    int ucur = 0;
    auto load_rows = [&](int blk, float* h) {
      const int n = col0(blk) + row;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        h[i] = (blk < nb && n < N && k < K) ? Hprev[size_t(n) * K + k] : 0.f;
      }
    };
    // H~_{p-1} rows of a block as the TMEM A operand of the H-side Vt tiles
    auto write_hp = [&](const float* h) {
      float hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { hi[i] = tf32_hi(h[i]); lo[i] = h[i] - hi[i]; }
      tmem_st4(lane_base + TM_HP + 4 * g, hi);
      tmem_st4(lane_base + TM_HP + 16 + 4 * g, lo);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_hp);
    };

    // W~_p rows of this CTA into TMEM (A operand of the W-side Vt tiles)
    {
      float hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        const float v = (row < FTr && k < K) ? Wt[size_t(row0 + row) * K + k] : 0.f;
        hi[i] = tf32_hi(v);
        lo[i] = v - hi[i];
      }
      tmem_st4(lane_base + TM_WT + 4 * g, hi);
      tmem_st4(lane_base + TM_WT + 16 + 4 * g, lo);
      tmem_st_wait();
    }
    load_rows(0, h0);
    load_rows(1, h1);
    load_rows(2, h2);
    if (do_h && nb > 0) write_hp(h0);
    else tc_fence_before();

    // U1(blk): AccH of the block read out (and sent to the peer CTA)
    float unum[4], uden[4];
    auto do_u1 = [&](int blk) {
      pwait(bar_acch, blk & 1, 3);
      BNMF_TRACE(48, blk);
      tc_fence_after();
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%16];\n\t"
          "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [%17];\n\t"
          "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [%18];\n\t"
          "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12,%13,%14,%15}, [%19];\n\t"
          "tcgen05.wait::ld.sync.aligned;"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(lane_base + TM_ACCH + 4 * g), "r"(lane_base + TM_ACCH + 16 + 4 * g),
            "r"(lane_base + TM_ACCH + 32 + 4 * g), "r"(lane_base + TM_ACCH + 48 + 4 * g)
          : "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accfree);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        unum[i] = __uint_as_float(r[i]) + __uint_as_float(r[4 + i]);
        uden[i] = den_ones ? 0.f : __uint_as_float(r[8 + i]) + __uint_as_float(r[12 + i]);
      }
      if (CL > 1) {
        const uint32_t peer = rank ^ 1u;
        if (blk > 0) pwait_cl(bar_xempty, (blk - 1) & 1, 4);
        if (threadIdx.x == 64) mbar_expect_tx_u32(smem_u32(bar_xfull), BN * 2 * KP * 4);
        const uint32_t my0 = sb + OFF_XCH + uint32_t(((2 * g) * BN + row) * 16);
        const uint32_t rbar = mapa_shared(smem_u32(bar_xfull), peer);
        st_async_v4(mapa_shared(my0, peer), make_float4(unum[0], unum[1], unum[2], unum[3]), rbar);
        st_async_v4(mapa_shared(my0 + BN * 16, peer), make_float4(uden[0], uden[1], uden[2], uden[3]),
                    rbar);
      }
    };
    // U2(blk): peer partial added (fp32 a + b is commutative, so both CTAs
    // form bitwise-identical totals), H~_p = H~_{p-1} (num/den)^gamma norms
    // published to SMEM (and HBM)
    auto do_u2 = [&](int blk) {
      const int n = col0(blk) + row;
      float hv[4];
      if (do_h) {
        if (CL > 1) {
          const uint32_t peer = rank ^ 1u;
          const uint32_t my0 = sb + OFF_XCH + uint32_t(((2 * g) * BN + row) * 16);
          pwait_cl(bar_xfull, blk & 1, 5);
          BNMF_TRACE(43, blk);
          const float4 pn = lds_f128(my0), pd = lds_f128(my0 + BN * 16);
          unum[0] += pn.x; unum[1] += pn.y; unum[2] += pn.z; unum[3] += pn.w;
          uden[0] += pd.x; uden[1] += pd.y; uden[2] += pd.z; uden[3] += pd.w;
          BNMF_TRACE(49, blk);
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(bar_xempty), peer));
          BNMF_TRACE(50, blk);
        }
        // ratio num / max(den, floor), ^gamma; k >= K has h0 = nrm = 0
        float r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          r[i] = unum[i] * rcp_fast(fmaxf(den_ones ? cs2[i] : uden[i], floor_f));
        if (gam != 1.f) {
#pragma unroll
          for (int i = 0; i < 4; ++i) r[i] = gam == 0.5f ? sqrtf(r[i]) : powf(r[i], gam);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) hv[i] = h0[i] * r[i] * nrm[i];
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) hv[i] = n < N ? h0[i] : 0.f;
      }
      BNMF_TRACE(45, blk);
      if (blk > 0) pwait(bar_wdone, (blk - 1) & 1, 6);   // W MMAs of blk-1 read Hn/HnT
      BNMF_TRACE(46, blk);
      {
        // Hn: this thread's 4 k of row n are one 16 B chunk of the core tile;
        // HnT: 8 conflict-free scalar stores (hi, lo of 4 k)
        float hi[4], lo[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { hi[i] = tf32_hi(hv[i]); lo[i] = hv[i] - hi[i]; }
        sts_f128(sb + OFF_HN + core_off(row, 4 * g), hi[0], hi[1], hi[2], hi[3]);
        sts_f128(sb + OFF_HN + HILO + core_off(row, 4 * g), lo[0], lo[1], lo[2], lo[3]);
        const uint32_t ta = sb + OFF_HNT + hnt_off(4 * g, row);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sts_f32(ta + i * 16, hi[i]);
          sts_f32(ta + 2 * HNT_SBO + i * 16, lo[i]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_hn);
      }
      BNMF_TRACE(47, blk);
      // global traffic only after the SMEM publish (the proxy fence above
      // would otherwise wait for these stores)
      if (do_h && (CL == 1 || (g >> 1) == int(rank)) && n < N) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * g + i < K) Hnew[size_t(n) * K + 4 * g + i] = hv[i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) { h0[i] = h1[i]; h1[i] = h2[i]; }
      load_rows(blk + 3, h2);
      ucur = blk + 1;
    };

    // add the TMEM W sums of the last FOLD blocks into the fp64 slab
    auto fold = [&]() {
      pwait(bar_accw, nfold & 1, 7);
      tc_fence_after();
      const int s = g >> 1, h = g & 1;   // num/den, k half
      float v0[8], v1[8];
      tmem_ld8(lane_base + TM_ACCW + 32 * s + 8 * h, v0);
      tmem_ld8(lane_base + TM_ACCW + 32 * s + 16 + 8 * h, v1);
      if (row < FTr) {
        double* dst = mypart + size_t(s) * F * K + size_t(row0 + row) * K;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int k = 8 * h + kk;
          // one owner thread per slab element: the first fold stores, later
          // folds are fire-and-forget fp64 reductions applied in program order
          if (k < K) {
            const double add = double(v0[kk]) + double(v1[kk]);
            if (nfold == 0) dst[k] = add;
            else atomicAdd(dst + k, add);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accwfree);
      ++nfold;
    };

    const bool rows_full = FTr == 32 * SH;
    float pc[PHI_TERMS];
    if (FBC == FBC_GEN) phi_coeffs(beta, pc);
    int c = 0;   // item counter (Vt / Z buffer c & 1)
    float objb = 0.f;   // objective of the current block (fp32, 32 terms per thread)
    // Vt tile of item c -> registers; the buffer is handed back right away
    auto load_d = [&](int buf, float* y) {
      tmem_ld8(lane_base + TM_D + 32 * buf + 8 * g, y);
    };
    // Z of item c -> TMEM (buffer free: dfull(c) retired the side products of c - 2)
    auto put_z = [&](int buf, const float* zn, const float* zd) {
      store_z(lane_base + TM_Z + 128 * buf + 32 * g, zn, zd);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_zfull[buf]);
      BNMF_TRACE(22, c);
      ++c;
    };
    // ---------------- H item: rows row0 + 32 idx + [0, 32) of block blk ----------------
    auto h_item = [&](int blk, int idx) {
      const int buf = c & 1;
      const int n0 = col0(blk);
      uint32_t ph;
      const int s = stage_of(blk, idx, ph);
      BNMF_TRACE(20, c);
      pwait(&bar_dfull[buf], (c >> 1) & 1, 0);
      BNMF_TRACE(21, c);
      pwait(&bar_full[s], ph, 1);
      tc_fence_after();
      float y[8], zn[8], zd[8];
      load_d(buf, y);
      if (idx == SH - 1 && blk + 1 < nb) {   // Vt tiles of blk are done: stage H~ of blk + 1
        const bool first = blk + 1 == ucur + 1;
        float t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = first ? h1[i] : h2[i];
        write_hp(t);
      }
      const uint32_t xa = sb + OFF_STAGE + s * STAGE_BYTES + (8 * g) * VROWB + row * 4;
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = lds_f32(xa + i * VROWB);
      if (KAPPA) {
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] += kappa;
      }
      zpair8<FBC>(x, y, beta, zn, zd);
      if (!(n0 + BN <= N && (rows_full || 32 * idx + 32 <= FTr))) {
        const bool nok = n0 + row < N;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool ok = nok && (32 * idx + 8 * g + i < FTr);
          zn[i] = ok ? zn[i] : 0.f;
          zd[i] = ok ? zd[i] : 0.f;
        }
      }
      put_z(buf, zn, zd);
    };
    // ---------------- W item: columns n0 + 32 idx + [0, 32) of block blk ----------------
    auto w_item = [&](int blk, int idx, uint32_t xrow) {
      const int buf = c & 1;
      const int n0 = col0(blk);
      BNMF_TRACE(30, c);
      pwait(&bar_dfull[buf], (c >> 1) & 1, 2);
      BNMF_TRACE(31, c);
      tc_fence_after();
      float y[8], x[8], zn[8], zd[8];
      load_d(buf, y);
      if (q < SH) {
        const uint32_t xa = xrow + (32 * idx + 8 * g) * 4;
        const float4 v0 = lds_f128(xa), v1 = lds_f128(xa + 16);
        x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
        x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = 0.f;
      }
#ifndef BNMF_NO_F2
      if (FBC == FBC_15 && n0 + BN <= N && row < FTr) {
        // beta = 1.5, full tile: Z and the objective two lanes per instruction
        if (KAPPA) {
#pragma unroll
          for (int i = 0; i < 8; ++i) y[i] += kappa;
        }
        zpair8<FBC>(x, y, beta, zn, zd);
        const uint64_t two = f2pack(2.f, 2.f);
        uint64_t acc = 0ull;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const uint64_t sx = f2pack(sqrt_fast(x[i]), sqrt_fast(x[i + 1]));
          const uint64_t zdp = f2pack(zd[i], zd[i + 1]);
          const uint64_t dq = f2sub(sx, zdp);
          acc = f2fma(f2mul(dq, dq), f2fma(two, sx, zdp), acc);
        }
        float o0, o1;
        f2unpack(acc, o0, o1);
        objb += o0 + o1;
      } else
#endif
      if (n0 + BN <= N && row < FTr) {
        float o0 = 0.f, o1 = 0.f;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float y0 = KAPPA ? y[i] + kappa : y[i], y1 = KAPPA ? y[i + 1] + kappa : y[i + 1];
          z_and_obj<FBC>(x[i], y0, 0.f, beta, zn[i], zd[i], o0, pc);
          z_and_obj<FBC>(x[i + 1], y1, 0.f, beta, zn[i + 1], zd[i + 1], o1, pc);
        }
        objb += o0 + o1;
      } else {
        const bool fok = row < FTr;
        float o0 = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float yy = KAPPA ? y[i] + kappa : y[i];
          const bool ok = fok && (n0 + 32 * idx + 8 * g + i < N);
          float t = 0.f;
          z_and_obj<FBC>(x[i], yy, 0.f, beta, zn[i], zd[i], t, pc);
          zn[i] = ok ? zn[i] : 0.f;
          zd[i] = ok ? zd[i] : 0.f;
          o0 += ok ? t : 0.f;
        }
        objb += o0;
      }
      put_z(buf, zn, zd);
    };

    for (int bi = 0; bi < nb; ++bi) {
      if (do_h) {
        for (int j = bi == 0 ? 0 : 2; j < SH; ++j) h_item(bi, j);
      } else {
        for (int j = 0; j < SH; ++j) {
          uint32_t ph;
          const int s = stage_of(bi, j, ph);
          mbar_wait(&bar_full[s], ph);
        }
      }
      {
        if (do_h) {
          if (bi + 1 < nb) h_item(bi + 1, 0);
          BNMF_PROF_T0(tu1);
          BNMF_TRACE(40, c);
          do_u1(bi);
          BNMF_TRACE(41, c);
          BNMF_PROF_ADD(8, tu1);
          if (bi + 1 < nb) h_item(bi + 1, 1);
        }
        BNMF_PROF_T0(tu2);
        BNMF_TRACE(42, c);
        do_u2(bi);
        BNMF_TRACE(44, c);
        BNMF_PROF_ADD(9, tu2);
      }
      uint32_t phq;
      const uint32_t xrow = sb + OFF_STAGE + stage_of(bi, q < SH ? q : 0, phq) * STAGE_BYTES + lane * VROWB;
      objb = 0.f;
      for (int u = 0; u < SW; ++u) w_item(bi, u, xrow);
      obj += FBC == FBC_15 ? double(objb) * (2.0 / 3.0) : double(objb);
      if (lane == 0)
        for (int j = 0; j < SH; ++j) {
          uint32_t ph;
          mbar_arrive(&bar_empty[stage_of(bi, j, ph)]);
        }
      if ((bi % FOLD) == FOLD - 1 || bi == nb - 1) {
        BNMF_PROF_T0(tf);
        BNMF_TRACE(50, c);
        fold();
        BNMF_TRACE(51, c);
        BNMF_PROF_ADD(10, tf);
      }
    }
    if (nfold == 0) {   // CTA without blocks: zero its slab rows
      const int s = g >> 1, h = g & 1;
      if (row < FTr)
        for (int kk = 0; kk < 8; ++kk) {
          const int k = 8 * h + kk;
          if (k < K) mypart[size_t(s) * F * K + size_t(row0 + row) * K + k] = 0.0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
    if (lane == 0) s_red[e] = obj;
  }
#ifdef BNMF_TC_PROF
  if (trace_buf) trace_buf[4095] = trace_n;
  if (rec) pcs[pbase + 11] = clock64() - t_start;
  __syncthreads();
  if (prof)
    for (int i = threadIdx.x; i < 48; i += blockDim.x) prof[i] = (long long)pcs[i];
#endif
#undef BNMF_PROF_T0
#undef BNMF_PROF_ADD
#undef BNMF_TRACE
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < NEPI; ++i) t += s_red[i];
    a.opart[blockIdx.x] = t;
  }
  if (CL > 1) cluster_sync_all();   // no CTA leaves while its peer may still signal it
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace ftc
}  // namespace bnmf
