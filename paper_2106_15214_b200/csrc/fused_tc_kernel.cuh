// tcgen05 implementation of the fused single-read pass (fp32 carried as
// 3xTF32, F <= 256 rows, rank K <= 16).  Same contract as fused_pass_simt.
//
// One persistent CTA per SM walks 128-column blocks of V.  Warp roles:
//   warp 0      TMA producer: V tiles into a 16 KB smem ring, in consumption
//               order (per block: F/32 tiles [32 f x 128 n] for the H phase,
//               then 4*FT tiles [128 f x 32 n], 128B-swizzled, for the W
//               phase -- that second read is served by L2)
//   warp 1      MMA issuer (warp-uniform loop, elected lane issues) + TMEM owner
//   warps 2..17 epilogue: TMEM -> registers, the beta-dependent terms, the
//               hi/lo TF32 split written back to TMEM as MMA A operands, the
//               H update, the objective, fp64 folding of the W sums
// Per block (columns n0 .. n0+127):
//   H phase, f sub-tile j (32 rows):
//     D    [n x f] = Hp (128x16) * Wa[j]^T            6 MMAs  M128 N32 (3xTF32)
//     ZT   [n x f] = Zn, Zd of (V, D + kappa)         epilogue -> TMEM
//     AccH [n x k] += ZT * chi[j]                     24 MMAs M128 N16 (A in TMEM)
//   H update: H~_p = Hp * (AccHn / max(AccHd, floor))^gamma * norms -> smem, HBM
//   W phase, f tile t (128 rows) x n sub-tile u (32 cols):
//     D    [f x n] = W~_p[t] * H~_p[u]^T              6 MMAs  M128 N32
//     Z    [f x n] = Zn, Zd of (V, D + kappa); objective
//     AccW [t]    += Z * H~_p[u]                      24 MMAs M128 N16 (A in TMEM)
//   AccW stays in TMEM for FOLD blocks, then is added into the CTA's fp64
//   partial slab (fixed order => deterministic).
// All smem MMA operands are K-major "core-tiled" (8 rows x 16 B core matrices).
#pragma once

#include <cuda.h>

#include "fused_common.cuh"
#include "tc_primitives.cuh"

namespace bnmf {
namespace ftc {

using namespace bnmf::tc;

constexpr int BN = 128;            // columns per block
constexpr int KP = 16;             // padded rank
constexpr int NEPI = 16;           // epilogue warps (4 per TMEM lane quadrant)
constexpr int NTHREADS = 32 * (2 + NEPI);
constexpr int FOLD = 8;            // blocks accumulated in TMEM before the fp64 fold
constexpr uint32_t STAGE_BYTES = 32 * 128 * 4;

// TMEM columns
constexpr uint32_t TM_ACCW = 0;    // tile t: num at 32t, den at 32t+16
constexpr uint32_t TM_ACCH = 64;   // num 64..79, den 80..95
constexpr uint32_t TM_D = 96;      // D[i] at 96 + 32 i, i < 3 (triple buffered)
constexpr uint32_t TM_Z = 192;     // Z[b] at 192 + 128 b: num_hi, num_lo, den_hi, den_lo (32 each)
constexpr uint32_t TM_WT = 448;    // W~_p as TMEM A operand: tile t hi at 448 + 32t, lo at +16

// beta class of the fused TC epilogue (adds the beta = 1.5 fast form)
enum { FBC_GEN = 0, FBC_0 = 1, FBC_1 = 2, FBC_2 = 3, FBC_15 = 4 };

struct TcLayout {
  int FP, FT, SH, SW, nstage;
  uint32_t off_stage, off_wa, off_wt, off_c1, off_c2, off_hp, off_hn, off_hnt, off_bar;
  uint32_t bytes;
};

__host__ __device__ inline TcLayout tc_layout(int F, int nstage) {
  TcLayout L;
  L.FT = (F + 127) / 128;
  L.FP = L.FT * 128;
  L.SH = (F + 31) / 32;
  L.SW = 4 * L.FT;
  L.nstage = nstage;
  uint32_t o = 0;
  L.off_stage = o; o += nstage * STAGE_BYTES;
  const uint32_t wbytes = uint32_t(L.FP) * KP * 4;   // one hi or lo copy of an F x 16 operand
  L.off_wa = o; o += 2 * wbytes;
  L.off_wt = 0;   // W~_p lives in TMEM (TM_WT)
  L.off_c1 = o; o += 2 * wbytes;
  L.off_c2 = o; o += 2 * wbytes;
  L.off_hp = o; o += 2 * BN * KP * 4;
  L.off_hn = o; o += 2 * BN * KP * 4;
  L.off_hnt = o; o += 2 * BN * KP * 4;
  L.off_bar = o; o += 256;
  L.bytes = o;
  return L;
}

// element (k, c) of a K-major [16 rows x C] tile whose K dimension is C:
// 8-row groups at SBO = C*32 bytes, 4-wide chunks of c at 128 B
__host__ __device__ __forceinline__ uint32_t coreT_off(int k, int c, int C) {
  return uint32_t((k >> 3) * (C * 32) + (c >> 2) * 128 + (k & 7) * 16 + (c & 3) * 4);
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
    // d_{3/2}(x|y) = (2/3) (sqrt x - sqrt y)^2 (2 sqrt x + sqrt y); zd = sqrt y
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

// smem descriptor arithmetic: the start-address field is addr >> 4 in the low
// 14 bits, so desc(addr + off) == desc(addr) + (off >> 4) for smem < 256 KB.
__device__ __forceinline__ uint64_t dplus(uint64_t d, uint32_t off) { return d + (off >> 4); }

// D (+)= A * B^T over K = 16 in 3xTF32: (hi,hi) + (hi,lo) + (lo,hi), 2 k-steps
// each; A and B K-major core-tiled (LBO 128, SBO 512).
__device__ __forceinline__ void issue_big(uint32_t dcol, uint64_t a_hi, uint64_t a_lo,
                                          uint64_t b_hi, uint64_t b_lo, uint32_t idesc,
                                          int dbg = 0) {
  if (dbg == 2) return;
  mma_ss(dcol, a_hi, b_hi, idesc, 0u);
  mma_ss(dcol, dplus(a_hi, 256), dplus(b_hi, 256), idesc, 1u);
  mma_ss(dcol, a_hi, b_lo, idesc, 1u);
  mma_ss(dcol, dplus(a_hi, 256), dplus(b_lo, 256), idesc, 1u);
  mma_ss(dcol, a_lo, b_hi, idesc, 1u);
  mma_ss(dcol, dplus(a_lo, 256), dplus(b_hi, 256), idesc, 1u);
}

// Same with A (M x 16, hi/lo) in TMEM columns a_hi / a_lo (8 columns per k-step).
__device__ __forceinline__ void issue_big_ts(uint32_t dcol, uint32_t a_hi, uint32_t a_lo,
                                             uint64_t b_hi, uint64_t b_lo, uint32_t idesc,
                                             int dbg = 0) {
  if (dbg == 2) return;
  mma_ts(dcol, a_hi, b_hi, idesc, 0u);
  mma_ts(dcol, a_hi + 8, dplus(b_hi, 256), idesc, 1u);
  mma_ts(dcol, a_hi, b_lo, idesc, 1u);
  mma_ts(dcol, a_hi + 8, dplus(b_lo, 256), idesc, 1u);
  mma_ts(dcol, a_lo, b_hi, idesc, 1u);
  mma_ts(dcol, a_lo + 8, dplus(b_hi, 256), idesc, 1u);
}

// D (+)= Z * B over a 32-wide K slab: Z (hi/lo) in TMEM columns, B K-major
// [16 x K]; 3xTF32, 4 k-steps each.
__device__ __forceinline__ void issue_side(uint32_t dcol, uint32_t z_hi, uint32_t z_lo,
                                           uint64_t b_hi, uint64_t b_lo, uint32_t idesc,
                                           bool fresh, int dbg = 0) {
  if (dbg == 2) return;
#pragma unroll
  for (int s = 0; s < 4; ++s)
    mma_ts(dcol, z_hi + 8 * s, dplus(b_hi, 256 * s), idesc, (fresh && s == 0) ? 0u : 1u);
#pragma unroll
  for (int s = 0; s < 4; ++s) mma_ts(dcol, z_hi + 8 * s, dplus(b_lo, 256 * s), idesc, 1u);
#pragma unroll
  for (int s = 0; s < 4; ++s) mma_ts(dcol, z_lo + 8 * s, dplus(b_hi, 256 * s), idesc, 1u);
}

// store 8 Z values (hi/lo split) at TMEM columns col (hi) and col + 32 (lo)
__device__ __forceinline__ void store_z8(uint32_t col, const float* z) {
  float hi[8], lo[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { hi[i] = tf32_trunc(z[i]); lo[i] = z[i] - hi[i]; }
  tmem_st8(col, hi);
  tmem_st8(col + 32, lo);
}

template <int FBC, bool KAPPA>
__global__ void __launch_bounds__(NTHREADS, 1)
fused_pass_tc(FusedArgs a, const __grid_constant__ CUtensorMap mapH,
              const __grid_constant__ CUtensorMap mapW, int nstage, const RunState* st, int slot,
              int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // 1024-align the working base (128B-swizzled TMA tiles need it)
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int F = a.F, N = a.N, K = a.K;
  const TcLayout L = tc_layout(F, nstage);
  const uint32_t s_base = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* bar_full = bars;                 // [nstage]
  uint64_t* bar_empty = bars + 8;            // [nstage]
  uint64_t* bar_dfull = bars + 16;           // [3]
  uint64_t* bar_zfull = bars + 19;           // [2]
  uint64_t* bar_zempty = bars + 21;          // [2]
  uint64_t* bar_hp = bars + 23;
  uint64_t* bar_hn = bars + 24;
  uint64_t* bar_acch = bars + 25;
  uint64_t* bar_accw = bars + 26;
  uint64_t* bar_accw_free = bars + 27;
  uint64_t* bar_wdone = bars + 28;           // all W-side MMAs of a block retired
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 29);
  __shared__ double s_red[NEPI];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int par = iter_parity(st, slot, p_override);
  const float* Hprev = a.do_h ? a.Hbuf[par ^ 1] : a.Hbuf[par];
  float* Hnew = a.Hout[par];
  const float* Wt = a.Wt2[par];
  const float* Wa = a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn;
  const int do_h = a.do_h;
  const int den_ones = a.den_ones;
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  const int nblocks = (N + BN - 1) / BN;
  const uint32_t wb = uint32_t(L.FP) * KP * 4;   // hi -> lo offset of F x 16 operands
  const uint32_t hb = BN * KP * 4;               // hi -> lo offset of 128 x 16 operands

  // ---- setup: barriers, TMEM, constant operands ---------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], NEPI);
    }
    for (int b = 0; b < 3; ++b) mbar_init(&bar_dfull[b], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_zfull[b], NEPI);
      mbar_init(&bar_zempty[b], 1);
    }
    mbar_init(bar_hp, NEPI);
    mbar_init(bar_hn, NEPI);
    mbar_init(bar_acch, 1);
    mbar_init(bar_accw, 1);
    mbar_init(bar_accw_free, NEPI);
    mbar_init(bar_wdone, 1);
    mbar_fence_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapH);
    tma_prefetch(&mapW);
  }
  if (warp == 1) tmem_alloc<512>(s_tmem);
  if (warp >= 2) {
    const int te = threadIdx.x - 64;
    for (int i = te; i < L.FP * KP; i += NEPI * 32) {
      const int f = i / KP, k = i - f * KP;
      const bool ok = f < F && k < K;
      const size_t gi = size_t(f) * K + k;
      const uint32_t o = core_off(f, k), ot = coreT_off(k, f, L.FP);
      float v, hi;
      v = ok ? Wa[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(s_base + L.off_wa + o, hi); sts_f32(s_base + L.off_wa + wb + o, v - hi);
      v = ok ? a.C1[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(s_base + L.off_c1 + ot, hi); sts_f32(s_base + L.off_c1 + wb + ot, v - hi);
      v = ok ? a.C2[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(s_base + L.off_c2 + ot, hi); sts_f32(s_base + L.off_c2 + wb + ot, v - hi);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  // W~_p (A operand of the W-phase Vt MMAs) into TMEM: warps with g < FT write
  // tile t = g, lane f, 16 hi + 16 lo columns.
  if (warp >= 2) {
    const int e = warp - 2, q = warp & 3, g = e >> 2;
    if (g < L.FT) {
      const int f = 128 * g + 32 * q + lane;
      float hi[16], lo[16];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const float v = (f < F && k < K) ? Wt[size_t(f) * K + k] : 0.f;
        hi[k] = tf32_hi(v);
        lo[k] = v - hi[k];
      }
      const uint32_t ta = tmem + (uint32_t(32 * q) << 16) + TM_WT + 32 * g;
      tmem_st16(ta, hi);
      tmem_st16(ta + 16, lo);
      tmem_st_wait();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ======================= TMA producer ===================================
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int n0 = b * BN;
        if (do_h) {
          for (int j = 0; j < L.SH; ++j) {
            mbar_wait(&bar_empty[stage], ph ^ 1);
            mbar_expect_tx(&bar_full[stage], STAGE_BYTES);
            tma_load_2d(smem + L.off_stage + stage * STAGE_BYTES, &mapH, &bar_full[stage], n0,
                        32 * j);
            if (++stage == nstage) { stage = 0; ph ^= 1; }
          }
        }
        for (int w = 0; w < L.SW; ++w) {
          mbar_wait(&bar_empty[stage], ph ^ 1);
          mbar_expect_tx(&bar_full[stage], STAGE_BYTES);
          tma_load_2d(smem + L.off_stage + stage * STAGE_BYTES, &mapW, &bar_full[stage],
                      n0 + 32 * (w & 3), 128 * (w >> 2));
          if (++stage == nstage) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (warp-uniform) ======================
    // Sub-tiles are numbered c = bi * SB + s (s < SH: H phase, else W phase).
    // D(c) is issued up to two sub-tiles ahead of the side MMAs of c, into
    // one of three D buffers; the side MMAs of c wait for Z(c) from the
    // epilogue and release the Z buffer through zempty.
    const uint32_t id_big = idesc_tf32(128, 32, 0, 0);
    const uint32_t id_side = idesc_tf32(128, 16, 0, 0);
    const uint64_t d_wa = sdesc(s_base + L.off_wa, 128, 512);
    const uint64_t d_hp = sdesc(s_base + L.off_hp, 128, 512);
    const uint64_t d_hn = sdesc(s_base + L.off_hn, 128, 512);
    const uint64_t d_c1 = sdesc(s_base + L.off_c1, 128, uint32_t(L.FP) * 32);
    const uint64_t d_c2 = sdesc(s_base + L.off_c2, 128, uint32_t(L.FP) * 32);
    const uint64_t d_hnt = sdesc(s_base + L.off_hnt, 128, BN * 32);
    const int SHh = do_h ? L.SH : 0;
    const int SB = SHh + L.SW;
    const int nb_cta = blockIdx.x < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int total = a.debug >= 3 ? 0 : nb_cta * SB;
    int nd = 0;
    for (int cs = 0; cs < total; ++cs) {
      // ---- issue D's ahead (three buffers) ----
      while (nd < total && nd <= cs + 2) {
        const int bi_d = nd / SB, s_d = nd - bi_d * SB;
        const uint32_t dcol = tmem + TM_D + 32 * (nd % 3);
        if (s_d < SHh) {
          if (s_d == 0) {
            mbar_wait(bar_hp, bi_d & 1);
            tc_fence_after();
          }
          if (elect_one())
            issue_big(dcol, d_hp, dplus(d_hp, hb), dplus(d_wa, s_d * 2048),
                      dplus(d_wa, s_d * 2048 + wb), id_big, a.debug);
        } else {
          const int w = s_d - SHh, t = w >> 2, u = w & 3;
          if (w == 0) {
            // H~_p of this block needs every side MMA issued before it (the
            // epilogue's H update waits for them): no run-ahead past here
            if (cs < bi_d * SB + SHh) break;
            mbar_wait(bar_hn, bi_d & 1);
            tc_fence_after();
          }
          if (elect_one())
            issue_big_ts(dcol, tmem + TM_WT + 32 * t, tmem + TM_WT + 32 * t + 16,
                         dplus(d_hn, u * 2048), dplus(d_hn, u * 2048 + hb), id_big, a.debug);
        }
        if (elect_one()) mma_commit(&bar_dfull[nd % 3]);
        __syncwarp();
        ++nd;
      }
      // ---- side MMAs of sub-tile cs ----
      mbar_wait(&bar_zfull[cs & 1], (cs >> 1) & 1);
      tc_fence_after();
      const int bi = cs / SB, s_c = cs - bi * SB;
      const uint32_t zb = tmem + TM_Z + 128 * (cs & 1);
      if (s_c < SHh) {
        const uint64_t b1 = dplus(d_c1, s_c * 1024);
        const uint64_t b2 = dplus(d_c2, s_c * 1024);
        if (elect_one()) {
          issue_side(tmem + TM_ACCH, zb, zb + 32, b1, dplus(b1, wb), id_side, s_c == 0, a.debug);
          if (!den_ones)
            issue_side(tmem + TM_ACCH + 16, zb + 64, zb + 96, b2, dplus(b2, wb), id_side, s_c == 0,
                       a.debug);
          mma_commit(&bar_zempty[cs & 1]);
          if (s_c == SHh - 1) mma_commit(bar_acch);
        }
        __syncwarp();
      } else {
        const int w = s_c - SHh, t = w >> 2, u = w & 3;
        const bool fresh = (bi % FOLD) == 0 && u == 0;
        if (w == 0 && (bi % FOLD) == 0 && bi > 0) {
          mbar_wait(bar_accw_free, ((bi / FOLD) - 1) & 1);
          tc_fence_after();
        }
        const uint64_t bh = dplus(d_hnt, u * 1024);
        const uint64_t bl = dplus(bh, hb);
        const bool last_w = w == L.SW - 1;
        const bool fold_end = (bi % FOLD) == FOLD - 1 || bi == nb_cta - 1;
        if (elect_one()) {
          issue_side(tmem + TM_ACCW + 32 * t, zb, zb + 32, bh, bl, id_side, fresh, a.debug);
          issue_side(tmem + TM_ACCW + 32 * t + 16, zb + 64, zb + 96, bh, bl, id_side, fresh, a.debug);
          mma_commit(&bar_zempty[cs & 1]);
          if (last_w && fold_end) mma_commit(bar_accw);
          if (last_w) mma_commit(bar_wdone);
        }
        __syncwarp();
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue =======================================
    const int e = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant
    const int g = e >> 2;            // 8-column slice of a 32-wide sub-tile
    const int row = 32 * q + lane;   // TMEM lane (n in the H phase, f_local in the W phase)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    double obj = 0.0;
    float hprev[4];
    int stage = 0;
    uint32_t ph = 0;
    uint32_t c = 0;
    int bi = 0;
    int nfold = 0;
    double* mypart = a.part + size_t(blockIdx.x) * 2 * F * K;

    // H~_{p-1} rows of a block (this thread: n = row, k in [4g, 4g+4))
    auto load_hprev = [&](int n0) {
      const int n = n0 + row;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        hprev[i] = (n < N && k < K) ? Hprev[size_t(n) * K + k] : 0.f;
        const float hi = tf32_hi(hprev[i]);
        const uint32_t o = s_base + L.off_hp + core_off(row, k);
        sts_f32(o, hi);
        sts_f32(o + hb, hprev[i] - hi);
      }
    };
    auto store_hnew = [&](int n0, const float* hv) {
      const int n = n0 + row;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
        const float v = (n < N && k < K) ? hv[i] : 0.f;
        if (do_h && n < N && k < K) Hnew[size_t(n) * K + k] = v;
        const float hi = tf32_hi(v);
        const uint32_t o = s_base + L.off_hn + core_off(row, k);
        const uint32_t ot = s_base + L.off_hnt + coreT_off(k, row, BN);
        sts_f32(o, hi);
        sts_f32(o + hb, v - hi);
        sts_f32(ot, hi);
        sts_f32(ot + hb, v - hi);
      }
    };
    // add the TMEM W sums of the last FOLD blocks into the fp64 slab
    auto fold = [&]() {
      if (a.debug >= 3) { ++nfold; return; }
      mbar_wait(bar_accw, nfold & 1);
      tc_fence_after();
      if (g < 2 * L.FT) {
        const int t = g >> 1, s = g & 1;   // tile, num/den
        float v[16];
        tmem_ld16(lane_base + TM_ACCW + 32 * t + 16 * s, v);
        const int f = 128 * t + row;
        if (f < F) {
          double* dst = mypart + size_t(s) * F * K + size_t(f) * K;
#pragma unroll
          for (int k = 0; k < KP; ++k)
            if (k < K) dst[k] = (nfold == 0 ? 0.0 : dst[k]) + double(v[k]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accw_free);
      ++nfold;
    };

    int b = blockIdx.x;
    if (b < nblocks) {
      load_hprev(b * BN);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_hp);
    }
    for (; b < nblocks; b += gridDim.x, ++bi) {
      const int n0 = b * BN;
      const bool ncols_full = n0 + BN <= N;
      if (do_h) {
        // ---------------- H phase ----------------
        for (int j = 0; j < L.SH; ++j, ++c) {
          const uint32_t buf = c & 1, dbuf = c % 3;
          const bool nomma = a.debug >= 3;
          if (!nomma) mbar_wait(&bar_dfull[dbuf], (c / 3) & 1);
          mbar_wait(&bar_full[stage], ph);
          tc_fence_after();
          float y[8], x[8], zn[8], zd[8];
          if (!nomma) tmem_ld8(lane_base + TM_D + 32 * dbuf + 8 * g, y);
          else for (int i = 0; i < 8; ++i) y[i] = 1.f;
          const uint32_t xa = s_base + L.off_stage + stage * STAGE_BYTES + (8 * g * 128 + row) * 4;
          if (a.debug == 1 || a.debug == 4) {
#pragma unroll
            for (int i = 0; i < 8; ++i) { zn[i] = y[i]; zd[i] = y[i]; }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = lds_f32(xa + i * 512);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              zpair<FBC>(x[i], KAPPA ? y[i] + kappa : y[i], beta, zn[i], zd[i]);
          }
          if (!(ncols_full && 32 * j + 32 <= F)) {
            const bool nok = n0 + row < N;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const bool ok = nok && (32 * j + 8 * g + i < F);
              zn[i] = ok ? zn[i] : 0.f;
              zd[i] = ok ? zd[i] : 0.f;
            }
          }
          const uint32_t zb = lane_base + TM_Z + 128 * buf + 8 * g;
          if (c >= 2 && !nomma) {   // side MMAs of c-2 released this Z buffer
            mbar_wait(&bar_zempty[buf], ((c - 2) >> 1) & 1);
            tc_fence_after();
          }
          if (!nomma) {
            store_z8(zb, zn);
            if (!den_ones) store_z8(zb + 64, zd);
          } else if (zn[0] == 12345.f && zd[1] == 1.f) {
            obj += 1.0;
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&bar_zfull[buf]);
            mbar_arrive(&bar_empty[stage]);
          }
          if (++stage == nstage) { stage = 0; ph ^= 1; }
        }
        // ---------------- H update ----------------
        float nv[4], dv[4], hv[4];
        if (a.debug < 3) {
          mbar_wait(bar_acch, bi & 1);
          tc_fence_after();
          tmem_ld4(lane_base + TM_ACCH + 4 * g, nv);
          if (!den_ones) tmem_ld4(lane_base + TM_ACCH + 16 + 4 * g, dv);
        } else {
          for (int i = 0; i < 4; ++i) { nv[i] = 1.f; dv[i] = 1.f; }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = 4 * g + i;
          float v = 0.f;
          if (k < K) {
            const double den = den_ones ? a.csum2[k] : double(dv[i]);
            const double r = double(nv[i]) / fmax(den, a.sc.floor);
            v = float(double(hprev[i]) * apply_exponent<double>(r, a.sc.gamma) * a.norms[k]);
          }
          hv[i] = v;
        }
        tc_fence_before();
        if (bi > 0 && a.debug < 3) mbar_wait(bar_wdone, (bi - 1) & 1);   // W MMAs of bi-1 read H~ smem
        store_hnew(n0, hv);
      } else {
        if (bi > 0 && a.debug < 3) mbar_wait(bar_wdone, (bi - 1) & 1);
        store_hnew(n0, hprev);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_hn);
      // prefetch the next block's H~_{p-1} rows (D1 MMAs of this block are done)
      if (b + (int)gridDim.x < nblocks) {
        load_hprev((b + gridDim.x) * BN);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_hp);
      }
      // ---------------- W phase ----------------
      for (int w = 0; w < L.SW; ++w, ++c) {
        const uint32_t buf = c & 1, dbuf = c % 3;
        const int t = w >> 2, u = w & 3;
        const bool nomma = a.debug >= 3;
        if (!nomma) mbar_wait(&bar_dfull[dbuf], (c / 3) & 1);
        mbar_wait(&bar_full[stage], ph);
        tc_fence_after();
        float y[8], x[8], zn[8], zd[8], dd[8];
        if (!nomma) tmem_ld8(lane_base + TM_D + 32 * dbuf + 8 * g, y);
        else for (int i = 0; i < 8; ++i) y[i] = 1.f;
        const uint32_t ta = s_base + L.off_stage + stage * STAGE_BYTES + row * 128;
        if (a.debug == 1 || a.debug == 4) {
#pragma unroll
          for (int i = 0; i < 8; ++i) { zn[i] = y[i]; zd[i] = y[i]; dd[i] = 0.f; }
        } else {
#pragma unroll
          for (int cq = 0; cq < 2; ++cq) {
            const float4 v4 = lds_f128(ta + (((2 * g + cq) ^ (row & 7)) << 4));
            x[4 * cq + 0] = v4.x; x[4 * cq + 1] = v4.y; x[4 * cq + 2] = v4.z; x[4 * cq + 3] = v4.w;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float yy = KAPPA ? y[i] + kappa : y[i];
            zpair<FBC>(x[i], yy, beta, zn[i], zd[i]);
            dd[i] = dterm<FBC>(x[i], yy, zd[i], beta);
          }
        }
        if (!(ncols_full && 128 * t + 128 <= F)) {
          const int f = 128 * t + row;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool ok = f < F && (n0 + 32 * u + 8 * g + i < N);
            zn[i] = ok ? zn[i] : 0.f;
            zd[i] = ok ? zd[i] : 0.f;
            dd[i] = ok ? dd[i] : 0.f;
          }
        }
        obj += double((dd[0] + dd[1]) + (dd[2] + dd[3]) + ((dd[4] + dd[5]) + (dd[6] + dd[7])));
        const uint32_t zb = lane_base + TM_Z + 128 * buf + 8 * g;
        if (c >= 2 && !nomma) {
          mbar_wait(&bar_zempty[buf], ((c - 2) >> 1) & 1);
          tc_fence_after();
        }
        if (!nomma) {
          store_z8(zb, zn);
          store_z8(zb + 64, zd);
        } else if (zn[0] == 12345.f && zd[1] == 1.f) {
          obj += 1.0;
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bar_zfull[buf]);
          mbar_arrive(&bar_empty[stage]);
        }
        if (++stage == nstage) { stage = 0; ph ^= 1; }
      }
      if ((bi % FOLD) == FOLD - 1 || b + (int)gridDim.x >= nblocks) fold();
    }
    if (nfold == 0 && g < 2 * L.FT) {   // CTA without blocks: zero slab rows
      const int t = g >> 1, s = g & 1;
      const int f = 128 * t + row;
      if (f < F)
        for (int k = 0; k < K; ++k) mypart[size_t(s) * F * K + size_t(f) * K + k] = 0.0;
    }
    for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
    if (lane == 0) s_red[e] = obj;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < NEPI; ++i) t += s_red[i];
    a.opart[blockIdx.x] = t;
  }
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace ftc
}  // namespace bnmf
