// tcgen05 implementation of the fused single-read pass (fp32 in 3xTF32,
// F <= 256 rows, rank K <= 16).  Same contract as fused_pass_simt.
//
// One persistent CTA per SM walks 128-column blocks of V.  Warp roles:
//   warp 0      TMA producer: V tiles into a 16 KB smem ring, in the order
//               the epilogue consumes them (per block: F/32 tiles [32 f x 128 n]
//               for the H phase, then 4*FT tiles [128 f x 32 n], 128B
//               swizzled, for the W phase -- the second read hits L2)
//   warp 1      MMA issuer (one thread) + TMEM owner
//   warps 2..9  epilogue: TMEM -> registers, the beta-dependent terms, the
//               hi/lo TF32 split written back to TMEM as MMA A operands,
//               the H update, the objective, fp64 folding of the W sums
// Per block (n0 .. n0+127):
//   H phase, f sub-tile j (32 rows):
//     D   [n x f]  = Hp (128x16) * Wa[j]^T           6 MMAs  M128 N32  (3xTF32)
//     ZT  [n x f]  = Zn, Zd of (V, D + kappa)        epilogue -> TMEM
//     AccH[n x k] += ZT * chi[j]                     24 MMAs M128 N16  (A in TMEM)
//   H update: H~_p = Hp * (AccHn / max(AccHd, floor))^gamma * norms -> smem, HBM
//   W phase, f tile t (128 rows) x n sub-tile u (32 cols):
//     D   [f x n]  = W~_p[t] * H~_p[u]^T             6 MMAs  M128 N32
//     Z   [f x n]  = Zn, Zd of (V, D + kappa); objective
//     AccW[t]     += Z * H~_p[u]                     24 MMAs M128 N16  (A in TMEM)
//   AccW is folded into fp64 registers once per block.
// All smem operands are K-major "core-tiled" (8 rows x 16 B core matrices).
#pragma once

#include <cuda.h>

#include "fused_common.cuh"
#include "tc_primitives.cuh"

namespace bnmf {
namespace ftc {

using namespace bnmf::tc;

constexpr int BN = 128;            // columns per block
constexpr int KP = 16;             // padded rank
constexpr int NEPI = 8;            // epilogue warps
constexpr int NTHREADS = 32 * (2 + NEPI);
constexpr uint32_t STAGE_BYTES = 32 * 128 * 4;

// TMEM columns
constexpr uint32_t TM_ACCW = 0;    // tile t: num at 32t, den at 32t+16
constexpr uint32_t TM_ACCH = 64;   // num 64..79, den 80..95
constexpr uint32_t TM_D = 96;      // D[buf] at 96 + 32 buf
constexpr uint32_t TM_Z = 160;     // Z[buf] at 160 + 128 buf: num_hi, num_lo, den_hi, den_lo (32 each)

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
  L.off_wt = o; o += 2 * wbytes;
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
// (rows k, 8-row groups at SBO = C*32 bytes, 4-wide chunks of c at 128 B)
__device__ __forceinline__ uint32_t coreT_off(int k, int c, int C) {
  return uint32_t((k >> 3) * (C * 32) + (c >> 2) * 128 + (k & 7) * 16 + (c & 3) * 4);
}

template <int FBC>
__device__ __forceinline__ void zpair(float x, float y, float beta, float& zn, float& zd) {
  if (FBC == FBC_15) {
    float r = rsqrtf(y);
    zn = x * r;
    zd = y * r;
  } else if (FBC == FBC_2) {
    zn = x; zd = y;
  } else if (FBC == FBC_1) {
    zn = __fdividef(x, y); zd = 1.f;
  } else if (FBC == FBC_0) {
    float r = __frcp_rn(y);
    zn = x * r * r; zd = r;
  } else {
    bases32<BC_GEN>(x, y, beta, zn, zd);
  }
}

template <int FBC>
__device__ __forceinline__ float dterm(float x, float y, float zd, float beta) {
  if (FBC == FBC_15) {
    // d_{3/2}(x|y) = (2/3) (sqrt x - sqrt y)^2 (2 sqrt x + sqrt y); zd = sqrt y
    float sx = x > 0.f ? x * rsqrtf(x) : 0.f;
    float dq = sx - zd;
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

__device__ __forceinline__ void split_store(char* base_hi, char* base_lo, uint32_t off, float v) {
  float hi = to_tf32(v);
  *reinterpret_cast<float*>(base_hi + off) = hi;
  *reinterpret_cast<float*>(base_lo + off) = to_tf32(v - hi);
}

template <int FBC>
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
  char* s_stage = reinterpret_cast<char*>(smem + L.off_stage);
  char* s_wa[2] = {reinterpret_cast<char*>(smem + L.off_wa),
                   reinterpret_cast<char*>(smem + L.off_wa + L.FP * KP * 4)};
  char* s_wt[2] = {reinterpret_cast<char*>(smem + L.off_wt),
                   reinterpret_cast<char*>(smem + L.off_wt + L.FP * KP * 4)};
  char* s_c1[2] = {reinterpret_cast<char*>(smem + L.off_c1),
                   reinterpret_cast<char*>(smem + L.off_c1 + L.FP * KP * 4)};
  char* s_c2[2] = {reinterpret_cast<char*>(smem + L.off_c2),
                   reinterpret_cast<char*>(smem + L.off_c2 + L.FP * KP * 4)};
  char* s_hp[2] = {reinterpret_cast<char*>(smem + L.off_hp),
                   reinterpret_cast<char*>(smem + L.off_hp + BN * KP * 4)};
  char* s_hn[2] = {reinterpret_cast<char*>(smem + L.off_hn),
                   reinterpret_cast<char*>(smem + L.off_hn + BN * KP * 4)};
  char* s_hnt[2] = {reinterpret_cast<char*>(smem + L.off_hnt),
                    reinterpret_cast<char*>(smem + L.off_hnt + BN * KP * 4)};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* bar_full = bars;                 // [nstage]
  uint64_t* bar_empty = bars + 8;            // [nstage]
  uint64_t* bar_dfull = bars + 16;           // [2]
  uint64_t* bar_zfull = bars + 18;           // [2]
  uint64_t* bar_hp = bars + 20;
  uint64_t* bar_hn = bars + 21;
  uint64_t* bar_acch = bars + 22;
  uint64_t* bar_accw = bars + 23;
  uint64_t* bar_accw_free = bars + 24;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 26);
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

  // ---- setup: barriers, TMEM, constant operands ---------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) {
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
    mbar_init(bar_accw, 1);
    mbar_init(bar_accw_free, NEPI);
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
      const uint32_t o = core_off(f, k);
      split_store(s_wa[0], s_wa[1], o, ok ? Wa[gi] : 0.f);
      split_store(s_wt[0], s_wt[1], o, ok ? Wt[gi] : 0.f);
      const uint32_t ot = coreT_off(k, f, L.FP);
      split_store(s_c1[0], s_c1[1], ot, ok ? a.C1[gi] : 0.f);
      split_store(s_c2[0], s_c2[1], ot, ok ? a.C2[gi] : 0.f);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;

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
            tma_load_2d(s_stage + stage * STAGE_BYTES, &mapH, &bar_full[stage], n0, 32 * j);
            if (++stage == nstage) { stage = 0; ph ^= 1; }
          }
        }
        for (int w = 0; w < L.SW; ++w) {
          mbar_wait(&bar_empty[stage], ph ^ 1);
          mbar_expect_tx(&bar_full[stage], STAGE_BYTES);
          tma_load_2d(s_stage + stage * STAGE_BYTES, &mapW, &bar_full[stage], n0 + 32 * (w & 3),
                      128 * (w >> 2));
          if (++stage == nstage) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =====================================
    if (lane == 0) {
      const uint32_t id_big = idesc_tf32(128, 32, 0, 0);
      const uint32_t id_side = idesc_tf32(128, 16, 0, 0);
      const uint32_t sb_wa[2] = {smem_u32(s_wa[0]), smem_u32(s_wa[1])};
      const uint32_t sb_wt[2] = {smem_u32(s_wt[0]), smem_u32(s_wt[1])};
      const uint32_t sb_c1[2] = {smem_u32(s_c1[0]), smem_u32(s_c1[1])};
      const uint32_t sb_c2[2] = {smem_u32(s_c2[0]), smem_u32(s_c2[1])};
      const uint32_t sb_hp[2] = {smem_u32(s_hp[0]), smem_u32(s_hp[1])};
      const uint32_t sb_hn[2] = {smem_u32(s_hn[0]), smem_u32(s_hn[1])};
      const uint32_t sb_hnt[2] = {smem_u32(s_hnt[0]), smem_u32(s_hnt[1])};
      const uint32_t sbo_c = uint32_t(L.FP) * 32;   // chi^T rows k, K-dim FP
      const uint32_t sbo_hnt = BN * 32;            // H~^T rows k, K-dim 128
      // 3xTF32 product list: (a_hi,b_hi), (a_hi,b_lo), (a_lo,b_hi)
      const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};
      uint32_t c = 0;   // sub-tile counter (D / Z double buffer)
      int bi = 0;
      int last_w = -1;  // pending W-side sub-tile of the previous block
      auto issue_sideW = [&](uint32_t cc, int w, int first_of_block) {
        const uint32_t buf = cc & 1;
        const int t = w >> 2, u = w & 3;
        const uint32_t zbase = tmem + TM_Z + 128 * buf;
        for (int q = 0; q < 2; ++q) {          // num, den
          if (q == 1 && den_ones == 2) break;  // (never: W den needs Zd = 1 for beta = 1)
          const uint32_t dcol = tmem + TM_ACCW + 32 * t + 16 * q;
          for (int pr = 0; pr < 3; ++pr) {
            const uint32_t acol = zbase + 64 * q + 32 * pa[pr];
            for (int s = 0; s < 4; ++s) {
              const uint64_t bd = sdesc(sb_hnt[pb[pr]] + u * 1024 + s * 256, 128, sbo_hnt);
              const uint32_t acc = (first_of_block && (u == 0) && pr == 0 && s == 0) ? 0u : 1u;
              mma_ts(dcol, acol + 8 * s, bd, id_side, acc);
            }
          }
        }
      };
      auto issue_sideH = [&](uint32_t cc, int j) {
        const uint32_t buf = cc & 1;
        const uint32_t zbase = tmem + TM_Z + 128 * buf;
        for (int q = 0; q < 2; ++q) {
          if (q == 1 && den_ones) break;
          const uint32_t dcol = tmem + TM_ACCH + 16 * q;
          const uint32_t* cb = q == 0 ? sb_c1 : sb_c2;
          for (int pr = 0; pr < 3; ++pr) {
            const uint32_t acol = zbase + 64 * q + 32 * pa[pr];
            for (int s = 0; s < 4; ++s) {
              const uint64_t bd = sdesc(cb[pb[pr]] + j * 1024 + s * 256, 128, sbo_c);
              const uint32_t acc = (j == 0 && pr == 0 && s == 0) ? 0u : 1u;
              mma_ts(dcol, acol + 8 * s, bd, id_side, acc);
            }
          }
        }
      };
      for (int b = blockIdx.x; b < nblocks; b += gridDim.x, ++bi) {
        if (do_h) {
          mbar_wait(bar_hp, bi & 1);
          tc_fence_after();
          for (int j = 0; j < L.SH; ++j, ++c) {
            const uint32_t buf = c & 1;
            const uint32_t dcol = tmem + TM_D + 32 * buf;
            int m = 0;
            for (int pr = 0; pr < 3; ++pr)
              for (int s = 0; s < 2; ++s, ++m)
                mma_ss(dcol, sdesc(sb_hp[pa[pr]] + s * 256, 128, 512),
                       sdesc(sb_wa[pb[pr]] + j * 2048 + s * 256, 128, 512), id_big, m > 0);
            mma_commit(&bar_dfull[buf]);
            if (j > 0) {
              mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
              tc_fence_after();
              issue_sideH(c - 1, j - 1);
            } else if (last_w >= 0) {
              mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
              tc_fence_after();
              issue_sideW(c - 1, last_w, last_w < 4 ? 0 : 0);
              mma_commit(bar_accw);
              last_w = -1;
            }
          }
          mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
          tc_fence_after();
          issue_sideH(c - 1, L.SH - 1);
          mma_commit(bar_acch);
        } else if (last_w >= 0) {
          mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
          tc_fence_after();
          issue_sideW(c - 1, last_w, 0);
          mma_commit(bar_accw);
          last_w = -1;
        }
        mbar_wait(bar_hn, bi & 1);
        tc_fence_after();
        for (int w = 0; w < L.SW; ++w, ++c) {
          const uint32_t buf = c & 1;
          const uint32_t dcol = tmem + TM_D + 32 * buf;
          const int t = w >> 2, u = w & 3;
          int m = 0;
          for (int pr = 0; pr < 3; ++pr)
            for (int s = 0; s < 2; ++s, ++m)
              mma_ss(dcol, sdesc(sb_wt[pa[pr]] + t * 8192 + s * 256, 128, 512),
                     sdesc(sb_hn[pb[pr]] + u * 2048 + s * 256, 128, 512), id_big, m > 0);
          mma_commit(&bar_dfull[buf]);
          if (w > 0) {
            mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
            tc_fence_after();
            if (w == 1 && bi > 0) {
              mbar_wait(bar_accw_free, (bi - 1) & 1);
              tc_fence_after();
            }
            issue_sideW(c - 1, w - 1, 1);
          }
        }
        last_w = L.SW - 1;
      }
      if (last_w >= 0) {
        mbar_wait(&bar_zfull[(c - 1) & 1], ((c - 1) >> 1) & 1);
        tc_fence_after();
        issue_sideW(c - 1, last_w, 0);
        mma_commit(bar_accw);
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue =======================================
    const int e = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant
    const int h = e >> 2;            // column half / tile index
    const int row = 32 * q + lane;   // TMEM lane (n in the H phase, f_local in the W phase)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    double obj = 0.0;
    double accw_n[KP], accw_d[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) { accw_n[k] = 0.0; accw_d[k] = 0.0; }
    float hprev[8];
    int stage = 0;
    uint32_t ph = 0;
    uint32_t c = 0;
    int bi = 0;

    // rows of the block's H~_{p-1} (this thread: n = row, k in [8h, 8h+8))
    auto load_hprev = [&](int n0) {
      const int n = n0 + row;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = 8 * h + i;
        hprev[i] = (n < N && k < K) ? Hprev[size_t(n) * K + k] : 0.f;
        split_store(s_hp[0], s_hp[1], core_off(row, k), hprev[i]);
      }
    };
    auto store_hnew = [&](int n0, const float* hv) {
      const int n = n0 + row;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = 8 * h + i;
        const float v = (n < N && k < K) ? hv[i] : 0.f;
        if (do_h && n < N && k < K) Hnew[size_t(n) * K + k] = v;
        split_store(s_hn[0], s_hn[1], core_off(row, k), v);
        split_store(s_hnt[0], s_hnt[1], coreT_off(k, row, BN), v);
      }
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
      if (do_h) {
        // ---------------- H phase ----------------
        for (int j = 0; j < L.SH; ++j, ++c) {
          const uint32_t buf = c & 1;
          mbar_wait(&bar_dfull[buf], (c >> 1) & 1);
          mbar_wait(&bar_full[stage], ph);
          tc_fence_after();
          float y[16], zn[16], zd[16];
          tmem_ld16(lane_base + TM_D + 32 * buf + 16 * h, y);
          const float* tile = reinterpret_cast<const float*>(s_stage + stage * STAGE_BYTES);
          const bool nvalid = n0 + row < N;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int fl = 16 * h + i;
            const float x = tile[fl * 128 + row];
            const bool ok = nvalid && (32 * j + fl < F);
            float a1 = 0.f, a2 = 0.f;
            if (ok) zpair<FBC>(x, y[i] + kappa, beta, a1, a2);
            zn[i] = a1;
            zd[i] = a2;
          }
          float hi[16], lo[16];
          const uint32_t zb = lane_base + TM_Z + 128 * buf + 16 * h;
#pragma unroll
          for (int i = 0; i < 16; ++i) { hi[i] = to_tf32(zn[i]); lo[i] = to_tf32(zn[i] - hi[i]); }
          tmem_st16(zb + 0, hi);
          tmem_st16(zb + 32, lo);
          if (!den_ones) {
#pragma unroll
            for (int i = 0; i < 16; ++i) { hi[i] = to_tf32(zd[i]); lo[i] = to_tf32(zd[i] - hi[i]); }
            tmem_st16(zb + 64, hi);
            tmem_st16(zb + 96, lo);
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
        mbar_wait(bar_acch, bi & 1);
        tc_fence_after();
        float nv[8], dv[8], hv[8];
        tmem_ld8(lane_base + TM_ACCH + 8 * h, nv);
        if (!den_ones) tmem_ld8(lane_base + TM_ACCH + 16 + 8 * h, dv);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = 8 * h + i;
          float v = 0.f;
          if (k < K) {
            const double den = den_ones ? a.csum2[k] : double(dv[i]);
            const double r = double(nv[i]) / fmax(den, a.sc.floor);
            v = float(double(hprev[i]) * apply_exponent<double>(r, a.sc.gamma) * a.norms[k]);
          }
          hv[i] = v;
        }
        tc_fence_before();
        store_hnew(n0, hv);
      } else {
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
        const uint32_t buf = c & 1;
        const int t = w >> 2, u = w & 3;
        mbar_wait(&bar_dfull[buf], (c >> 1) & 1);
        mbar_wait(&bar_full[stage], ph);
        tc_fence_after();
        float y[16], zn[16], zd[16];
        tmem_ld16(lane_base + TM_D + 32 * buf + 16 * h, y);
        const char* tile = s_stage + stage * STAGE_BYTES;
        const int f = 128 * t + row;
        float x[16];
#pragma unroll
        for (int cq = 0; cq < 4; ++cq) {
          const int chunk = 4 * h + cq;
          const float4 v4 = *reinterpret_cast<const float4*>(tile + row * 128 +
                                                             ((chunk ^ (row & 7)) << 4));
          x[4 * cq + 0] = v4.x; x[4 * cq + 1] = v4.y; x[4 * cq + 2] = v4.z; x[4 * cq + 3] = v4.w;
        }
        float osum = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + 32 * u + 16 * h + i;
          const bool ok = f < F && n < N;
          float a1 = 0.f, a2 = 0.f;
          if (ok) {
            const float yy = y[i] + kappa;
            zpair<FBC>(x[i], yy, beta, a1, a2);
            osum += dterm<FBC>(x[i], yy, a2, beta);
          }
          zn[i] = a1;
          zd[i] = a2;
        }
        obj += double(osum);
        float hi[16], lo[16];
        const uint32_t zb = lane_base + TM_Z + 128 * buf + 16 * h;
#pragma unroll
        for (int i = 0; i < 16; ++i) { hi[i] = to_tf32(zn[i]); lo[i] = to_tf32(zn[i] - hi[i]); }
        tmem_st16(zb + 0, hi);
        tmem_st16(zb + 32, lo);
#pragma unroll
        for (int i = 0; i < 16; ++i) { hi[i] = to_tf32(zd[i]); lo[i] = to_tf32(zd[i] - hi[i]); }
        tmem_st16(zb + 64, hi);
        tmem_st16(zb + 96, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bar_zfull[buf]);
          mbar_arrive(&bar_empty[stage]);
        }
        if (++stage == nstage) { stage = 0; ph ^= 1; }
      }
      // ---------------- fold AccW into fp64 ----------------
      mbar_wait(bar_accw, bi & 1);
      tc_fence_after();
      if (h < L.FT) {
        float vn[16], vd[16];
        tmem_ld16(lane_base + TM_ACCW + 32 * h, vn);
        tmem_ld16(lane_base + TM_ACCW + 32 * h + 16, vd);
#pragma unroll
        for (int k = 0; k < KP; ++k) { accw_n[k] += double(vn[k]); accw_d[k] += double(vd[k]); }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_accw_free);
    }
    // ---- per-CTA outputs ----
    double* mypart = a.part + size_t(blockIdx.x) * 2 * F * K;
    if (h < L.FT) {
      const int f = 128 * h + row;
      if (f < F) {
        for (int k = 0; k < K; ++k) {
          mypart[size_t(f) * K + k] = accw_n[k];
          mypart[size_t(F) * K + size_t(f) * K + k] = accw_d[k];
        }
      }
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
