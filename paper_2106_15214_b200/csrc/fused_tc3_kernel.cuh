// tcgen05 pass pair for the fp32 shapes outside the single-read kernel's limits
// (F > 256 or 16 < K <= 32: BASELINE configs 2 and 3).  V of these shapes is L2-resident
// (34 / 67 MB against 126 MB), so the single-read constraint that forced the row-split cluster
// and its DSMEM exchange does not apply: the pass is two launches over a 2-D grid
//   (column group x, 128-row slice y)
// with the same roles as fused_tc2_kernel.cuh (TMA producer, Vt issuer, side issuer, two item
// teams, a U team) and the same item arithmetic, and no communication between CTAs:
//
//   hpass_tc  (MODE_H)  per 128-column block: H items over the slice's rows.
//             D[n x 32 f] = H~_{p-1} Wa^T (3xTF32, A from TMEM), Z -> TMEM,
//             AccH[n x 2K] += Z [chi_hi | chi_lo].  The slice's partial sums go to
//             hpart[slice][n][num K | den K] (fp32); tc3_h_finish adds the slices in order
//             and applies the H update (updates.py:223-235 / 173-181, solver.py:167-171).
//   wpass_tc  (MODE_W)  per block: H~_p rows published to SMEM (both operand layouts), W
//             items over the slice's rows: D[f x 32 n] = W~_p H~_p^T, objective,
//             AccW[f x 2K] += Z [H~_hi | H~_lo], folded into the fp64 slab every FOLD blocks
//             (updates.py:203-220, solver.py:304-309).
//
// KP (the padded rank) is 16 or 32.  TMEM: Vt 2 x 32 | Z 2 x 128 | Acc 4 KP | A operand 2 KP
// (448 / 512 columns).  SMEM: 7 V stages + the slice's B operands (Wa, chi1, chi2 in MODE_H;
// H~_p and its transpose in MODE_W).
#pragma once

#include "fused_tc2_kernel.cuh"

namespace bnmf {
namespace ftc3 {

using namespace bnmf::tc;
using namespace bnmf::ftc;
using bnmf::ftc2::tmem_ld32;

constexpr int MODE_H = 0, MODE_W = 1;
constexpr int TW = 4;                      // warps per item team (one per TMEM lane quadrant)
// Item teams and item width.  TMEM holds 64 Vt columns and 256 Z columns for the items in
// flight: 2 teams x 32-column items or 4 teams x 16-column items.  Four teams double the warps
// that overlap the MUFU / FMA / ALU work of different items (a lone warp issues one
// instruction every ~2.7 cycles) for 6 more small Vt MMAs per 32 columns: that pays for the
// classes with a long objective (beta = 0, 1, generic: config 3 0.161 -> 0.140 ms) and costs
// for the short ones (beta = 2, 1.5: config 2 0.077 -> 0.083 ms), so the class picks.
__host__ __device__ constexpr int teams_of(int fbc) {
#ifdef BNMF_TC3_NT
  return BNMF_TC3_NT;
#else
  return (fbc == FBC_2 || fbc == FBC_15) ? 2 : 4;
#endif
}
constexpr int W_TMA = 0, W_VT = 1, W_SIDE = 2, W_TEAM0 = 3;
__host__ __device__ constexpr int threads_of(int fbc) { return 32 * (W_TEAM0 + teams_of(fbc) * TW + 4); }

template <int KP>
struct Lay {
  static constexpr uint32_t OPB = FR * KP * 4;                 // one [128 x KP] fp32 tile
  static constexpr uint32_t CORE_SBO = (KP / 4) * 128;         // 8-row group of a [rows x KP] tile
  static constexpr uint32_t TB = (2 * KP / 8) * 4096;          // [2 KP rows x 128] K-major over 128
  static constexpr uint32_t HNTB = (2 * KP / 8) * HNT_SBO;     // same, 144-byte chunk pitch
  static constexpr uint32_t OFF_A = NSTAGE * STAGE_BYTES;      // MODE_H: Wa hi | lo; MODE_W: H~_p hi | lo
  static constexpr uint32_t OFF_B = OFF_A + 2 * OPB;           // MODE_H: chi1; MODE_W: H~_p^T
  static constexpr uint32_t OFF_C = OFF_B + TB;                // MODE_H: chi2
  static constexpr uint32_t END_H = OFF_C + TB;
  static constexpr uint32_t END_W = OFF_B + HNTB;
  static constexpr uint32_t OFF_BAR = END_H > END_W ? END_H : END_W;
  static constexpr uint32_t SMEM = OFF_BAR + 512 + 1024;
  static constexpr uint32_t TM_ACC = 320;                      // num [hi part KP | lo part KP], den at + 2 KP
  static constexpr uint32_t TM_OP = 320 + 4 * KP;              // A operand of the Vt tiles: hi KP | lo KP
  static_assert(SMEM <= 232448, "tc3: shared memory over the 227 KB limit");
  static_assert(TM_OP + 2 * KP <= 512, "tc3: TMEM over 512 columns");
  __host__ __device__ static constexpr uint32_t core(int r, int k) {
    return uint32_t((r >> 3) * CORE_SBO + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
  }
};

// D = A B^T over K = KP in 3xTF32: (hi, hi) + (hi, lo) + (lo, hi), KP / 8 k-steps each
template <int KP>
__device__ __forceinline__ void issue_vt3(uint32_t dcol, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi,
                                          uint64_t b_lo, uint32_t idesc) {
#pragma unroll
  for (int s = 0; s < KP / 8; ++s) mma_ts(dcol, a_hi + 8 * s, dplus(b_hi, 256 * s), idesc, s ? 1u : 0u);
#pragma unroll
  for (int s = 0; s < KP / 8; ++s) mma_ts(dcol, a_hi + 8 * s, dplus(b_lo, 256 * s), idesc, 1u);
#pragma unroll
  for (int s = 0; s < KP / 8; ++s) mma_ts(dcol, a_lo + 8 * s, dplus(b_hi, 256 * s), idesc, 1u);
}

template <int FBC, bool KAPPA, int KP, int MODE>
__global__ void __launch_bounds__(threads_of(FBC), 1)
pass_tc3(FusedArgs a, const __grid_constant__ CUtensorMap mapV, float* __restrict__ hpart,
         const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  // the H pass opens a timed iteration: the start of its timer (begin_iter folded in)
  if (MODE == MODE_H && a.tmark && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
    *a.tmark = globaltimer();
  using L = Lay<KP>;
  constexpr int NT = teams_of(FBC);          // item teams
  constexpr int IW = 64 / NT;                // columns of an item
  constexpr int NCH = IW / 8;                // Z k-steps of an item
  constexpr int HIT = 32 / IW;               // H items per V stage
  constexpr int WIT = BN / IW;               // W items per block
  constexpr int W_UTEAM = W_TEAM0 + NT * TW;
  constexpr int NWARPS3 = W_UTEAM + 4;       // 15 or 23
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* bar_full = bars;           // [NSTAGE]
  uint64_t* bar_empty = bars + 8;      // [NSTAGE]
  uint64_t* bar_dfull = bars + 16;     // [NT]
  uint64_t* bar_dfree = bars + 20;     // [NT]
  uint64_t* bar_zfull = bars + 24;     // [NT]
  uint64_t* bar_zfree = bars + 28;     // [NT]
  uint64_t* bar_op = bars + 32;        // the block's A operand (MODE_H) / B operands (MODE_W) are in place
  uint64_t* bar_opfree = bars + 33;    // the block's Vt tiles (MODE_H) / W-side products (MODE_W) retired
  uint64_t* bar_acc = bars + 34;       // Acc complete (MODE_H: every block; MODE_W: every fold)
  uint64_t* bar_accfree = bars + 35;   // Acc read out
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 40);
  __shared__ double s_red[NT * TW];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // optional wait-cycle counters (-DBNMF_TC_PROF): [CTA][warp][12] like fused_tc2_kernel.cuh
#ifdef BNMF_TC_PROF
  long long pc_[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) pc_[i] = 0;
  const long long t_start_ = clock64();
#define W3(call, cat) do { const long long t0_ = clock64(); call; pc_[cat] += clock64() - t0_; } while (0)
#else
#define W3(call, cat) call
#endif
  const int F = a.F, N = a.N, K = a.K;
  const int row0 = blockIdx.y * FR;
  const int FTr = min(FR, F - row0);
  const int SH = max(1, (FTr + 31) / 32);
  const int GX = gridDim.x, gx = blockIdx.x;
  const int nblocks = (N + BN - 1) / BN;
  const int nb = gx < nblocks ? (nblocks - 1 - gx) / GX + 1 : 0;
  const int par = iter_parity(st, slot, p_override);
  // KKT passes (a.kkt): the gradient core g = y^(beta-2) (y - x) of the finished iterate
  // (W~_p, H~_p) takes the place of Z_n and nothing that of Z_d, so that
  //   MODE_W: AccW num = g H~_p^T = grad_W (into the slab's num half)
  //   MODE_H: AccH num = W~_p^T g = grad_H (chi1 := W~_p; into hpart's num half)
  const int kkt = a.kkt;
  const float* Hsrc = (MODE == MODE_H && !kkt) ? a.Hbuf[par ^ 1] : (a.do_h ? a.Hout[par] : a.Hbuf[par]);
  const float* Wt = a.Wt2[par];
  const float* Wa = kkt ? Wt : (a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn);
  const float* C1g = kkt ? Wt : a.C1;
  const int den_ones = kkt ? 1 : a.den_ones;   // no denominator products in the KKT passes
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  auto col0 = [&](int blk) { return (gx + blk * GX) * BN; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], MODE == MODE_H ? HIT * TW : NT * TW);
    }
    for (int b = 0; b < NT; ++b) {
      mbar_init(&bar_dfull[b], 1);
      mbar_init(&bar_dfree[b], TW);
      mbar_init(&bar_zfull[b], TW);
      mbar_init(&bar_zfree[b], 1);
    }
    mbar_init(bar_op, 4);
    mbar_init(bar_opfree, 1);
    mbar_init(bar_acc, 1);
    mbar_init(bar_accfree, 4);
    mbar_fence_init();
  }
  if (warp == W_TMA && lane == 0) tma_prefetch(&mapV);
  if (warp == W_VT) tmem_alloc<512>(s_tmem);
  if (MODE == MODE_H && warp >= W_TEAM0) {
    // Wa (B of the Vt product): [f x k] core tiles, hi then lo; chi1 / chi2 (B of the side
    // products): K-major over f, rows k (hi) and KP + k (lo)
    for (int i = threadIdx.x - 32 * W_TEAM0; i < FR * KP; i += 32 * (NWARPS3 - W_TEAM0)) {
      const int fl = i / KP, k = i - fl * KP;
      const bool ok = fl < FTr && k < K;
      const size_t gi = size_t(row0 + fl) * K + k;
      float v, hi;
      v = ok ? Wa[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + L::OFF_A + L::core(fl, k), hi);
      sts_f32(sb + L::OFF_A + L::OPB + L::core(fl, k), v - hi);
      v = ok ? C1g[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + L::OFF_B + coreT_off(k, fl), hi);
      sts_f32(sb + L::OFF_B + coreT_off(k + KP, fl), v - hi);
      v = ok ? a.C2[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + L::OFF_C + coreT_off(k, fl), hi);
      sts_f32(sb + L::OFF_C + coreT_off(k + KP, fl), v - hi);
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  const int nit = MODE == MODE_H ? SH * HIT : WIT;   // items per block

  if (warp == W_TMA) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int bi = 0; bi < nb; ++bi) {
        const int n0 = col0(bi);
        for (int j = 0; j < SH; ++j) {
          W3(mbar_wait(&bar_empty[s], ph ^ 1u), 0);
          mbar_expect_tx(&bar_full[s], STAGE_BYTES);
          tma_load_2d(smem + s * STAGE_BYTES, &mapV, &bar_full[s], n0, row0 + 32 * j);
          if (++s == NSTAGE) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == W_VT) {
    // ======================= Vt issuer =======================================
    const uint32_t id_vt = idesc_tf32(128, IW, 0, 0);
    const uint64_t d_b = sdesc(sb + L::OFF_A, 128, L::CORE_SBO);
    int c = 0;
    for (int bi = 0; bi < nb; ++bi) {
      W3(mbar_wait(bar_op, bi & 1), 0);
      for (int j = 0; j < nit; ++j) {
        const int b = c & (NT - 1), m = c / NT;
        ++c;
        if (m > 0) W3(mbar_wait(&bar_dfree[b], (m - 1) & 1), 1);
        tc_fence_after();
        if (elect_one()) {
          // rows IW j.. of the B tile: IW / 8 eight-row groups per item
          issue_vt3<KP>(tmem + TM_D + IW * b, tmem + L::TM_OP, tmem + L::TM_OP + KP,
                        dplus(d_b, j * (IW / 8) * L::CORE_SBO),
                        dplus(d_b, j * (IW / 8) * L::CORE_SBO + L::OPB), id_vt);
          mma_commit(&bar_dfull[b]);
          if (MODE == MODE_H && j == nit - 1) mma_commit(bar_opfree);
        }
        __syncwarp();
      }
    }
  } else if (warp == W_SIDE) {
    // ======================= side issuer =====================================
    const uint32_t id_hi = idesc_tf32(128, 2 * KP, 0, 0);
    const uint32_t id_lo = idesc_tf32(128, KP, 0, 0);
    const uint64_t d_b1 = MODE == MODE_H ? sdesc(sb + L::OFF_B, 128, 4096)
                                         : sdesc(sb + L::OFF_B, HNT_LBO, HNT_SBO);
    const uint64_t d_b2 = sdesc(sb + L::OFF_C, 128, 4096);
    auto side = [&](uint32_t acc, uint32_t z, uint64_t bdesc, uint32_t kstride, bool fresh) {
#pragma unroll
      for (int s = 0; s < NCH; ++s) {
        mma_ts(acc, z + 32 * s, dplus(bdesc, kstride * s), id_hi, (fresh && s == 0) ? 0u : 1u);
        mma_ts(acc, z + 32 * s + 8, dplus(bdesc, kstride * s), id_lo, 1u);
      }
    };
    int c = 0, nfold = 0;
    for (int bi = 0; bi < nb; ++bi) {
      for (int j = 0; j < nit; ++j) {
        const int b = c & (NT - 1), m = c / NT;
        ++c;
        const uint32_t zb = tmem + TM_Z + 4 * IW * b;
        W3(mbar_wait(&bar_zfull[b], m & 1), 0);
        bool fresh;
        if (MODE == MODE_H) {
          fresh = j == 0;
          if (fresh && bi > 0) W3(mbar_wait(bar_accfree, (bi - 1) & 1), 1);
        } else {
          fresh = (bi % FOLD) == 0 && j == 0;
          if (fresh && bi > 0) { W3(mbar_wait(bar_accfree, nfold & 1), 1); ++nfold; }
        }
        tc_fence_after();
#ifdef BNMF_TC_PROF
        const long long ti_ = clock64();
#endif
        if (elect_one()) {
          if (MODE == MODE_H) {
            side(tmem + L::TM_ACC, zb, dplus(d_b1, j * IW * 32), 256, fresh);
            if (!den_ones) side(tmem + L::TM_ACC + 2 * KP, zb + 16, dplus(d_b2, j * IW * 32), 256, fresh);
            mma_commit(&bar_zfree[b]);
            if (j == nit - 1) mma_commit(bar_acc);
          } else {
            const uint64_t bh = dplus(d_b1, j * (IW / 4) * HNT_LBO);
            side(tmem + L::TM_ACC, zb, bh, 2 * HNT_LBO, fresh);
            if (!kkt) side(tmem + L::TM_ACC + 2 * KP, zb + 16, bh, 2 * HNT_LBO, fresh);
            mma_commit(&bar_zfree[b]);
            if (j == nit - 1) {
              mma_commit(bar_opfree);
              if ((bi % FOLD) == FOLD - 1 || bi == nb - 1) mma_commit(bar_acc);
            }
          }
        }
        __syncwarp();
#ifdef BNMF_TC_PROF
        pc_[2] += clock64() - ti_;
#endif
      }
    }
  } else if (warp < W_UTEAM) {
    // ======================= item teams ======================================
    const int team = (warp - W_TEAM0) / TW;
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    const uint32_t dcol = lane_base + TM_D + IW * team;
    const uint32_t zcol = lane_base + TM_Z + 4 * IW * team;
    const uint32_t dfull_a = smem_u32(&bar_dfull[team]), dfree_a = smem_u32(&bar_dfree[team]);
    const uint32_t zfull_a = smem_u32(&bar_zfull[team]), zfree_a = smem_u32(&bar_zfree[team]);
    const uint32_t full_a = smem_u32(bar_full), empty_a = smem_u32(bar_empty);
    const bool fok = row < FTr;
    double obj = 0.0;
    int m = 0, c = 0;
    float pc[PHI_TERMS];
    if (FBC == FBC_GEN) phi_coeffs(beta, pc);
    int s_cur = 0;
    uint32_t p_cur = 0;
    auto slot_of = [&](int j, uint32_t& ph) {
      int s = s_cur + j;
      ph = p_cur;
      if (s >= NSTAGE) { s -= NSTAGE; ph ^= 1u; }
      return s;
    };
    auto take_tile = [&](float* y) {
      W3(mbar_wait_a(dfull_a, m & 1), 0);
      tc_fence_after();
      if (IW == 32) tmem_ld32(dcol, y);
      else tmem_ld16(dcol, y);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_a(dfree_a);
    };
    auto wait_zfree = [&]() {
      if (m > 0) {
        W3(mbar_wait_a(zfree_a, (m - 1) & 1), 1);
        tc_fence_after();
      }
    };
    auto give_z = [&]() {
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_a(zfull_a);
      ++m;
    };
    for (int bi = 0; bi < nb; ++bi) {
      const int n0 = col0(bi);
      if (MODE == MODE_H) {
        // the team's items of the block: item it has sequence number c + it
        const int it0 = (team - c) & (NT - 1);
        c += SH * HIT;
        for (int it = it0; it < SH * HIT; it += NT) {
          // ---------- H item: rows row0 + r0 + [0, IW) of column n0 + row ----------
          const int j = it / HIT, r0 = IW * it;
          uint32_t ph;
          const int s = slot_of(j, ph);
          float x[IW], y[IW];
          W3(mbar_wait_a(full_a + 8 * s, ph), 2);
          const uint32_t xa = sb + s * STAGE_BYTES + (r0 - 32 * j) * VROWB + row * 4;
#pragma unroll
          for (int i = 0; i < IW; ++i) x[i] = lds_f32(xa + i * VROWB);
          take_tile(y);
          const bool full = n0 + BN <= N && r0 + IW <= FTr;
          const bool nok = n0 + row < N;
#pragma unroll
          for (int s4 = 0; s4 < NCH; ++s4) {
            float zn[8], zd[8];
            if (KAPPA) {
#pragma unroll
              for (int i = 0; i < 8; ++i) y[8 * s4 + i] += kappa;
            }
            if (kkt) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const bool ok = nok && (r0 + 8 * s4 + i < FTr);
                zn[i] = ok ? gcore32<FBC>(x[8 * s4 + i], y[8 * s4 + i], beta) : 0.f;
                zd[i] = 0.f;
              }
            } else {
              zpair8<FBC>(x + 8 * s4, y + 8 * s4, beta, zn, zd);
              if (!full) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const bool ok = nok && (r0 + 8 * s4 + i < FTr);
                  zn[i] = ok ? zn[i] : 0.f;
                  zd[i] = ok ? zd[i] : 0.f;
                }
              }
            }
            if (s4 == 0) wait_zfree();
            store_z(zcol + 32 * s4, zn, zd);
          }
          give_z();
          // the stage has been consumed: hand it back (one team reads an H stage)
          if (lane == 0) mbar_arrive_a(empty_a + 8 * s);
        }
      } else {
        uint32_t xrow = 0;
        if (q < SH) {
          uint32_t ph;
          const int s = slot_of(q, ph);
          W3(mbar_wait_a(full_a + 8 * s, ph), 2);
          xrow = sb + s * STAGE_BYTES + lane * VROWB;
        }
        const int u0 = (team - c) & (NT - 1);
        c += WIT;
        for (int u = u0; u < WIT; u += NT) {
          // ---------- W item: row row0 + row, columns n0 + IW u + [0, IW) ----------
          float x[IW], y[IW];
          if (q < SH) {
#pragma unroll
            for (int i = 0; i < IW; i += 4) {
              const float4 v = lds_f128(xrow + 4 * IW * u + 4 * i);
              x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < IW; ++i) x[i] = 0.f;
          }
          take_tile(y);
          const bool full = n0 + BN <= N && fok;
          float objb = 0.f;
#pragma unroll
          for (int s4 = 0; s4 < NCH; ++s4) {
            float zn[8], zd[8];
            float* yy = y + 8 * s4;
            const float* xx = x + 8 * s4;
            if (KAPPA) {
#pragma unroll
              for (int i = 0; i < 8; ++i) yy[i] += kappa;
            }
            if (kkt) {
              // KKT pass: the gradient core in place of Z_n, nothing in place of Z_d
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const bool ok = fok && (n0 + IW * u + 8 * s4 + i < N);
                zn[i] = ok ? gcore32<FBC>(xx[i], yy[i], beta) : 0.f;
                zd[i] = 0.f;
              }
            } else if (full) {
              float o0 = 0.f, o1 = 0.f;
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                z_and_obj<FBC>(xx[i], yy[i], 0.f, beta, zn[i], zd[i], o0, pc);
                z_and_obj<FBC>(xx[i + 1], yy[i + 1], 0.f, beta, zn[i + 1], zd[i + 1], o1, pc);
              }
              objb += o0 + o1;
            } else {
              float o0 = 0.f;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const bool ok = fok && (n0 + IW * u + 8 * s4 + i < N);
                float t = 0.f;
                z_and_obj<FBC>(xx[i], yy[i], 0.f, beta, zn[i], zd[i], t, pc);
                zn[i] = ok ? zn[i] : 0.f;
                zd[i] = ok ? zd[i] : 0.f;
                o0 += ok ? t : 0.f;
              }
              objb += o0;
            }
            if (s4 == 0) wait_zfree();
            store_z(zcol + 32 * s4, zn, zd);
          }
          obj += FBC == FBC_15 ? double(objb) * (2.0 / 3.0) : double(objb);
          give_z();
        }
        // both teams hand the V stages of the block back
        if (lane == 0) {
          for (int j = 0; j < SH; ++j) {
            uint32_t ph;
            mbar_arrive_a(empty_a + 8 * slot_of(j, ph));
          }
        }
      }
      s_cur += SH;
      if (s_cur >= NSTAGE) { s_cur -= NSTAGE; p_cur ^= 1u; }
    }
    for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
    if (lane == 0) s_red[warp - W_TEAM0] = obj;
  } else {
    // ======================= U team ==========================================
    const int q = warp & 3;
    const int row = 32 * q + lane;   // column n0 + row (MODE_H, publish) / row row0 + row (folds)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    // rows of H~ (MODE_H: H~_{p-1}, the A operand; MODE_W: H~_p, the B operands) of a block
    float h[KP];
    auto load_rows = [&](int blk) {
      const int n = col0(blk) + row;
      const bool ok = blk < nb && n < N;
      const float* src = Hsrc + size_t(n) * K;
      if (ok && (K & 3) == 0) {
#pragma unroll
        for (int k = 0; k < KP; k += 4) {
          if (k < K) {
            const float4 t = *reinterpret_cast<const float4*>(src + k);
            h[k] = t.x; h[k + 1] = t.y; h[k + 2] = t.z; h[k + 3] = t.w;
          } else {
            h[k] = h[k + 1] = h[k + 2] = h[k + 3] = 0.f;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < KP; ++k) h[k] = (ok && k < K) ? src[k] : 0.f;
      }
    };
    // hi | lo of a [lane x KP] row block into TMEM (the A operand of the Vt tiles)
    auto write_op = [&](const float* v) {
#pragma unroll
      for (int c0 = 0; c0 < 2 * KP; c0 += 32) {
        float z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int cc = c0 + i;                       // column: hi k (cc < KP) or lo k (cc - KP)
          const float x = v[cc < KP ? cc : cc - KP];
          const float hi = tf32_hi(x);
          z[i] = cc < KP ? hi : x - hi;
        }
        tmem_st32(lane_base + L::TM_OP + c0, z);
      }
      tmem_st_wait();
      tc_fence_before();
    };
    if (MODE == MODE_W) {
      // W~_p rows of the slice: the A operand of every Vt tile of this CTA
      float wv[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) wv[k] = (row < FTr && k < K) ? Wt[size_t(row0 + row) * K + k] : 0.f;
      write_op(wv);
    }
    double* mypart = a.part + size_t(blockIdx.x) * 2 * F * K;
    int nfold = 0;
    load_rows(0);
    if (MODE == MODE_H && nb > 0) {
      write_op(h);
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_op);
      load_rows(1);
    }
    for (int bi = 0; bi < nb; ++bi) {
      const int n = col0(bi) + row;
      if (MODE == MODE_H) {
        // the next block's A operand as soon as the Vt tiles of this block have retired (the
        // side products of this block are still running)
        if (bi + 1 < nb) {
          W3(mbar_wait(bar_opfree, bi & 1), 0);
          tc_fence_after();
          write_op(h);
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_op);
          load_rows(bi + 2);
        }
        // the slice's partial sums of the block: AccH -> hpart[slice][n][num KP | den KP]
        W3(mbar_wait(bar_acc, bi & 1), 1);
        tc_fence_after();
        float* dst = hpart + (size_t(blockIdx.y) * N + n) * (2 * KP);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          float v[2 * KP];
          if (s == 0 || !den_ones) {
#pragma unroll
            for (int c0 = 0; c0 < 2 * KP; c0 += 32) tmem_ld32(lane_base + L::TM_ACC + 2 * KP * s + c0, v + c0);
          }
          if (s == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_accfree);
          }
          if (n < N && (s == 0 || !den_ones)) {
#pragma unroll
            for (int k = 0; k < KP; k += 4)
              *reinterpret_cast<float4*>(dst + KP * s + k) =
                  make_float4(v[k] + v[KP + k], v[k + 1] + v[KP + k + 1], v[k + 2] + v[KP + k + 2],
                              v[k + 3] + v[KP + k + 3]);
          }
        }
      } else {
        // publish H~_p of the block: Hn rows (core tiles, hi then lo) and HnT scalars
        float lo[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const float x = n < N ? h[k] : 0.f;
          const float hi = tf32_hi(x);
          lo[k] = x - hi;
          h[k] = hi;
        }
        // the split above runs ahead of the wait: the operand buffers are single
        if (bi > 0) W3(mbar_wait(bar_opfree, (bi - 1) & 1), 0);   // W-side products of bi-1 retired
#pragma unroll
        for (int g = 0; g < KP / 4; ++g) {
          sts_f128(sb + L::OFF_A + L::core(row, 4 * g), h[4 * g], h[4 * g + 1], h[4 * g + 2], h[4 * g + 3]);
          sts_f128(sb + L::OFF_A + L::OPB + L::core(row, 4 * g), lo[4 * g], lo[4 * g + 1], lo[4 * g + 2],
                   lo[4 * g + 3]);
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          sts_f32(sb + L::OFF_B + hnt_off(k, row), h[k]);
          sts_f32(sb + L::OFF_B + hnt_off(k + KP, row), lo[k]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_op);
        load_rows(bi + 1);
        if ((bi % FOLD) == FOLD - 1 || bi == nb - 1) {
          // AccW of the last FOLD blocks into the fp64 slab (one owner thread per element)
          W3(mbar_wait(bar_acc, nfold & 1), 1);
          tc_fence_after();
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            float v[2 * KP];
            if (s == 0 || !kkt) {
#pragma unroll
              for (int c0 = 0; c0 < 2 * KP; c0 += 32) tmem_ld32(lane_base + L::TM_ACC + 2 * KP * s + c0, v + c0);
            }
            if (s == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bar_accfree);
            }
            if (row < FTr && (s == 0 || !kkt)) {
              double* dstd = mypart + size_t(s) * F * K + size_t(row0 + row) * K;
#pragma unroll
              for (int k = 0; k < KP; ++k) {
                if (k < K) {
                  const double add = double(v[k]) + double(v[KP + k]);
                  if (nfold == 0) dstd[k] = add;
                  else atomicAdd(dstd + k, add);
                }
              }
            }
          }
          ++nfold;
        }
      }
    }
    if (MODE == MODE_W && nfold == 0 && row < FTr) {   // CTA without blocks: zero its slab rows
      for (int s = 0; s < 2; ++s)
        for (int k = 0; k < K; ++k) mypart[size_t(s) * F * K + size_t(row0 + row) * K + k] = 0.0;
    }
  }
#ifdef BNMF_TC_PROF
  if (a.prof && lane == 0) {
    pc_[11] = clock64() - t_start_;
    long long* dstp = a.prof + ((size_t(blockIdx.y) * gridDim.x + blockIdx.x) * NWARPS3 + warp) * 12;
#pragma unroll
    for (int i = 0; i < 12; ++i) dstp[i] = pc_[i];
  }
#endif
#undef W3
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (MODE == MODE_W && threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < NT * TW; ++i) t += s_red[i];
    a.opart[size_t(blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
  if (warp == W_VT) tmem_dealloc<512>(tmem);
}

// H update from the slices' partial sums (fixed slice order):
//   H_p = H~_{p-1} (num / max(den, floor))^gamma, H~_p = H_p norms_p
template <int KP>
__global__ void tc3_h_finish(FusedArgs a, const float* __restrict__ hpart, int R,
                             const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  const int par = iter_parity(st, slot, p_override);
  const float* Hprev = a.Hbuf[par ^ 1];
  float* Hnew = a.Hout[par];
  const size_t total = size_t(a.N) * a.K;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t n = t / a.K;
    const int k = int(t - n * a.K);
    float num = 0.f, den = 0.f;
    for (int r = 0; r < R; ++r) {
      const float* p = hpart + (size_t(r) * a.N + n) * (2 * KP);
      num += p[k];
      if (!a.den_ones) den += p[KP + k];
    }
    const double d = a.den_ones ? a.csum2[k] : double(den);
    const double ratio = double(num) / fmax(d, a.sc.floor);
    const double hp = double(Hprev[t]) * apply_exponent<double>(ratio, a.sc.gamma);
    Hnew[t] = float(hp * a.norms[k]);
  }
}

// res_H partial sums of the H-side KKT pass: |min(H~_p, grad_H)| with grad_H the slices'
// partial sums added in order; one partial per block (fixed tree)
template <int KP>
__global__ void __launch_bounds__(256) tc3_kkt_h_finish(FusedArgs a, const float* __restrict__ hpart,
                                                        int R, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const float* Hp = a.Hbuf[iter_parity(st, slot, -1)];
  const size_t total = size_t(a.N) * a.K;
  __shared__ double red[256];
  double s = 0.0;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t n = t / a.K;
    const int k = int(t - n * a.K);
    float g = 0.f;
    for (int r = 0; r < R; ++r) g += hpart[(size_t(r) * a.N + n) * (2 * KP) + k];
    s += fabs(fmin(double(Hp[t]), double(g)));
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.opart[blockIdx.x] = red[0];
}

}  // namespace ftc3
}  // namespace bnmf
