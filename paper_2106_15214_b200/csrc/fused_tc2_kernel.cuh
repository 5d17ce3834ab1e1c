// tcgen05 fused single-read pass, second generation (fp32, rank K <= 16,
// F <= 256).  Same contract, block decomposition, SMEM layout, TMEM map and
// arithmetic as fused_tc_kernel.cuh (the v1 kernel; read its header first);
// what changes is who does what:
//
//   warp 0        TMA producer (V stages in item order, L2 prefetch two blocks ahead)
//   warp 1        Vt issuer: the W~H~ tiles of every item (3xTF32), TMEM owner
//   warp 2        side issuer: the W-side / H-side products of every item
//   warps 3..6    item team 0: items with an even sequence number
//   warps 7..10   item team 1: items with an odd sequence number
//   warps 11..14  U team: H~_{p-1} rows into TMEM, AccH read-out, the DSMEM
//                 exchange with the peer CTA, the H update, H~_p published
//                 to SMEM / HBM, AccW folded into the fp64 slab
//
// v1 walked all 16 epilogue warps through every item in lock-step, 8 elements
// per thread per item, and the same warps did the block-boundary work (U1/U2):
// ~50 thread-instructions per V element, most of them hand-off overhead.  Here
// an item belongs to one team of 4 warps (one per TMEM lane quadrant), a
// thread owns a whole TMEM lane of the tile (32 elements per item), the two
// teams alternate items so that one team's arithmetic covers the other's
// hand-off, and the block-boundary work runs beside the items on its own
// warps.  The two issuing warps keep the Vt tiles and the side products on
// independent in-order queues: a Vt tile waiting for H~_p (the U chain) does
// not hold back the side products of the items in flight.
//
// Hand-off per item c (buffer b = c & 1 belongs to team b):
//   dfull[b]  Vt issuer -> team     Vt tile complete            (tcgen05.commit)
//   dfree[b]  team -> Vt issuer     tile read into registers
//   zfull[b]  team -> side issuer   Z stored to TMEM
//   zfree[b]  side issuer -> team   side products of the item retired (commit)
//
// Item order and the V ring.  The H update of block b (AccH read-out, DSMEM
// exchange with the peer, ratio, publish: ~3000 cycles on the U team) stands
// between the last H item of b and its first W item, and only H items of later
// blocks can run beside it.  The items therefore go H(0), H(1), W(0), H(2),
// W(1), H(3), W(2), ...: all H items of block b+1 ahead of the W items of
// block b, so that the update of b runs under the W items of b-1.  The 7-stage
// ring follows that sequence instead of the block structure of V: an H item
// takes one stage (its 32 rows, released by its team after the Z store), the W
// items of a block take the block's SH stages (released by both teams after
// the last W item).  Every V row thus enters shared memory twice, the second
// time from L2 (the producer prefetches two blocks ahead); DRAM traffic is
// unchanged.  This is the default single-read kernel; BNMF_TC_V2=0 selects v1.
#pragma once

#include "fused_tc_kernel.cuh"

namespace bnmf {
namespace ftc2 {

using namespace bnmf::tc;
using namespace bnmf::ftc;

#ifndef BNMF_TC2_NT
#define BNMF_TC2_NT 2
#endif
constexpr int NTEAM = BNMF_TC2_NT;            // item teams: 2 (32-wide items) or 4 (16-wide items)
static_assert(NTEAM == 2 || NTEAM == 4, "2 or 4 item teams");
#ifndef BNMF_TC2_LOOKAHEAD
#define BNMF_TC2_LOOKAHEAD 4
#endif
// H items of block bi + 1 that run ahead of the W items of block bi (all of them by default):
// they and the W items of block bi - 1 ... cover the H-update chain of block bi (AccH read-out,
// DSMEM exchange, ratio, publish), which nothing else can overlap
constexpr int TC2_LOOKAHEAD = BNMF_TC2_LOOKAHEAD;
constexpr int TEAM_WARPS = 4;                 // one warp per TMEM lane quadrant
// TMEM holds 64 Vt columns and 256 Z columns for the items in flight: NTEAM items of IW columns
constexpr int IW = 64 / NTEAM;                // width of an item: rows (H item) / columns (W item)
constexpr int EPT = IW;                       // elements of an item per thread
constexpr int NCH = IW / 8;                   // 8-element chunks (one Z k-step each)
constexpr int HIT = 32 / IW;                  // H items per V stage
constexpr int WIT = BN / IW;                  // W items per block
constexpr int U_WARPS = 4;
constexpr int W_TMA = 0, W_VT = 1, W_SIDE = 2, W_TEAM0 = 3, W_UTEAM = W_TEAM0 + NTEAM * TEAM_WARPS;
constexpr int NWARPS2 = W_UTEAM + U_WARPS;    // 23 (15 with 4-warp teams)
constexpr int NTHREADS2 = 32 * NWARPS2;         // 480

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Item sequence of a CTA (every role walks it block by block): block bi lists its own H
// items (all of them for bi == 0, else 2..SH-1), then the first two H items of block bi + 1
// (they cover the H update of bi), then the W items of bi.  Items alternate between the two
// teams by sequence number.

template <int FBC, bool KAPPA>
__global__ void __launch_bounds__(NTHREADS2, 1)
fused_pass_tc2(FusedArgs a, const __grid_constant__ CUtensorMap mapV, int CL, int F0,
               const RunState* st, int slot, int p_override) {
  if (p_override < 0 && !iter_active(st, slot)) return;
  // first kernel of an iteration: the start of its timer (begin_iter folded in, solver.py:302)
  if (a.tmark && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *a.tmark = globaltimer();
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* bar_full = bars;           // [NSTAGE] TMA -> teams
  uint64_t* bar_empty = bars + 8;      // [NSTAGE] teams -> TMA
  uint64_t* bar_dfull = bars + 16;     // [NTEAM]
  uint64_t* bar_dfree = bars + 20;     // [NTEAM]
  uint64_t* bar_zfull = bars + 24;     // [NTEAM]
  uint64_t* bar_zfree = bars + 28;     // [NTEAM]
  uint64_t* bar_hp = bars + 32;        // H~_{p-1} rows of a block in TMEM
  uint64_t* bar_hpfree = bars + 33;    // the H-side Vt tiles of a block retired
  uint64_t* bar_hn = bars + 34;        // H~_p of a block in SMEM
  uint64_t* bar_wdone = bars + 35;     // W-side products of a block retired
  uint64_t* bar_acch = bars + 36;      // AccH of a block complete
  uint64_t* bar_accfree = bars + 37;   // AccH read out
  uint64_t* bar_accw = bars + 38;      // AccW of a fold complete
  uint64_t* bar_accwfree = bars + 39;  // AccW read out
  uint64_t* bar_xfull = bars + 40;     // peer's AccH partial landed (tx)
  uint64_t* bar_xempty = bars + 41;    // peer consumed my partial (remote arrivals)
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 48);
  __shared__ double s_red[NTEAM * TEAM_WARPS];
  __shared__ float s_nrm[KP], s_cs2[KP];
  __shared__ double s_redu[U_WARPS];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // optional wait-cycle counters (build with BNMF_TC_PROF=1): lane 0 of every warp
  // accumulates the cycles it spends in each wait category, [CTA][warp][12]
#ifdef BNMF_TC_PROF
  long long pcy_[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) pcy_[i] = 0;
  const long long t_start = clock64();
#define PWAIT(bar, parity, cat)                       \
  do {                                                \
    const long long t0_ = clock64();                  \
    mbar_wait(bar, parity);                           \
    pcy_[cat] += clock64() - t0_;                       \
  } while (0)
#define PWAITA(addr, parity, cat)                     \
  do {                                                \
    const long long t0_ = clock64();                  \
    mbar_wait_a(addr, parity);                        \
    pcy_[cat] += clock64() - t0_;                       \
  } while (0)
#define PTIME_BEGIN(v) const long long v = clock64()
#define PTIME_END(v, cat) pcy_[cat] += clock64() - v
#define PTIME_VAR(v) long long v = 0
#define PTIME_SET(v) v = clock64()
#else
#define PWAIT(bar, parity, cat) mbar_wait(bar, parity)
#define PWAITA(addr, parity, cat) mbar_wait_a(addr, parity)
#define PTIME_BEGIN(v)
#define PTIME_END(v, cat)
#define PTIME_VAR(v)
#define PTIME_SET(v)
#endif
  const int F = a.F, N = a.N, K = a.K;
  const uint32_t rank = CL > 1 ? cluster_ctarank() : 0u;
  const int row0 = rank ? F0 : 0;
  const int FTr = rank ? F - F0 : (F < F0 ? F : F0);
  const int SH = max(2, (FTr + 31) / 32);
  const int LA = TC2_LOOKAHEAD < SH ? TC2_LOOKAHEAD : SH;   // H items of block bi + 1 ahead of the W items of bi
  const int npairs = gridDim.x / CL, pi = blockIdx.x / CL;
  const int nblocks = (N + BN - 1) / BN;
  const int nb = pi < nblocks ? (nblocks - 1 - pi) / npairs + 1 : 0;
  const int par = iter_parity(st, slot, p_override);
  const int do_h = a.do_h;
  // KKT pass: the H items run on the finished iterate (W~_p, H~_p) with W~_p as both chi
  // maps, so AccH holds W~^T Zn and W~^T Zd; no W items, no update, no publish
  const int kkt = a.kkt;
  const float* Hprev = (do_h && !kkt) ? a.Hbuf[par ^ 1] : a.Hbuf[par];
  float* Hnew = a.Hout[par];
  const float* Wt = a.Wt2[par];
  const float* Wa = kkt ? Wt : (a.algorithm == 0 ? a.Wt2[par ^ 1] : a.Wn);
  const float* C1g = kkt ? Wt : a.C1;
  const float* C2g = kkt ? Wt : a.C2;
  const int den_ones = kkt ? 0 : a.den_ones;
  const int n_w = kkt ? 0 : WIT;  // W items per block
  const float kappa = float(a.sc.kappa), beta = float(a.sc.beta);
  auto col0 = [&](int blk) { return (pi + blk * npairs) * BN; };

  // ---- setup: barriers, TMEM, constant operands ---------------------------
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], NTEAM * TEAM_WARPS);
    }
    for (int b = 0; b < NTEAM; ++b) {
      mbar_init(&bar_dfull[b], 1);
      mbar_init(&bar_dfree[b], TEAM_WARPS);
      mbar_init(&bar_zfull[b], TEAM_WARPS);
      mbar_init(&bar_zfree[b], 1);
    }
    mbar_init(bar_hp, U_WARPS);
    mbar_init(bar_hpfree, 1);
    mbar_init(bar_hn, U_WARPS);
    mbar_init(bar_wdone, 1);
    mbar_init(bar_acch, 1);
    mbar_init(bar_accfree, U_WARPS);
    mbar_init(bar_accw, 1);
    mbar_init(bar_accwfree, U_WARPS);
    mbar_init(bar_xfull, 1);
    mbar_init(bar_xempty, U_WARPS);
    mbar_fence_init();
  }
  if (warp == W_TMA && lane == 0) tma_prefetch(&mapV);
  if (warp == W_VT) tmem_alloc<512>(s_tmem);
  if (warp >= W_TEAM0) {
    // Wa (B of the H-side Vt product): [f x k] core tiles, hi then lo.
    // chi1/chi2 (B of the H-side products): K-major over f, rows k (hi) and 16+k (lo).
    for (int i = threadIdx.x - 32 * W_TEAM0; i < FR * KP; i += 32 * (NWARPS2 - W_TEAM0)) {
      const int fl = i / KP, k = i - fl * KP;
      const bool ok = fl < FTr && k < K;
      const size_t gi = size_t(row0 + fl) * K + k;
      float v, hi;
      v = ok ? Wa[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + OFF_WA + core_off(fl, k), hi);
      sts_f32(sb + OFF_WA + HILO + core_off(fl, k), v - hi);
      v = ok ? C1g[gi] : 0.f; hi = tf32_hi(v);
      sts_f32(sb + OFF_C1 + coreT_off(k, fl), hi);
      sts_f32(sb + OFF_C1 + coreT_off(k + 16, fl), v - hi);
      v = ok ? C2g[gi] : 0.f; hi = tf32_hi(v);
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

  if (warp == W_TMA) {
    // ======================= TMA producer ===================================
    // The ring follows the item sequence: an H item takes one stage (its 32 rows), the W items
    // of a block take SH stages (all rows of the CTA).  The rows of a block are therefore
    // loaded twice, the second time from L2.
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      auto load = [&](int blk, int j) {
        PWAIT(&bar_empty[s], ph ^ 1u, 0);
        mbar_expect_tx(&bar_full[s], STAGE_BYTES);
        tma_load_2d(smem + OFF_STAGE + s * STAGE_BYTES, &mapV, &bar_full[s], col0(blk), row0 + 32 * j);
        if (++s == NSTAGE) { s = 0; ph ^= 1u; }
      };
      auto prefetch = [&](int blk) {
        if (blk < nb)
          for (int j = 0; j < SH; ++j) tma_prefetch_l2_2d(&mapV, col0(blk), row0 + 32 * j);
      };
      prefetch(0);
      prefetch(1);
      for (int bi = 0; bi < nb; ++bi) {
        prefetch(bi + 2);
        if (do_h) {
          const int j0 = (bi == 0 || kkt) ? 0 : LA;
          const int n_own = SH - j0, n_all = n_own + ((bi + 1 < nb && !kkt) ? LA : 0);
          for (int t = 0; t < n_all; ++t) {
            const bool own = t < n_own;
            load(own ? bi : bi + 1, own ? j0 + t : t - n_own);
          }
        }
        if (n_w)
          for (int j = 0; j < SH; ++j) load(bi, j);
      }
    }
  } else if (warp == W_VT) {
    // ======================= Vt issuer =======================================
    const uint32_t id_vt = idesc_tf32(128, IW, 0, 0);
    const uint64_t d_wa = sdesc(sb + OFF_WA, 128, 512);
    const uint64_t d_hn = sdesc(sb + OFF_HN, 128, 512);
    int c = 0;
    // Vt tile of the next item in sequence: waits until its team has read the previous tile of
    // the buffer, issues 6 MMAs, commits to dfull.  it = item within the block: B rows IW it..
    auto vt = [&](bool hside, int it, bool last_h) {
      const int b = c & (NTEAM - 1), m = c / NTEAM;
      ++c;
      if (m > 0) PWAIT(&bar_dfree[b], (m - 1) & 1, 2);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t off = uint32_t(it) * (IW / 8) * 512;
        if (hside) {
          issue_vt(tmem + TM_D + IW * b, tmem + TM_HP, tmem + TM_HP + 16, dplus(d_wa, off),
                   dplus(d_wa, off + HILO), id_vt);
        } else {
          issue_vt(tmem + TM_D + IW * b, tmem + TM_WT, tmem + TM_WT + 16, dplus(d_hn, off),
                   dplus(d_hn, off + HILO), id_vt);
        }
        mma_commit(&bar_dfull[b]);
        if (last_h) mma_commit(bar_hpfree);
      }
      __syncwarp();
    };
    for (int bi = 0; bi < nb; ++bi) {
      if (do_h) {
        const int j0 = (bi == 0 || kkt) ? 0 : LA;
        const int n_own = SH - j0, n_all = n_own + ((bi + 1 < nb && !kkt) ? LA : 0);
        for (int t = 0; t < n_all; ++t) {
          const bool own = t < n_own;
          const int j = own ? j0 + t : t - n_own;
          if (j == 0) PWAIT(bar_hp, (own ? bi : bi + 1) & 1, 0);
          for (int h = 0; h < HIT; ++h) vt(true, j * HIT + h, j == SH - 1 && h == HIT - 1);
        }
      }
      if (n_w) PWAIT(bar_hn, bi & 1, 1);
      for (int u = 0; u < n_w; ++u) vt(false, u, false);
    }
  } else if (warp == W_SIDE) {
    // ======================= side issuer =====================================
    const uint32_t id32 = idesc_tf32(128, 32, 0, 0);
    const uint32_t id16 = idesc_tf32(128, 16, 0, 0);
    const uint64_t d_c1 = sdesc(sb + OFF_C1, 128, 4096);
    const uint64_t d_c2 = sdesc(sb + OFF_C2, 128, 4096);
    const uint64_t d_hnt = sdesc(sb + OFF_HNT, HNT_LBO, HNT_SBO);
    // acc[:, 0:32] (+)= Z_hi [B_hi | B_lo], acc[:, 0:16] += Z_lo B_hi over the item's NCH k-steps
    auto side = [&](uint32_t acc, uint32_t z, uint64_t bdesc, uint32_t kstride, bool fresh) {
#pragma unroll
      for (int s = 0; s < NCH; ++s) {
        mma_ts(acc, z + 32 * s, dplus(bdesc, kstride * s), id32, (fresh && s == 0) ? 0u : 1u);
        mma_ts(acc, z + 32 * s + 8, dplus(bdesc, kstride * s), id16, 1u);
      }
    };
    int c = 0;
    // it = H item within the block (IW rows each)
    auto side_h = [&](int blk, int it) {
      const int b = c & (NTEAM - 1), m = c / NTEAM;
      ++c;
      const uint32_t zb = tmem + TM_Z + 4 * IW * b;
      PWAIT(&bar_zfull[b], m & 1, 0);
      if (it == 0 && blk > 0) PWAIT(bar_accfree, (blk - 1) & 1, 1);
      tc_fence_after();
      if (elect_one()) {
        side(tmem + TM_ACCH, zb, dplus(d_c1, it * IW * 32), 256, it == 0);
        if (!den_ones) side(tmem + TM_ACCH + 32, zb + 16, dplus(d_c2, it * IW * 32), 256, it == 0);
        mma_commit(&bar_zfree[b]);
        if (it == SH * HIT - 1) mma_commit(bar_acch);
      }
      __syncwarp();
    };
    for (int bi = 0; bi < nb; ++bi) {
      if (do_h) {
        const int j0 = (bi == 0 || kkt) ? 0 : LA;
        const int n_own = SH - j0, n_all = n_own + ((bi + 1 < nb && !kkt) ? LA : 0);
        for (int t = 0; t < n_all; ++t) {
          const bool own = t < n_own;
          const int j = own ? j0 + t : t - n_own;
          for (int h = 0; h < HIT; ++h) side_h(own ? bi : bi + 1, j * HIT + h);
        }
      }
      const bool fold_end = (bi % FOLD) == FOLD - 1 || bi == nb - 1;
      for (int u = 0; u < n_w; ++u) {
        const int b = c & (NTEAM - 1), m = c / NTEAM;
        ++c;
        const uint32_t zb = tmem + TM_Z + 4 * IW * b;
        const bool fresh = (bi % FOLD) == 0 && u == 0;
        PWAIT(&bar_zfull[b], m & 1, 0);
        if (fresh && bi > 0) PWAIT(bar_accwfree, ((bi / FOLD) - 1) & 1, 2);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t bh = dplus(d_hnt, u * (IW / 4) * HNT_LBO);
          side(tmem + TM_ACCW, zb, bh, 2 * HNT_LBO, fresh);
          side(tmem + TM_ACCW + 32, zb + 16, bh, 2 * HNT_LBO, fresh);
          mma_commit(&bar_zfree[b]);
          if (u == WIT - 1) {
            mma_commit(bar_wdone);
            if (fold_end) mma_commit(bar_accw);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp < W_UTEAM) {
    // ======================= item teams ======================================
    const int team = (warp - W_TEAM0) / TEAM_WARPS;
    const int q = warp & 3;          // TMEM lane quadrant
    const int row = 32 * q + lane;   // TMEM lane: n (H items) or f - row0 (W items)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    const uint32_t dcol = lane_base + TM_D + IW * team;
    const uint32_t zcol = lane_base + TM_Z + 4 * IW * team;
    const uint32_t dfull_a = smem_u32(&bar_dfull[team]), dfree_a = smem_u32(&bar_dfree[team]);
    const uint32_t zfull_a = smem_u32(&bar_zfull[team]), zfree_a = smem_u32(&bar_zfree[team]);
    const uint32_t full_a = smem_u32(bar_full), empty_a = smem_u32(bar_empty);
    const bool rows_full = FTr == 32 * SH;
    const bool fok = row < FTr;
    double obj = 0.0;
    float pc[PHI_TERMS];
    if (FBC == FBC_GEN) phi_coeffs(beta, pc);
    int m = 0;   // own items done (phase counter of this team's buffers)

    // Vt tile of the item -> registers (buffer handed back), then wait until the side
    // products of the previous own item have retired so that Z may be overwritten
    auto take_tile = [&](float* y, int cat) {
      PWAITA(dfull_a, m & 1, cat);
      tc_fence_after();
      if (EPT == 32) tmem_ld32(dcol, y);
      else tmem_ld16(dcol, y);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_a(dfree_a);
    };
    // before the first Z store of an item: the side products of the previous own item have
    // retired (the arithmetic of the item runs ahead of this wait)
    auto wait_zfree = [&]() {
      if (m > 0) {
        PWAITA(zfree_a, (m - 1) & 1, 4);
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

    // ---------------- H item: rows row0 + IW it + [0, IW) of column n0 + row (stage s) -------
    auto h_item = [&](int n0, int it, int s, uint32_t ph) {
      PTIME_BEGIN(t_it);
      PTIME_BEGIN(t_p0);
      float x[EPT], y[EPT];
      PWAITA(full_a + 8 * s, ph, 2);
      const int r0 = IW * it;
      const uint32_t xa = sb + OFF_STAGE + s * STAGE_BYTES + (r0 & 31) * VROWB + row * 4;
#pragma unroll
      for (int i = 0; i < EPT; ++i) x[i] = lds_f32(xa + i * VROWB);
      PTIME_END(t_p0, 7);
      PTIME_BEGIN(t_p1);
      take_tile(y, 0);
      PTIME_END(t_p1, 8);
      PTIME_BEGIN(t_p2);
      const bool full = n0 + BN <= N && (rows_full || r0 + IW <= FTr);
      const bool nok = n0 + row < N;
#pragma unroll
      for (int s4 = 0; s4 < NCH; ++s4) {
        float zn[8], zd[8];
        if (KAPPA) {
#pragma unroll
          for (int i = 0; i < 8; ++i) y[8 * s4 + i] += kappa;
        }
        zpair8<FBC>(x + 8 * s4, y + 8 * s4, beta, zn, zd);
        if (!full) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool ok = nok && (r0 + 8 * s4 + i < FTr);
            zn[i] = ok ? zn[i] : 0.f;
            zd[i] = ok ? zd[i] : 0.f;
          }
        }
        if (s4 == 0) wait_zfree();
        store_z(zcol + 32 * s4, zn, zd);
      }
      PTIME_END(t_p2, 9);
      PTIME_BEGIN(t_p3);
      give_z();
      PTIME_END(t_p3, 10);
      PTIME_END(t_it, 5);
    };

    // ---------------- W item: row row0 + row, columns n0 + IW idx + [0, IW) ------------------
    auto w_item = [&](int n0, int idx, uint32_t xrow) {
      PTIME_BEGIN(t_it);
      float x[EPT], y[EPT];
      if (q < SH) {
#pragma unroll
        for (int i = 0; i < EPT; i += 4) {
          const float4 v = lds_f128(xrow + 4 * IW * idx + 4 * i);
          x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < EPT; ++i) x[i] = 0.f;
      }
      take_tile(y, 1);
      const bool full = n0 + BN <= N && fok;
      {
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
          if (FBC == FBC_15 && full) {
            // beta = 1.5, full tile: Z and the objective two lanes per instruction
            zpair8<FBC>(xx, yy, beta, zn, zd);
            const uint64_t two = f2pack(2.f, 2.f);
            uint64_t acc = 0ull;
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const uint64_t sx = f2pack(sqrt_fast(xx[i]), sqrt_fast(xx[i + 1]));
              const uint64_t zdp = f2pack(zd[i], zd[i + 1]);
              const uint64_t dq = f2sub(sx, zdp);
              acc = f2fma(f2mul(dq, dq), f2fma(two, sx, zdp), acc);
            }
            float o0, o1;
            f2unpack(acc, o0, o1);
            objb += o0 + o1;
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
              const bool ok = fok && (n0 + IW * idx + 8 * s4 + i < N);
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
      }
      give_z();
      PTIME_END(t_it, 6);
    };

    int c = 0;                 // sequence number of the next item
    int sl = 0;                // ring slot of the next stage in load order
    uint32_t sp = 0;           // and its phase
    for (int bi = 0; bi < nb; ++bi) {
      if (do_h) {
        const int j0 = (bi == 0 || kkt) ? 0 : LA;
        const int n_own = SH - j0, n_all = n_own + ((bi + 1 < nb && !kkt) ? LA : 0);
        // the team's items of the list: item i of the list has sequence number c + i
        for (int i = (team - c) & (NTEAM - 1); i < n_all * HIT; i += NTEAM) {
          const int t = i / HIT;
          const bool own = t < n_own;
          const int j = own ? j0 + t : t - n_own;
          int s = sl + t;
          uint32_t ph = sp;
          if (s >= NSTAGE) { s -= NSTAGE; ph ^= 1u; }
          h_item(col0(own ? bi : bi + 1), j * HIT + (i - t * HIT), s, ph);
          // the stage goes back after the item's Z store (its x values are consumed); only
          // HIT of the NTEAM teams touch a stage, each arrives for NTEAM / HIT
          if (lane == 0) mbar_arrive_cnt_a(empty_a + 8 * s, NTEAM / HIT);
        }
        c += n_all * HIT;
        sl += n_all;
        if (sl >= NSTAGE) { sl -= NSTAGE; sp ^= 1u; }
      }
      if (n_w) {
        // this warp's V rows of the block are stage q of the block's SH stages
        uint32_t xrow = 0;
        if (q < SH) {
          int s = sl + q;
          uint32_t ph = sp;
          if (s >= NSTAGE) { s -= NSTAGE; ph ^= 1u; }
          PWAITA(full_a + 8 * s, ph, 3);
          xrow = sb + OFF_STAGE + s * STAGE_BYTES + lane * VROWB;
        }
        const int n0 = col0(bi);
        for (int u = (team - c) & (NTEAM - 1); u < n_w; u += NTEAM) w_item(n0, u, xrow);
        c += n_w;
        // every team hands the V stages of the block back
        if (lane == 0) {
          for (int j = 0; j < SH; ++j) {
            int s = sl + j;
            if (s >= NSTAGE) s -= NSTAGE;
            mbar_arrive_a(empty_a + 8 * s);
          }
        }
        sl += SH;
        if (sl >= NSTAGE) { sl -= NSTAGE; sp ^= 1u; }
      }
    }
    for (int o = 16; o > 0; o >>= 1) obj += __shfl_down_sync(0xffffffffu, obj, o);
    if (lane == 0) s_red[warp - W_TEAM0] = obj;
  } else {
    // ======================= U team ==========================================
    const int q = warp & 3;
    const int row = 32 * q + lane;   // column n0 + row (H update) / row row0 + row (folds)
    const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16);
    double* mypart = a.part + size_t(blockIdx.x) * 2 * F * K;
    // per-k constants of the H update live in shared memory (registers are what bounds this role)
    if (threadIdx.x - 32 * W_UTEAM < KP) {
      const int k = threadIdx.x - 32 * W_UTEAM;
      s_nrm[k] = (do_h && k < K) ? float(a.norms[k]) : 0.f;
      s_cs2[k] = (do_h && den_ones && k < K) ? float(a.csum2[k]) : 1.f;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * U_WARPS) : "memory");
    const float gam = float(a.sc.gamma);
    const float floor_f = fmaxf(float(a.sc.floor), 1.17549435e-38f);
    // H~_{p-1} rows of blocks b, b+1 (b = next block to finish its H update)
    float h0[KP], h1[KP];
    auto load_rows = [&](int blk, float* h) {
      const int n = col0(blk) + row;
      const bool ok = blk < nb && n < N;
      const float* src = Hprev + size_t(n) * K;
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
    // H~_{p-1} rows of a block as the TMEM A operand of the H-side Vt tiles
    auto write_hp = [&](const float* h) {
      float z[32];
#pragma unroll
      for (int k = 0; k < KP; ++k) { z[k] = tf32_hi(h[k]); z[KP + k] = h[k] - z[k]; }
      tmem_st32(lane_base + TM_HP, z);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_hp);
    };
    // W~_p rows of this CTA into TMEM (A operand of the W-side Vt tiles)
    {
      float z[32];
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const float v = (row < FTr && k < K) ? Wt[size_t(row0 + row) * K + k] : 0.f;
        z[k] = tf32_hi(v);
        z[KP + k] = v - z[k];
      }
      tmem_st32(lane_base + TM_WT, z);
      tmem_st_wait();
    }
    load_rows(0, h0);
    load_rows(1, h1);
    if (do_h && nb > 0) write_hp(h0);
    else tc_fence_before();
    int nfold = 0;
    double kres = 0.0;
    bool fold_pending = false;
    // add the TMEM W sums of the last FOLD blocks into the fp64 slab; one owner thread per
    // slab element: the first fold stores, later folds are fire-and-forget fp64 reductions
    // applied in program order
    auto fold = [&]() {
      PWAIT(bar_accw, nfold & 1, 5);
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        float v[32];
        tmem_ld32(lane_base + TM_ACCW + 32 * s, v);
        if (s == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_accwfree);
        }
        if (row < FTr) {
          double* dst = mypart + size_t(s) * F * K + size_t(row0 + row) * K;
#pragma unroll
          for (int k = 0; k < KP; ++k) {
            if (k < K) {
              const double add = double(v[k]) + double(v[KP + k]);
              if (nfold == 0) dst[k] = add;
              else atomicAdd(dst + k, add);
            }
          }
        }
      }
      ++nfold;
    };
    for (int bi = 0; bi < nb; ++bi) {
      const int n = col0(bi) + row;
      float hv[KP];
      PTIME_VAR(t_chain);
      // H~_{p-1} of the next block: its H items run before the H update of bi
      if (do_h && bi + 1 < nb) {
        PWAIT(bar_hpfree, bi & 1, 0);
        tc_fence_after();
        write_hp(h1);
      }
      if (fold_pending) fold();
      if (do_h) {
        // U1: AccH of the block read out (and sent to the peer CTA)
        float unum[KP], uden[KP];
        PWAIT(bar_acch, bi & 1, 1);
        PTIME_SET(t_chain);
        tc_fence_after();
        {
          float r[32];
          tmem_ld32(lane_base + TM_ACCH, r);
#pragma unroll
          for (int k = 0; k < KP; ++k) unum[k] = r[k] + r[KP + k];
          if (!den_ones) {
            tmem_ld32(lane_base + TM_ACCH + 32, r);
#pragma unroll
            for (int k = 0; k < KP; ++k) uden[k] = r[k] + r[KP + k];
          } else {
#pragma unroll
            for (int k = 0; k < KP; ++k) uden[k] = 0.f;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_accfree);
        PTIME_END(t_chain, 8);
        if (CL > 1) {
          const uint32_t peer = rank ^ 1u;
          if (bi > 0) PWAIT(bar_xempty, (bi - 1) & 1, 2);
          // only the ceil(K / 4) used 16-byte groups travel (and no denominators when they are ones)
          const int ng = (K + 3) >> 2;
          if (threadIdx.x == 32 * W_UTEAM)
            mbar_expect_tx_u32(smem_u32(bar_xfull), uint32_t(BN * 16 * ng * (den_ones ? 1 : 2)));
          const uint32_t rbar = mapa_shared(smem_u32(bar_xfull), peer);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (g < ng) {
              const uint32_t my0 = sb + OFF_XCH + uint32_t(((2 * g) * BN + row) * 16);
              st_async_v4(mapa_shared(my0, peer),
                          make_float4(unum[4 * g], unum[4 * g + 1], unum[4 * g + 2], unum[4 * g + 3]),
                          rbar);
              if (!den_ones)
                st_async_v4(mapa_shared(my0 + BN * 16, peer),
                            make_float4(uden[4 * g], uden[4 * g + 1], uden[4 * g + 2], uden[4 * g + 3]),
                            rbar);
            }
          }
          PTIME_END(t_chain, 6);
          // U2: peer partial added (fp32 a + b is commutative, so both CTAs form
          // bitwise-identical totals)
          PWAIT(bar_xfull, bi & 1, 3);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (g < ng) {
              const uint32_t my0 = sb + OFF_XCH + uint32_t(((2 * g) * BN + row) * 16);
              const float4 pn = lds_f128(my0);
              unum[4 * g] += pn.x; unum[4 * g + 1] += pn.y; unum[4 * g + 2] += pn.z; unum[4 * g + 3] += pn.w;
              if (!den_ones) {
                const float4 pd = lds_f128(my0 + BN * 16);
                uden[4 * g] += pd.x; uden[4 * g + 1] += pd.y; uden[4 * g + 2] += pd.z; uden[4 * g + 3] += pd.w;
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(bar_xempty), peer));
          PTIME_END(t_chain, 10);
        }
        if (kkt) {
          // res_H partial: |min(H~_p, W~_p^T Zd - W~_p^T Zn)| (diagnostics.py:55-58); each
          // column is counted by one CTA of the pair
          if ((CL == 1 || (q >> 1) == int(rank)) && n < N) {
            float t = 0.f;
#pragma unroll
            for (int k = 0; k < KP; ++k)
              if (k < K) t += fabsf(fminf(h0[k], uden[k] - unum[k]));
            kres += double(t);
          }
#pragma unroll
          for (int k = 0; k < KP; ++k) h0[k] = h1[k];
          load_rows(bi + 2, h1);
          continue;
        }
        // H~_p = H~_{p-1} (num / max(den, floor))^gamma norms; k >= K has h0 = nrm = 0
        float r[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k)
          r[k] = unum[k] * rcp_fast(fmaxf(den_ones ? s_cs2[k] : uden[k], floor_f));
        if (gam == 0.5f) {
#pragma unroll
          for (int k = 0; k < KP; ++k) r[k] = sqrt_fast(r[k]);
        } else if (gam != 1.f) {
          // rare exponents (beta outside [1, 3]): one copy of powf (code size)
          float rr[KP];
#pragma unroll
          for (int k = 0; k < KP; ++k) rr[k] = r[k];
#pragma unroll 1
          for (int k = 0; k < KP; ++k) {
            const float t = powf(rr[0], gam);
#pragma unroll
            for (int i = 0; i + 1 < KP; ++i) rr[i] = rr[i + 1];
            rr[KP - 1] = t;
          }
#pragma unroll
          for (int k = 0; k < KP; ++k) r[k] = rr[k];
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) hv[k] = h0[k] * r[k] * s_nrm[k];
      } else {
#pragma unroll
        for (int k = 0; k < KP; ++k) hv[k] = n < N ? h0[k] : 0.f;
      }
      if (do_h) { PTIME_END(t_chain, 9); }
      if (bi > 0) PWAIT(bar_wdone, (bi - 1) & 1, 4);   // W MMAs of bi-1 read Hn/HnT
      {
        // Hn: row n of the core tiles (4 chunks of 4 k, hi then lo);
        // HnT: one scalar per (k, hi/lo), conflict-free across the warp
        float lo[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k) { const float hi = tf32_hi(hv[k]); lo[k] = hv[k] - hi; hv[k] = hi; }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          sts_f128(sb + OFF_HN + core_off(row, 4 * g), hv[4 * g], hv[4 * g + 1], hv[4 * g + 2],
                   hv[4 * g + 3]);
          sts_f128(sb + OFF_HN + HILO + core_off(row, 4 * g), lo[4 * g], lo[4 * g + 1],
                   lo[4 * g + 2], lo[4 * g + 3]);
        }
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          sts_f32(sb + OFF_HNT + hnt_off(k, row), hv[k]);
          sts_f32(sb + OFF_HNT + hnt_off(k + 16, row), lo[k]);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_hn);
        if (do_h) { PTIME_END(t_chain, 7); }
        // global traffic only after the SMEM publish
        if (do_h && (CL == 1 || (q >> 1) == int(rank)) && n < N) {
          float* dst = Hnew + size_t(n) * K;
          if ((K & 3) == 0) {
#pragma unroll
            for (int k = 0; k < KP; k += 4)
              if (k < K)
                *reinterpret_cast<float4*>(dst + k) =
                    make_float4(hv[k] + lo[k], hv[k + 1] + lo[k + 1], hv[k + 2] + lo[k + 2],
                                hv[k + 3] + lo[k + 3]);
          } else {
#pragma unroll
            for (int k = 0; k < KP; ++k)
              if (k < K) dst[k] = hv[k] + lo[k];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < KP; ++k) h0[k] = h1[k];
      load_rows(bi + 2, h1);
      // the fold of a finished group waits for the W products of this block, which now run
      // after the H items of the next one: it is taken at the top of the next iteration so
      // that it does not hold back H~_{p-1} of the block after next
      fold_pending = !kkt && ((bi % FOLD) == FOLD - 1 || bi == nb - 1);
    }
    if (fold_pending) fold();
    if (kkt) {
      for (int o = 16; o > 0; o >>= 1) kres += __shfl_down_sync(0xffffffffu, kres, o);
      if (lane == 0) s_redu[warp - W_UTEAM] = kres;
    } else if (nfold == 0 && row < FTr) {   // CTA without blocks: zero its slab rows
      for (int s = 0; s < 2; ++s)
        for (int k = 0; k < K; ++k) mypart[size_t(s) * F * K + size_t(row0 + row) * K + k] = 0.0;
    }
  }
#ifdef BNMF_TC_PROF
  if (a.prof && lane == 0) {
    pcy_[11] = clock64() - t_start;
    long long* dst = a.prof + (size_t(blockIdx.x) * NWARPS2 + warp) * 12;
#pragma unroll
    for (int i = 0; i < 12; ++i) dst[i] = pcy_[i];
  }
#endif
#undef PWAIT
#undef PWAITA
#undef PTIME_BEGIN
#undef PTIME_VAR
#undef PTIME_SET
#undef PTIME_END
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < NTEAM * TEAM_WARPS; ++i) t += s_red[i];
    if (kkt) {
      t = 0.0;
      for (int i = 0; i < U_WARPS; ++i) t += s_redu[i];
    }
    a.opart[blockIdx.x] = t;
  }
  if (CL > 1) cluster_sync_all();   // no CTA leaves while its peer may still signal it
  if (warp == W_VT) tmem_dealloc<512>(tmem);
}

}  // namespace ftc2
}  // namespace bnmf
