// Fused single-read schedule (fp32, sub_iters == 1): host orchestration.
//
// Per outer iteration p (one CUDA-graph slot):
//   pass p            one read of V: H update of iteration p, objective of
//                     iterate p, W-side partial sums of iteration p+1
//   fused_reduce      fixed-order sum of the per-CTA partials -> comm
//   ncclAllReduce     (N-sharded runs) comm across ranks
//   finish_iter       trace row p + stop rule (solver.py:309-319)
//   fused_update      W_{p+1}, norms, W~_{p+1}, chi maps for pass p+1
// The pass kernel is the tcgen05 kernel (fused_pass_tc, see fused_tc_kernel.cuh)
// when its shape limits hold, else the register-tiled SIMT pair fs2::hpass +
// fs2::wpass (fused_simt2.cuh).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include <cuda.h>

#include "engine.h"
#include "fused_simt.cuh"
#include "fused_simt2.cuh"
#include "fused_tc_kernel.cuh"
#include "fused_tc2_kernel.cuh"
#include "fused_tc3_kernel.cuh"
#include "small_kernels.cuh"

namespace bnmf {

struct FusedState {
  int F = 0, N = 0, K = 0;
  float* H[2] = {nullptr, nullptr};
  float* W2[2] = {nullptr, nullptr};
  float* Wn = nullptr;
  float* C1 = nullptr;
  float* C2 = nullptr;
  double* norms = nullptr;
  double* csum2 = nullptr;
  double* part = nullptr;
  double* opart = nullptr;
  int bc = BC_GEN;
  // SIMT pair: wpass grid (s2_rc row chunks x s2_S column segments)
  int s2_rc = 0, s2_S = 0, s2_seg = 0;
  // tensor-core pass
  bool tc = false;
  int tc_grid = 0;
  int tc_cl = 1;      // CTAs per cluster (row split of F)
  int tc_f0 = 0;      // rows of cluster rank 0
  size_t tc_smem = 0;
  CUtensorMap mapV;
  long long* prof = nullptr;   // BNMF_TC_PROF=1: wait-cycle counters [grid][48]
  size_t prof_n = 0;
  int cap = 0;                 // BNMF_TC_MAX_CLUSTERS at creation (test knob)
  bool v1 = false;             // true with BNMF_TC_V2=0 (first-generation kernel, A/B knob)
  // tcgen05 pass pair over a (column group, 128-row slice) grid: F > 256 or 16 < K <= 32
  bool tc3 = false;
  int t3_gx = 0, t3_r = 0, t3_kp = 16;
  float* hpart = nullptr;      // [slice][N][num KP | den KP] H-side partial sums
  double* kcomm = nullptr;     // KKT pass of the pair: grad_W (F x K) summed over the slabs
  double* kpart = nullptr;     // KKT pass: per-CTA sums of |min(H~, grad_H)|
  int kparts = 0;
  double* kcs = nullptr;       // KKT pass, beta = 1 on the SIMT pair: colsum(W~_p) (K)
};

// The single-read pass runs the second-generation kernel (fused_tc2_kernel.cuh: item teams, two
// issuing warps, a dedicated U team, the H items of the next block ahead of the W items of the
// current one).  BNMF_TC_V2=0 selects the first-generation kernel (fused_tc_kernel.cuh), kept
// as the A/B twin (profiles/r02_fused_pass_experiments.md).
static bool env_tc_v1() {
  const char* c = getenv("BNMF_TC_V2");
  return c && c[0] == '0';
}

// BNMF_TC3=0 keeps the F > 256 / 16 < K <= 32 shapes on the SIMT pair (A/B knob)
static bool tc3_wanted(int K) {
  const char* e = getenv("BNMF_TC3");
  const char* f = getenv("BNMF_FUSED_SIMT");
  return K <= 32 && !(e && e[0] == '0') && !(f && f[0] == '1');
}

// BNMF_TC_PAIR=1: the pass pair also for the single-read kernel's shapes (A/B knob)
static bool env_force_pair() {
  const char* e = getenv("BNMF_TC_PAIR");
  return e && e[0] == '1';
}

static int env_cluster_cap() {
  const char* c = getenv("BNMF_TC_MAX_CLUSTERS");
  return c ? std::max(0, atoi(c)) : 0;
}

static FusedState* g_last_tc = nullptr;

constexpr int TC3_KKT_BLOCKS = 592;   // blocks (= partial sums) of the pair's H-side KKT finish

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool fused_tc_shape_ok(int F, int K) {
  return F >= 1 && F <= 256 && K >= 1 && K <= ftc::KP;
}

template <int FBC, bool KAPPA>
static cudaLaunchConfig_t tc_config(const FusedState* fs, cudaStream_t stream,
                                    cudaLaunchAttribute* attr, bool v2) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(fs->tc_grid, 1, 1);
  cfg.blockDim = dim3(v2 ? ftc2::NTHREADS2 : ftc::NTHREADS, 1, 1);
  cfg.dynamicSmemBytes = fs->tc_smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = fs->tc_cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

#define FCK(call)                                                           \
  do {                                                                      \
    cudaError_t e_ = (call);                                                \
    if (e_ != cudaSuccess) {                                                \
      err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return -1;                                                            \
    }                                                                       \
  } while (0)

// one thread per row of W for F <= 1024 (no serial latency chain per column)
constexpr int FU_THREADS = 1024;

bool fused_supported(int dtype, int F, int K, int algorithm, int L, int Lw, int Lh, double beta) {
  (void)F; (void)beta;
  if (dtype != BNMF_FP32) return false;
  if (K > FS_KMAX) return false;
  if (algorithm == BNMF_JMM) return L == 1;
  return Lw == 1 && Lh == 1;
}

template <int BC, int KJ>
static int wpass_occ(int K) {
  auto k = fs2::wpass<BC, KJ>;
  const int sm = int(fs2::w_smem(K));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, fs2::THREADS, sm) != cudaSuccess) {
    cudaGetLastError();
    n = 2;
  }
  return std::max(1, n);
}

template <int KJ>
static int wpass_occ_bc(int bc, int K) {
  switch (bc) {
    case BC_0: return wpass_occ<BC_0, KJ>(K);
    case BC_1: return wpass_occ<BC_1, KJ>(K);
    case BC_2: return wpass_occ<BC_2, KJ>(K);
    default: return wpass_occ<BC_GEN, KJ>(K);
  }
}

// resident wpass CTAs per SM for this beta class and rank
static int wpass_occupancy(int bc, int K) {
  return K <= 32 ? wpass_occ_bc<1>(bc, K) : wpass_occ_bc<2>(bc, K);
}

int fused_create(FusedState** out, const FusedIO& io, std::string& err) {
  FusedState* fs = new FusedState;
  *out = fs;
  fs->F = io.F; fs->N = io.N; fs->K = io.K;
  size_t fk = size_t(io.F) * io.K, nk = size_t(io.N) * io.K;
  FCK(cudaMalloc(&fs->H[0], nk * sizeof(float)));
  FCK(cudaMalloc(&fs->H[1], nk * sizeof(float)));
  FCK(cudaMalloc(&fs->W2[0], fk * sizeof(float)));
  FCK(cudaMalloc(&fs->W2[1], fk * sizeof(float)));
  FCK(cudaMalloc(&fs->Wn, fk * sizeof(float)));
  FCK(cudaMalloc(&fs->C1, fk * sizeof(float)));
  FCK(cudaMalloc(&fs->C2, fk * sizeof(float)));
  FCK(cudaMalloc(&fs->norms, io.K * sizeof(double)));
  FCK(cudaMalloc(&fs->csum2, io.K * sizeof(double)));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  {
    // wpass: one wave of CTAs (row chunks x column segments <= resident
    // slots, rounded down: a partial second wave would double the tail), the
    // segments in whole 32-column steps
    const int ncb = (io.N + fs2::NC - 1) / fs2::NC;
    fs->s2_rc = (io.F + fs2::TF - 1) / fs2::TF;
    const int slots = nsm * wpass_occupancy(beta_class(io.sc.beta), io.K);
    int S = std::max(1, std::min(ncb, slots / fs->s2_rc));
    const int steps = (ncb + S - 1) / S;
    fs->s2_seg = steps * fs2::NC;
    fs->s2_S = (io.N + fs->s2_seg - 1) / fs->s2_seg;
  }
  const char* force_simt = getenv("BNMF_FUSED_SIMT");
  fs->tc = fused_tc_shape_ok(io.F, io.K) && encode_fn() != nullptr &&
           !(force_simt && force_simt[0] == '1') && !env_force_pair();
  if (fs->tc) {
    const int nb = (io.N + ftc::BN - 1) / ftc::BN;
    fs->tc_smem = ftc::SMEM_BYTES;
    if (io.F > ftc::FR) {
      fs->tc_cl = 2;
      // split rows in multiples of 32 so that rank 1 keeps >= 33 rows
      const int half = ((io.F + 1) / 2 + 31) / 32 * 32;
      fs->tc_f0 = std::min(ftc::FR, half);
    } else {
      fs->tc_cl = 1;
      fs->tc_f0 = io.F;
    }
    fs->v1 = env_tc_v1();
    auto kern = fs->v1 ? ftc::fused_pass_tc<ftc::FBC_15, false> : ftc2::fused_pass_tc2<ftc::FBC_15, false>;
    FCK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fs->tc_smem)));
    FCK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int clusters = nsm / fs->tc_cl;
    if (fs->tc_cl > 1) {
      cudaLaunchAttribute attr[1];
      FusedState probe = *fs;
      probe.tc_grid = fs->tc_cl * clusters;
      cudaLaunchConfig_t cfg = tc_config<ftc::FBC_15, false>(&probe, io.stream, attr, !fs->v1);
      int maxc = 0;
      if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) == cudaSuccess && maxc > 0)
        clusters = std::min(clusters, maxc);
      cudaGetLastError();
    }
    // test knob: cap the grid so that every cluster walks many column blocks
    // (the steady-state schedule of a full-size pass on a small matrix)
    fs->cap = env_cluster_cap();
    if (fs->cap > 0) clusters = std::min(clusters, fs->cap);
    fs->tc_grid = fs->tc_cl * std::max(1, std::min(nb, clusters));
  }
  // BNMF_TC3=0 keeps these shapes on the SIMT pair (A/B knob)
  fs->tc3 = !fs->tc && tc3_wanted(io.K) && encode_fn() != nullptr;
  if (fs->tc3) {
    const int nb = (io.N + ftc::BN - 1) / ftc::BN;
    fs->t3_kp = io.K <= 16 ? 16 : 32;
    fs->t3_r = (io.F + ftc::FR - 1) / ftc::FR;
    fs->t3_gx = std::max(1, std::min(nb, nsm / fs->t3_r));
    FCK(cudaMalloc(&fs->hpart, size_t(fs->t3_r) * io.N * 2 * fs->t3_kp * sizeof(float)));
    FCK(cudaMalloc(&fs->kcomm, (size_t(2) * io.F * io.K + 8) * sizeof(double)));
  }
  int gmax = std::max(std::max(fs->tc_grid, fs->s2_S), fs->t3_gx);
  const int gobj = std::max(std::max(gmax, fs->s2_S * fs->s2_rc), fs->t3_gx * fs->t3_r);
  const char* prof_env = getenv("BNMF_TC_PROF");
  if ((fs->tc || fs->tc3) && prof_env && prof_env[0] == '1') {
    const size_t np = size_t(std::max(fs->tc_grid, fs->t3_gx * fs->t3_r)) * 288 + 3 * 4096;
    fs->prof_n = np;
    FCK(cudaMalloc(&fs->prof, np * sizeof(long long)));
    FCK(cudaMemset(fs->prof, 0, np * sizeof(long long)));
    g_last_tc = fs;
  }
  fs->kparts = std::max(std::max(gmax, (io.N + fs2::NC - 1) / fs2::NC), TC3_KKT_BLOCKS);
  FCK(cudaMalloc(&fs->kpart, size_t(fs->kparts) * sizeof(double)));
  FCK(cudaMalloc(&fs->kcs, io.K * sizeof(double)));
  FCK(cudaMalloc(&fs->part, size_t(gmax) * 2 * fk * sizeof(double)));
  FCK(cudaMalloc(&fs->opart, size_t(gobj) * sizeof(double)));
  if (fs->tc || fs->tc3) {
    // V stages: [32 rows x 132 columns] boxes, unswizzled; the 4 extra
    // columns pad the SMEM rows to 528 B (conflict-free in both phases)
    cuuint64_t dims[2] = {cuuint64_t(io.N), cuuint64_t(io.F)};
    cuuint64_t strides[1] = {cuuint64_t(io.ldv) * 4};
    cuuint32_t box[2] = {cuuint32_t(ftc::VROW), 32}, es[2] = {1, 1};
    EncodeTiledFn enc = encode_fn();
    CUresult r1 = enc(&fs->mapV, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(io.V), dims,
                      strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 != CUDA_SUCCESS) {
      err = "cuTensorMapEncodeTiled failed";
      return -1;
    }
  }
  return 0;
}

void fused_destroy(FusedState* fs) {
  if (!fs) return;
  float* fp[] = {fs->H[0], fs->H[1], fs->W2[0], fs->W2[1], fs->Wn, fs->C1, fs->C2, fs->hpart};
  for (float* q : fp) if (q) cudaFree(q);
  double* dp[] = {fs->norms, fs->csum2, fs->part, fs->opart, fs->kpart, fs->kcs, fs->kcomm};
  for (double* q : dp) if (q) cudaFree(q);
  if (fs->prof) cudaFree(fs->prof);
  if (g_last_tc == fs) g_last_tc = nullptr;
  delete fs;
}

static FusedArgs make_args(FusedState* fs, const FusedIO& io, int do_h) {
  FusedArgs a;
  a.V = io.V; a.ldv = (long long)io.ldv;
  a.F = io.F; a.N = io.N; a.K = io.K;
  a.Hbuf[0] = fs->H[0]; a.Hbuf[1] = fs->H[1];
  a.Hout[0] = fs->H[0]; a.Hout[1] = fs->H[1];
  a.Wt2[0] = fs->W2[0]; a.Wt2[1] = fs->W2[1];
  a.Wn = fs->Wn; a.C1 = fs->C1; a.C2 = fs->C2;
  a.norms = fs->norms; a.csum2 = fs->csum2;
  a.part = fs->part; a.opart = fs->opart;
  a.algorithm = io.algorithm;
  a.do_h = do_h;
  a.den_ones = beta_class(io.sc.beta) == BC_1 ? 1 : 0;
  a.sc = io.sc;
  a.prof = fs->prof;
  a.kkt = 0;
  a.tmark = nullptr;
  return a;
}

template <int BC, int KJ>
static cudaError_t launch_simt2(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                                int p_override) {
  if (a.do_h) {
    auto hk = fs2::hpass<BC, KJ>;
    const int hs = int(fs2::h_smem(io.K));
    cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, hs);
    hk<<<(io.N + fs2::NC - 1) / fs2::NC, fs2::THREADS, hs, io.stream>>>(a, io.st, slot,
                                                                          p_override);
  }
  if (a.kkt) return cudaGetLastError();
  auto wk = fs2::wpass<BC, KJ>;
  const int ws = int(fs2::w_smem(io.K));
  cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, ws);
  wk<<<dim3(fs->s2_rc, fs->s2_S), fs2::THREADS, ws, io.stream>>>(a, io.st, slot, p_override,
                                                                 fs->s2_seg);
  return cudaGetLastError();
}

template <int BC>
static cudaError_t launch_simt(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                               int p_override) {
  if (io.K <= 32) return launch_simt2<BC, 1>(fs, a, io, slot, p_override);
  return launch_simt2<BC, 2>(fs, a, io, slot, p_override);
}

template <int FBC, bool KAPPA>
static cudaError_t launch_tc(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                             int p_override) {
  // the KKT pass exists in the second-generation kernel only
  const bool v2 = !fs->v1 || a.kkt;
  auto kern = v2 ? ftc2::fused_pass_tc2<FBC, KAPPA> : ftc::fused_pass_tc<FBC, KAPPA>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(fs->tc_smem));
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = tc_config<FBC, KAPPA>(fs, io.stream, attr, v2);
  return cudaLaunchKernelEx(&cfg, kern, a, fs->mapV, fs->tc_cl, fs->tc_f0, io.st, slot,
                            p_override);
}

template <int FBC>
static cudaError_t launch_tc_k(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                               int p_override) {
  if (io.sc.kappa != 0.0) return launch_tc<FBC, true>(fs, a, io, slot, p_override);
  return launch_tc<FBC, false>(fs, a, io, slot, p_override);
}

template <int FBC, int KP>
static cudaError_t launch_tc3(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                              int p_override) {
  const dim3 grid(fs->t3_gx, fs->t3_r);
  const int sm = int(ftc3::Lay<KP>::SMEM);
  if (a.kkt == 3) {   // H-side KKT pass: grad_H partials, then |min(H~, grad_H)| per block
    auto hk = ftc3::pass_tc3<FBC, true, KP, ftc3::MODE_H>;
    cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    hk<<<grid, ftc3::threads_of(FBC), sm, io.stream>>>(a, fs->mapV, fs->hpart, io.st, slot, p_override);
    ftc3::tc3_kkt_h_finish<KP><<<TC3_KKT_BLOCKS, 256, 0, io.stream>>>(a, fs->hpart, fs->t3_r, io.st,
                                                                      slot);
    return cudaGetLastError();
  }
  if (a.do_h && !a.kkt) {
    auto hk = ftc3::pass_tc3<FBC, true, KP, ftc3::MODE_H>;
    cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    hk<<<grid, ftc3::threads_of(FBC), sm, io.stream>>>(a, fs->mapV, fs->hpart, io.st, slot, p_override);
    const size_t nk = size_t(io.N) * io.K;
    ftc3::tc3_h_finish<KP><<<int(std::min<size_t>((nk + 255) / 256, 148 * 8)), 256, 0, io.stream>>>(
        a, fs->hpart, fs->t3_r, io.st, slot, p_override);
  }
  auto wk = ftc3::pass_tc3<FBC, true, KP, ftc3::MODE_W>;
  cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  wk<<<grid, ftc3::threads_of(FBC), sm, io.stream>>>(a, fs->mapV, fs->hpart, io.st, slot, p_override);
  return cudaGetLastError();
}

template <int FBC>
static cudaError_t launch_tc3_k(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                                int p_override) {
  if (fs->t3_kp == 16) return launch_tc3<FBC, 16>(fs, a, io, slot, p_override);
  return launch_tc3<FBC, 32>(fs, a, io, slot, p_override);
}

static cudaError_t launch_pass(FusedState* fs, const FusedArgs& a, const FusedIO& io, int slot,
                               int p_override) {
  if (fs->tc3 && a.kkt != 1) {   // kkt == 2: the W-side KKT pass of the pair
    const double beta = io.sc.beta;
    if (beta == 1.5) return launch_tc3_k<ftc::FBC_15>(fs, a, io, slot, p_override);
    if (beta == 0.0) return launch_tc3_k<ftc::FBC_0>(fs, a, io, slot, p_override);
    if (beta == 1.0) return launch_tc3_k<ftc::FBC_1>(fs, a, io, slot, p_override);
    if (beta == 2.0) return launch_tc3_k<ftc::FBC_2>(fs, a, io, slot, p_override);
    return launch_tc3_k<ftc::FBC_GEN>(fs, a, io, slot, p_override);
  }
  if (fs->tc) {
    const double beta = io.sc.beta;
    if (beta == 1.5) return launch_tc_k<ftc::FBC_15>(fs, a, io, slot, p_override);
    if (beta == 0.0) return launch_tc_k<ftc::FBC_0>(fs, a, io, slot, p_override);
    if (beta == 1.0) return launch_tc_k<ftc::FBC_1>(fs, a, io, slot, p_override);
    if (beta == 2.0) return launch_tc_k<ftc::FBC_2>(fs, a, io, slot, p_override);
    return launch_tc_k<ftc::FBC_GEN>(fs, a, io, slot, p_override);
  }
  switch (fs->bc) {
    case BC_0: return launch_simt<BC_0>(fs, a, io, slot, p_override);
    case BC_1: return launch_simt<BC_1>(fs, a, io, slot, p_override);
    case BC_2: return launch_simt<BC_2>(fs, a, io, slot, p_override);
    default: return launch_simt<BC_GEN>(fs, a, io, slot, p_override);
  }
}

// pass -> reduce -> allreduce -> (finish) -> update
static int enqueue_pass_and_update(FusedState* fs, const FusedIO& io, int slot, int p_override,
                                   bool finish, std::string& err) {
  FusedArgs a = make_args(fs, io, p_override == 0 ? 0 : 1);
  // a timed iteration: its first kernel marks the start of the timer (begin_iter, solver.py:302)
  if (finish) a.tmark = &io.st->t_begin;
  size_t fk2 = size_t(2) * io.F * io.K;
  if (io.ev_a) FCK(record_event(io.ev_a, io.stream));
  FCK(launch_pass(fs, a, io, slot, p_override));
  if (io.ev_b) FCK(record_event(io.ev_b, io.stream));
  const bool s2 = !fs->tc && !fs->tc3;
  const int gpart = fs->tc ? fs->tc_grid : (fs->tc3 ? fs->t3_gx : fs->s2_S);
  const int gobj = fs->tc3 ? fs->t3_gx * fs->t3_r : (s2 ? fs->s2_S * fs->s2_rc : gpart);
  fused_reduce<<<int((fk2 + 1 + 255) / 256), 256, 0, io.stream>>>(
      fs->part, fs->opart, gpart, gobj, int(fk2), io.K,
      fs->tc ? fs->tc_f0 : io.F, fs->tc ? fs->tc_cl : 1, io.comm, io.st, slot, p_override);
  FCK(cudaGetLastError());
  if (io.launches) *io.launches += fs->tc3 ? (a.do_h ? 4 : 2) : ((s2 && a.do_h) ? 3 : 2);
  if (io.nranks > 1) {
    ncclResult_t r = ncclAllReduce(io.comm, io.comm, fk2 + 1, ncclDouble, ncclSum, io.nccl,
                                   io.stream);
    if (r != ncclSuccess) { err = std::string("ncclAllReduce: ") + ncclGetErrorString(r); return -1; }
    if (io.launches) *io.launches += 1;
  }
  // the trace row and stop rule of the iteration (finish_iter) ride in fused_update
  WPair wp;
  wp.w[0] = fs->W2[0]; wp.w[1] = fs->W2[1];
  fused_update<<<io.K, FU_THREADS, 0, io.stream>>>(io.comm, io.F, io.K, wp, fs->Wn, fs->C1, fs->C2,
                                            fs->norms, fs->csum2, io.algorithm, a.den_ones, io.sc,
                                            io.st, slot, p_override, finish ? io.st : nullptr,
                                            io.tr_obj, io.tr_sec);
  FCK(cudaGetLastError());
  if (io.launches) *io.launches += 1;
  return 0;
}

// ---- KKT residuals of the finished iterate (diagnostics.py:46-59), untimed like the
// reference's (they follow finish_iter) ---------------------------------------------------------
//   res_W: grad_W = Zd H~^T - Zn H~^T at (W~_p, H~_p) are the W-side sums pass p has just
//          reduced into comm for iteration p+1, so it costs F K operations
//   res_H: one H-side-only pass (tcgen05: fused_pass_tc2 in KKT mode; else fs2::hpass in KKT
//          mode) with W~_p as both chi maps; per-CTA partials in kpart
static __global__ void kkt_colsum(WPair Wt2, int F, int K, double* out, const RunState* st,
                                  int slot) {
  if (!iter_active(st, slot)) return;
  const float* W = Wt2.w[iter_parity(st, slot, -1)];
  const int k = blockIdx.x;
  __shared__ double red[32];
  double s = 0.0;
  for (int f = threadIdx.x; f < F; f += blockDim.x) s += double(W[size_t(f) * K + k]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x + 31) / 32; ++w) t += red[w];
    out[k] = t;
  }
}

// comm[2FK + 1] = sum of the per-CTA res_H partials (fixed order: strided per thread, then a tree)
static __global__ void __launch_bounds__(1024) kkt_sum(const double* __restrict__ kpart, int G,
                                                       double* __restrict__ out,
                                                       const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  __shared__ double red[1024];
  double s = 0.0;
  for (int g = threadIdx.x; g < G; g += 1024) s += kpart[g];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

static __global__ void __launch_bounds__(1024) kkt_finish(const double* __restrict__ comm, WPair Wt2,
                                                          int F, int K, double kn,
                                                          double* __restrict__ tr_kkt,
                                                          const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const float* W = Wt2.w[iter_parity(st, slot, -1)];
  const size_t fk = size_t(F) * K;
  __shared__ double red[32];
  double s = 0.0;
  for (size_t i = threadIdx.x; i < fk; i += blockDim.x)
    s += fabs(fmin(double(W[i]), comm[fk + i] - comm[i]));
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    const long long it = st->base + slot;
    tr_kkt[2 * (it - 1) + 0] = t / double(fk);
    tr_kkt[2 * (it - 1) + 1] = comm[2 * fk + 1] / kn;
  }
}

// res_W from an explicit gradient (the pass pair's W-side KKT pass): grad[i] = kcomm[i]
static __global__ void __launch_bounds__(1024) kkt_finish_g(const double* __restrict__ grad,
                                                            const double* __restrict__ resh, WPair Wt2,
                                                            int F, int K, double kn,
                                                            double* __restrict__ tr_kkt,
                                                            const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const float* W = Wt2.w[iter_parity(st, slot, -1)];
  const size_t fk = size_t(F) * K;
  __shared__ double red[32];
  double s = 0.0;
  for (size_t i = threadIdx.x; i < fk; i += blockDim.x) s += fabs(fmin(double(W[i]), grad[i]));
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    const long long it = st->base + slot;
    tr_kkt[2 * (it - 1) + 0] = t / double(fk);
    tr_kkt[2 * (it - 1) + 1] = *resh / kn;
  }
}

static int enqueue_kkt(FusedState* fs, const FusedIO& io, int slot, std::string& err) {
  FusedArgs a = make_args(fs, io, 1);
  a.kkt = 1;
  a.opart = fs->kpart;
  a.csum2 = fs->kcs;
  WPair wp;
  wp.w[0] = fs->W2[0]; wp.w[1] = fs->W2[1];
  const size_t fk2 = size_t(2) * io.F * io.K;
  int nparts = fs->tc_grid;
  if (fs->tc3) {
    a.kkt = 3;
    nparts = TC3_KKT_BLOCKS;
  } else if (!fs->tc) {   // SIMT pair: fs2::hpass in KKT mode
    nparts = (io.N + fs2::NC - 1) / fs2::NC;
    if (a.den_ones) {
      kkt_colsum<<<io.K, 256, 0, io.stream>>>(wp, io.F, io.K, fs->kcs, io.st, slot);
      FCK(cudaGetLastError());
      if (io.launches) *io.launches += 1;
    }
  }
  FCK(launch_pass(fs, a, io, slot, -1));
  kkt_sum<<<1, 1024, 0, io.stream>>>(fs->kpart, nparts, io.comm + fk2 + 1, io.st, slot);
  FCK(cudaGetLastError());
  if (io.launches) *io.launches += 2;
  if (io.nranks > 1) {
    ncclResult_t r = ncclAllReduce(io.comm + fk2 + 1, io.comm + fk2 + 1, 1, ncclDouble, ncclSum,
                                   io.nccl, io.stream);
    if (r != ncclSuccess) { err = std::string("ncclAllReduce: ") + ncclGetErrorString(r); return -1; }
    if (io.launches) *io.launches += 1;
  }
  const double kn = double(io.K) * double(io.nranks > 1 ? io.n_global : io.N);
  if (fs->tc3) {
    // the pair accumulates Num_W and Den_W in fp32 TMEM folds; their difference is not a
    // usable gradient once they agree to a few digits, so grad_W gets its own W-side pass with
    // the gradient core formed per element (FusedArgs::kkt == 2)
    FusedArgs g = make_args(fs, io, 1);
    g.kkt = 2;
    FCK(launch_pass(fs, g, io, slot, -1));
    fused_reduce<<<int((fk2 + 1 + 255) / 256), 256, 0, io.stream>>>(
        fs->part, fs->opart, fs->t3_gx, fs->t3_gx * fs->t3_r, int(fk2), io.K, io.F, 1, fs->kcomm,
        io.st, slot, -1);
    FCK(cudaGetLastError());
    if (io.launches) *io.launches += 2;
    if (io.nranks > 1) {
      ncclResult_t r = ncclAllReduce(fs->kcomm, fs->kcomm, fk2 / 2, ncclDouble, ncclSum, io.nccl,
                                     io.stream);
      if (r != ncclSuccess) { err = std::string("ncclAllReduce: ") + ncclGetErrorString(r); return -1; }
      if (io.launches) *io.launches += 1;
    }
    kkt_finish_g<<<1, 1024, 0, io.stream>>>(fs->kcomm, io.comm + fk2 + 1, wp, io.F, io.K, kn,
                                            io.tr_kkt, io.st, slot);
  } else {
    kkt_finish<<<1, 1024, 0, io.stream>>>(io.comm, wp, io.F, io.K, kn, io.tr_kkt, io.st, slot);
  }
  FCK(cudaGetLastError());
  if (io.launches) *io.launches += 1;
  return 0;
}

bool fused_shape_matches(const FusedState* fs, int F, int N, int K) {
  return fs && fs->F == F && fs->N == N && fs->K == K && (!fs->tc || (fs->cap == env_cluster_cap() && fs->v1 == env_tc_v1())) &&
         (fs->tc || fs->tc3 == tc3_wanted(K)) && (!fs->tc || !env_force_pair());
}

void fused_info(const FusedState* fs, int* out4) {
  out4[0] = fs ? ((fs->tc || fs->tc3) ? 2 : 1) : 0;
  out4[1] = fs ? (fs->tc ? fs->tc_grid : (fs->tc3 ? fs->t3_gx * fs->t3_r : fs->s2_S * fs->s2_rc)) : 0;
  out4[2] = fs ? (fs->tc ? fs->tc_cl : 1) : 0;
  out4[3] = fs ? (fs->tc ? fs->tc_f0 : fs->F) : 0;
}

int fused_begin(FusedState* fs, const FusedIO& io, std::string& err) {
  fs->bc = beta_class(io.sc.beta);
  size_t fk = size_t(io.F) * io.K, nk = size_t(io.N) * io.K;
  // iterate 0 = the raw init: W~_0 = W0 (engine Wt), H~_0 = H0 (engine Ht)
  FCK(cudaMemcpyAsync(fs->W2[0], io.Wt, fk * sizeof(float), cudaMemcpyDeviceToDevice, io.stream));
  FCK(cudaMemcpyAsync(fs->H[0], io.Ht, nk * sizeof(float), cudaMemcpyDeviceToDevice, io.stream));
  // prologue: W-side sums of iteration 1 from Vt_0 = W0 H0 + kappa
  FusedIO pio = io;
  pio.ev_a = pio.ev_b = nullptr;
  pio.launches = nullptr;
  int rc = enqueue_pass_and_update(fs, pio, 0, 0, false, err);
  if (rc) return rc;
  FCK(cudaStreamSynchronize(io.stream));
  return 0;
}

int fused_enqueue_iteration(FusedState* fs, const FusedIO& io, int slot, std::string& err) {
  if (int rc = enqueue_pass_and_update(fs, io, slot, -1, true, err)) return rc;
  if (io.compute_kkt) return enqueue_kkt(fs, io, slot, err);
  return 0;
}

// Copy the iterate of parity(iters_done) into the engine's Wt / Ht.
__global__ void select_iterate(const RunState* st, const float* W0, const float* W1,
                               const float* H0, const float* H1, float* Wt, float* Ht,
                               size_t fk, size_t nk) {
  int par = int(st->iters_done & 1);
  const float* W = par ? W1 : W0;
  const float* H = par ? H1 : H0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < fk + nk;
       i += (size_t)gridDim.x * blockDim.x) {
    if (i < fk) Wt[i] = W[i];
    else Ht[i - fk] = H[i - fk];
  }
}

int fused_select(FusedState* fs, const FusedIO& io, std::string& err) {
  size_t fk = size_t(io.F) * io.K, nk = size_t(io.N) * io.K;
  int blocks = int(std::min<size_t>((fk + nk + 255) / 256, 148 * 8));
  select_iterate<<<blocks, 256, 0, io.stream>>>(io.st, fs->W2[0], fs->W2[1], fs->H[0], fs->H[1],
                                                io.Wt, io.Ht, fk, nk);
  FCK(cudaGetLastError());
  if (io.launches) *io.launches += 1;
  return 0;
}

int fused_export(FusedState* fs, const FusedIO& io, std::string& err) {
  FusedIO o = io;
  o.launches = nullptr;
  if (fused_select(fs, o, err)) return -1;
  FCK(cudaStreamSynchronize(io.stream));
  return 0;
}

}  // namespace bnmf

// Bring-up aid (not part of include/bnmf.h): copy the wait-cycle counters of
// the last tcgen05 pass (BNMF_TC_PROF=1) to the host; returns the count.
extern "C" int bnmf_tc_prof_read(long long* out, int max) {
  bnmf::FusedState* fs = bnmf::g_last_tc;
  if (!fs || !fs->prof) return 0;
  int n = std::min(max, int(fs->prof_n));
  if (cudaMemcpy(out, fs->prof, size_t(n) * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return n;
}
