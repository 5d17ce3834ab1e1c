// libbnmf: context, device buffers, the per-iteration schedule and the C ABI.
//
// The outer loop of the reference (solver.py:292-326) runs here, natively:
// every iteration is a fixed sequence of kernels on one stream, captured into
// CUDA graphs in chunks; the stop rule (solver.py:174-180) is evaluated on the
// device, so the host only synchronises once per chunk.
//
// Two schedules compute the same iterates:
//  * reference order (SIMT kernels, any dtype / beta / sub-iteration count):
//    W-side pass -> W update -> H-side pass -> objective pass -> normalise,
//    exactly the data flow of solver.py:239-280 / 292-319;
//  * fused single-read pass (fp32, L = 1; fused_tc.cu): one pass over V per
//    iteration finishes the H update of iteration t, forms the objective of
//    iterate t and the W-side sums of iteration t+1.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/bnmf.h"
#include "bnmf_common.cuh"
#include "engine.h"
#include "simt_kernels.cuh"
#include "small_kernels.cuh"

using namespace bnmf;

static thread_local std::string g_err;

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      return fail(BNMF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                             \
  } while (0)

#define CKN(call)                                                                 \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess) {                                                      \
      return fail(BNMF_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    }                                                                             \
  } while (0)

namespace bnmf {

// Host memcpy split over up to 8 threads (large pageable result / init arrays:
// the copy and its first-touch page faults are spread over cores).
static void par_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t per_min = size_t(4) << 20;
  const int nt = int(std::min<size_t>(8, std::max<size_t>(1, bytes / per_min)));
  if (nt <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + nt - 1) / nt;
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) {
    const size_t a = size_t(t) * per;
    if (a >= bytes) break;
    const size_t n = std::min(per, bytes - a);
    th.emplace_back([=] { memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, n); });
  }
  memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

int EngineBase::fail(int code, const std::string& msg) {
  err = msg;
  g_err = msg;
  return code;
}

static inline int grid_for(size_t count, int threads = 256) {
  size_t b = (count + threads - 1) / threads;
  return int(std::min<size_t>(std::max<size_t>(b, 1), 148 * 8));
}

template <typename T>
struct Engine : EngineBase {
  // sizes
  int F = 0, N = 0, K = 0;
  size_t ldv = 0;
  // data and factors (device)
  T* V = nullptr;
  T *Wt = nullptr, *Wc = nullptr, *Ht = nullptr, *Hc = nullptr;
  T *C1h = nullptr, *C2h = nullptr, *C1w = nullptr, *C2w = nullptr;
  // reduction buffers (device, fp64)
  double *wpart = nullptr, *comm = nullptr, *opart = nullptr, *hpart = nullptr;
  double *norms = nullptr, *colsum = nullptr;
  double *tr_obj = nullptr, *tr_sec = nullptr, *tr_kkt = nullptr;
  int64_t tr_cap = 0;
  RunState* st = nullptr;
  RunState* st_host = nullptr;
  void* staging = nullptr;
  size_t staging_bytes = 0;
  // pinned bounce buffers (2 x HB_CHUNK) for pageable host <-> device copies
  static constexpr size_t HB_CHUNK = size_t(32) << 20;
  char* hbounce = nullptr;
  cudaEvent_t hb_ev[2] = {nullptr, nullptr};
  double* fstats = nullptr;   // min / max / sum / non-finite of the uploaded factors
  // schedule
  int S = 1, seg_cols = 32;
  int S_obj = 1, seg_cols_obj = 32;   // the objective pass's own column segments
  int n_hblocks = 1, n_oblocks = 1;
  int num_sms = 148;
  bnmf_params p{};
  Scalars sc{};
  int bc = BC_GEN;
  int L = 1, Lw = 1, Lh = 1;
  bool begun = false;
  // fp64 JMM: Z tiles of the W-side pass kept for the H-side pass of the same outer iteration
  // (F x ldz each; allocated when they fit ZSHARE_MAX_BYTES), zs_use: 1 = write, 2 = read
  static constexpr size_t ZSHARE_MAX_BYTES = size_t(1) << 30;
  T* Zgn = nullptr;
  T* Zgd = nullptr;
  size_t ldz = 0;
  int zs_use = 0;
  bool chi_h_valid = false;   // C1h / C2h hold chi(H~, H~) of the live iterate (reference-order JMM)
  cudaGraphExec_t gexec = nullptr;
  int gchunk = 0;
  int launches = 0;
  int counting = 0;
  FusedState* fused = nullptr;
  // CUDA events around the dominant kernel of each graph slot (bench roofline)
  static constexpr int kChunk = 16;
  cudaEvent_t ev_a[kChunk] = {}, ev_b[kChunk] = {};
  bool prof = false;
  int prof_slots = 0;

  explicit Engine(int dev, int dt) {
    device = dev;
    dtype = dt;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0) num_sms = n;
  }

  int prof_mark(bool start, int slot) {
    if (!prof || slot >= kChunk) return 0;
    CK(record_event(start ? ev_a[slot] : ev_b[slot], stream));
    if (!start) prof_slots = std::max(prof_slots, slot + 1);
    return 0;
  }

  ~Engine() override {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (int i = 0; i < kChunk; ++i) {
      if (ev_a[i]) cudaEventDestroy(ev_a[i]);
      if (ev_b[i]) cudaEventDestroy(ev_b[i]);
    }
    T* tp[] = {V, Wt, Wc, Ht, Hc, C1h, C2h, C1w, C2w, Zgn, Zgd};
    for (T* q : tp) if (q) cudaFree(q);
    double* dp[] = {wpart, comm, opart, hpart, norms, colsum, tr_obj, tr_sec, tr_kkt};
    for (double* q : dp) if (q) cudaFree(q);
    if (st) cudaFree(st);
    if (st_host) cudaFreeHost(st_host);
    if (staging) cudaFree(staging);
    if (hbounce) cudaFreeHost(hbounce);
    for (cudaEvent_t e : hb_ev) if (e) cudaEventDestroy(e);
    if (fstats) cudaFree(fstats);
    if (stats_part) cudaFree(stats_part);
    if (stats_acc) cudaFree(stats_acc);
    if (fused) fused_destroy(fused);
    if (comm_nccl) ncclCommDestroy(comm_nccl);
    if (stream) cudaStreamDestroy(stream);
  }

  int init() {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&st, sizeof(RunState)));
    CK(cudaMallocHost(&st_host, sizeof(RunState)));
    return 0;
  }

  int ensure_staging(size_t bytes) {
    if (bytes <= staging_bytes) return 0;
    if (staging) CK(cudaFree(staging));
    CK(cudaMalloc(&staging, bytes));
    staging_bytes = bytes;
    return 0;
  }

  int ensure_bounce() {
    if (hbounce) return 0;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&hbounce), 2 * HB_CHUNK, cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&hb_ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&hb_ev[1], cudaEventDisableTiming));
    return 0;
  }

  // pageable host -> device through the pinned bounce buffers: the host copy
  // of chunk c overlaps the DMA of chunk c-1 (a direct pageable copy runs at
  // a fraction of the link rate)
  int h2d_bounce(void* dst, const void* src, size_t bytes) {
    if (bytes < 2 * HB_CHUNK) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
      return 0;
    }
    if (int rc = ensure_bounce()) return rc;
    const size_t nch = (bytes + HB_CHUNK - 1) / HB_CHUNK;
    for (size_t c = 0; c < nch; ++c) {
      const int b = int(c & 1);
      const size_t off = c * HB_CHUNK, n = std::min(HB_CHUNK, bytes - off);
      if (c >= 2) CK(cudaEventSynchronize(hb_ev[b]));
      par_memcpy(hbounce + b * HB_CHUNK, static_cast<const char*>(src) + off, n);
      CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, hbounce + b * HB_CHUNK, n,
                         cudaMemcpyHostToDevice, stream));
      CK(cudaEventRecord(hb_ev[b], stream));
    }
    CK(cudaStreamSynchronize(stream));
    return 0;
  }

  // device -> pageable host, the mirror image: the DMA of chunk c+1 overlaps
  // the host copy of chunk c
  int d2h_bounce(void* dst, const void* src, size_t bytes) {
    if (bytes < 2 * HB_CHUNK) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      return 0;
    }
    if (int rc = ensure_bounce()) return rc;
    const size_t nch = (bytes + HB_CHUNK - 1) / HB_CHUNK;
    auto issue = [&](size_t c) -> cudaError_t {
      const size_t off = c * HB_CHUNK, n = std::min(HB_CHUNK, bytes - off);
      cudaError_t e = cudaMemcpyAsync(hbounce + (c & 1) * HB_CHUNK,
                                      static_cast<const char*>(src) + off, n,
                                      cudaMemcpyDeviceToHost, stream);
      return e != cudaSuccess ? e : cudaEventRecord(hb_ev[c & 1], stream);
    };
    CK(issue(0));
    for (size_t c = 0; c < nch; ++c) {
      if (c + 1 < nch) CK(issue(c + 1));
      CK(cudaEventSynchronize(hb_ev[c & 1]));
      const size_t off = c * HB_CHUNK, n = std::min(HB_CHUNK, bytes - off);
      par_memcpy(static_cast<char*>(dst) + off, hbounce + (c & 1) * HB_CHUNK, n);
    }
    return 0;
  }

  // statistics of a rows x cols source block, accumulated into stats_acc
  double* stats_part = nullptr;
  double* stats_acc = nullptr;
  int64_t stats_count = 0;
  template <typename S_>
  int stats_of(const S_* src, size_t lds, int rows, size_t cols, bool first) {
    if (!stats_acc) CK(cudaMalloc(&stats_acc, 4 * sizeof(double)));
    return stats_into(src, lds, rows, cols, first, stats_acc);
  }
  template <typename S_>
  int stats_into(const S_* src, size_t lds, int rows, size_t cols, bool first, double* acc) {
    if (!stats_part) CK(cudaMalloc(&stats_part, STATS_BLOCKS * 4 * sizeof(double)));
    stats_partial<S_><<<STATS_BLOCKS, 256, 0, stream>>>(src, lds, rows, cols, stats_part);
    stats_final<<<1, 32, 0, stream>>>(stats_part, STATS_BLOCKS, acc, first ? 1 : 0);
    CK(cudaGetLastError());
    return 0;
  }
  int data_stats(double* out5) override {
    if (!stats_acc) return fail(BNMF_E_STATE, "no dense data");
    CK(cudaSetDevice(device));
    CK(cudaMemcpyAsync(out5, stats_acc, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    out5[4] = double(stats_count);
    return 0;
  }

  template <typename S_>
  int convert_in(const void* src, size_t lds, int rows, size_t cols, double kappa, int on_dev) {
    const size_t chunk_bytes = size_t(256) << 20;
    if (on_dev) {
      if (int rc = stats_of(reinterpret_cast<const S_*>(src), lds, rows, cols, true)) return rc;
      convert_rows<S_, T><<<grid_for(size_t(rows) * cols), 256, 0, stream>>>(
          reinterpret_cast<const S_*>(src), lds, V, ldv, rows, cols, kappa);
      CK(cudaGetLastError());
      return 0;
    }
    int rpc = int(std::max<size_t>(1, chunk_bytes / (cols * sizeof(S_))));
    rpc = std::min(rpc, rows);
    if (int rc = ensure_staging(size_t(rpc) * cols * sizeof(S_))) return rc;
    // one stream orders copy(c+1) after convert(c), so the staging buffer is
    // reused without host syncs and the link stays busy; contiguous rows
    // (lds == cols) go as one linear copy
    for (int r0 = 0; r0 < rows; r0 += rpc) {
      int nr = std::min(rpc, rows - r0);
      const S_* s0 = reinterpret_cast<const S_*>(src) + size_t(r0) * lds;
      if (lds == cols)
        CK(cudaMemcpyAsync(staging, s0, size_t(nr) * cols * sizeof(S_), cudaMemcpyHostToDevice,
                           stream));
      else
        CK(cudaMemcpy2DAsync(staging, cols * sizeof(S_), s0, lds * sizeof(S_),
                             cols * sizeof(S_), nr, cudaMemcpyHostToDevice, stream));
      if (int rc = stats_of(reinterpret_cast<const S_*>(staging), cols, nr, cols, r0 == 0)) return rc;
      convert_rows<S_, T><<<grid_for(size_t(nr) * cols), 256, 0, stream>>>(
          reinterpret_cast<const S_*>(staging), cols, V + size_t(r0) * ldv, ldv, nr, cols,
          kappa);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(stream));
    return 0;
  }

  int set_dense(const void* v, int src_dtype, int on_dev, int64_t F_, int64_t N_, int64_t ld,
                double kappa) override {
    if (F_ < 1 || N_ < 1 || ld < N_) return fail(BNMF_E_ARG, "bad matrix shape");
    if (F_ > INT_MAX / 2 || N_ > INT_MAX / 2) return fail(BNMF_E_ARG, "matrix too large");
    CK(cudaSetDevice(device));
    if (V) { CK(cudaFree(V)); V = nullptr; }
    F = int(F_); N = int(N_);
    ldv = (size_t(N) + 3) & ~size_t(3);
    CK(cudaMalloc(&V, size_t(F) * ldv * sizeof(T)));
    if (ldv != size_t(N)) CK(cudaMemsetAsync(V, 0, size_t(F) * ldv * sizeof(T), stream));
    int rc;
    stats_count = int64_t(F) * N;
    if (!on_dev && src_dtype == dtype && kappa == 0.0) {
      if (size_t(ld) == ldv)   // contiguous rows: one linear copy
        CK(cudaMemcpyAsync(V, v, size_t(F) * ldv * sizeof(T), cudaMemcpyHostToDevice, stream));
      else
        CK(cudaMemcpy2DAsync(V, ldv * sizeof(T), v, size_t(ld) * sizeof(T),
                             size_t(N) * sizeof(T), F, cudaMemcpyHostToDevice, stream));
      rc = stats_of(V, ldv, F, size_t(N), true);
    } else if (src_dtype == BNMF_FP64) {
      rc = convert_in<double>(v, size_t(ld), F, size_t(N), kappa, on_dev);
    } else {
      rc = convert_in<float>(v, size_t(ld), F, size_t(N), kappa, on_dev);
    }
    if (rc) return rc;
    CK(cudaStreamSynchronize(stream));
    begun = false;
    if (fused) { fused_destroy(fused); fused = nullptr; }
    return 0;
  }

  int aF = 0, aN = 0;
  int alloc_factors(int K_) {
    if (K == K_ && F == aF && N == aN && Wt) return 0;
    T** tp[] = {&Wt, &Wc, &Ht, &Hc, &C1h, &C2h, &C1w, &C2w, &Zgn, &Zgd};
    for (T** q : tp) if (*q) { CK(cudaFree(*q)); *q = nullptr; }
    double** dp[] = {&wpart, &comm, &opart, &hpart, &norms, &colsum};
    for (double** q : dp) if (*q) { CK(cudaFree(*q)); *q = nullptr; }
    K = K_;
    aF = F; aN = N;
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    CK(cudaMalloc(&Wt, fk * sizeof(T)));
    CK(cudaMalloc(&Wc, fk * sizeof(T)));
    CK(cudaMalloc(&C1w, fk * sizeof(T)));
    CK(cudaMalloc(&C2w, fk * sizeof(T)));
    CK(cudaMalloc(&Ht, nk * sizeof(T)));
    CK(cudaMalloc(&Hc, nk * sizeof(T)));
    CK(cudaMalloc(&C1h, nk * sizeof(T)));
    CK(cudaMalloc(&C2h, nk * sizeof(T)));
    // segments of the W-side / objective passes: ~4 CTAs per SM
    int ftiles = (F + ST_TF - 1) / ST_TF;
    int ctiles = (N + ST_NC - 1) / ST_NC;
    // (fp64: the DMMA passes hold ~125 registers and ~100 KB of stages, two CTAs per SM, and a
    // grid beyond one wave only adds a tail)
    int cps = std::is_same<T, double>::value ? 2 : 4;
    if (const char* e = getenv("BNMF_WSIDE_CPS")) cps = std::max(1, atoi(e));
    S = std::max(1, std::min(ctiles, (cps * num_sms + ftiles - 1) / ftiles));
    seg_cols = ((N + S - 1) / S + ST_NC - 1) / ST_NC * ST_NC;
    S = (N + seg_cols - 1) / seg_cols;
    n_hblocks = ctiles;
    // the objective pass is lighter (64 registers, one H~ stage): finer segments in fp64
    {
      int cpo = std::is_same<T, double>::value ? 4 : cps;
      if (const char* e = getenv("BNMF_OBJ_CPS")) cpo = std::max(1, atoi(e));
      S_obj = std::max(1, std::min(ctiles, (cpo * num_sms + ftiles - 1) / ftiles));
      seg_cols_obj = ((N + S_obj - 1) / S_obj + ST_NC - 1) / ST_NC * ST_NC;
      S_obj = (N + seg_cols_obj - 1) / seg_cols_obj;
    }
    n_oblocks = ftiles * S_obj;
    CK(cudaMalloc(&wpart, size_t(S) * 2 * fk * sizeof(double)));
    CK(cudaMalloc(&comm, (2 * fk + 8) * sizeof(double)));
    CK(cudaMalloc(&opart, size_t(std::max(n_oblocks, n_hblocks)) * sizeof(double)));
    CK(cudaMalloc(&hpart, size_t(n_hblocks) * sizeof(double)));
    CK(cudaMalloc(&norms, size_t(K) * sizeof(double)));
    CK(cudaMalloc(&colsum, size_t(K) * sizeof(double)));
    // fp64: room for the Z tiles the W-side pass hands to the H-side pass (JMM); large inputs
    // recompute them instead
    ldz = (size_t(N) + 3) / 4 * 4;
    if (std::is_same<T, double>::value && getenv("BNMF_NO_ZSHARE") == nullptr &&
        2 * size_t(F) * ldz * sizeof(T) <= ZSHARE_MAX_BYTES) {
      CK(cudaMalloc(&Zgn, size_t(F) * ldz * sizeof(T)));
      CK(cudaMalloc(&Zgd, size_t(F) * ldz * sizeof(T)));
    }
    return 0;
  }

  int set_factors(const double* w, const double* h, int64_t K_, int on_dev) override {
    if (!V) return fail(BNMF_E_STATE, "set_dense must precede set_factors");
    if (K_ < 1) return fail(BNMF_E_ARG, "rank must be positive");
    CK(cudaSetDevice(device));
    chi_h_valid = false;
    if (int rc = alloc_factors(int(K_))) return rc;
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    if (int rc = ensure_staging(std::max(fk, nk) * sizeof(double))) return rc;
    double* stg = reinterpret_cast<double*>(staging);
    if (!fstats) CK(cudaMalloc(&fstats, 4 * sizeof(double)));
    const double* wsrc = w;
    if (!on_dev) {
      if (int rc = h2d_bounce(stg, w, fk * sizeof(double))) return rc;
      wsrc = stg;
    }
    // the FactorPair checks (core.py:__post_init__ of the reference's
    // FactorPair) on the device copy, so large inits need no host scan
    if (int rc = stats_into(wsrc, fk, 1, fk, true, fstats)) return rc;
    from_double<T><<<grid_for(fk), 256, 0, stream>>>(wsrc, fk, Wt);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(stream));
    const double* hsrc = h;
    if (!on_dev) {
      if (int rc = h2d_bounce(stg, h, nk * sizeof(double))) return rc;
      hsrc = stg;
    }
    if (int rc = stats_into(hsrc, nk, 1, nk, false, fstats)) return rc;
    transpose_in<T><<<grid_for(nk), 256, 0, stream>>>(hsrc, K, size_t(N), Ht);
    CK(cudaGetLastError());
    double fs[4];
    CK(cudaMemcpyAsync(fs, fstats, sizeof(fs), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    begun = false;
    if (fs[3] > 0.0) return fail(BNMF_E_ARG, "factor entries must be finite");
    if (fs[0] <= 0.0) return fail(BNMF_E_ARG, "factor entries must be strictly positive");
    return 0;
  }

  int get_factors(double* w, double* h) override {
    if (!Wt) return fail(BNMF_E_STATE, "no factors");
    CK(cudaSetDevice(device));
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    if (int rc = ensure_staging(std::max(fk, nk) * sizeof(double))) return rc;
    double* stg = reinterpret_cast<double*>(staging);
    if (fused && fused_active) {
      if (fused_export(fused, io(), err)) return fail(BNMF_E_CUDA, err);
    }
    to_double<T><<<grid_for(fk), 256, 0, stream>>>(Wt, fk, stg);
    CK(cudaGetLastError());
    if (int rc = d2h_bounce(w, stg, fk * sizeof(double))) return rc;
    transpose_out<T><<<grid_for(nk), 256, 0, stream>>>(Ht, K, size_t(N), stg);
    CK(cudaGetLastError());
    return d2h_bounce(h, stg, nk * sizeof(double));
  }

  // ------------------------------------------------------------------------
  // kernel dispatch helpers

  size_t smem_wside() const {
    int ks = kstride(K);
    return size_t(ST_TF * ks + hside_nbuf() * 3 * ST_NC * ks + 2 * ST_TF * (ST_NC + 1)) * sizeof(T);
  }
  // the fp64 passes double-buffer their row / column stage when two copies fit
  int hside_nbuf() const {
    if (!std::is_same<T, double>::value) return 1;
    int ks = kstride(K);
    return size_t(ST_NC * ks + 6 * ST_TF * ks + 2 * ST_TF * (ST_NC + 1)) * sizeof(T) <= 200 * 1024 ? 2 : 1;
  }
  // CTAs per column block of the fp64 H-side pass: with fewer column blocks than SMs the pass is
  // bound by the latency of one block's walk over all F rows, so the rows are split over a
  // cluster (the largest of 4, 3, 2 that still fits two CTAs per SM and leaves >= 2 tiles each)
  int hside_cluster() const {
    if (!std::is_same<T, double>::value) return 1;
    if (const char* e = getenv("BNMF_HSIDE_CLUSTER")) return std::min(8, std::max(1, atoi(e)));
    const int ntile = (F + ST_TF - 1) / ST_TF;
    for (int c : {4, 3, 2})
      if (n_hblocks * c <= 2 * num_sms && ntile >= 2 * c) return c;
    return 1;
  }
  size_t smem_hside() const {
    int ks = kstride(K);
    return size_t(ST_NC * ks + hside_nbuf() * 3 * ST_TF * ks + 2 * ST_TF * (ST_NC + 1)) * sizeof(T);
  }
  size_t smem_obj() const { return size_t((ST_TF + 2 * ST_NC) * kstride(K)) * sizeof(T); }   // two H~ stages (fp64)

  template <int BC, int MODE>
  int launch_wside(const T* Wp, const T* Hp, const T* C1, const T* C2, int slot) {
    auto kern = wside_partials<BC, MODE, T>;
    size_t sm = smem_wside();
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    dim3 grid((F + ST_TF - 1) / ST_TF, S);
    T* zn = (zs_use == 1 && MODE == PM_UPDATE) ? Zgn : nullptr;
    T* zd = (zn && bc != BC_1) ? Zgd : nullptr;
    kern<<<grid, ST_THREADS, sm, stream>>>(V, ldv, F, N, K, Wp, Hp, C1, C2, seg_cols, sc,
                                           wpart, hside_nbuf(), st, slot, zn, zd, ldz);
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  template <int BC, int MODE>
  int launch_hside(const T* Wp, const T* Hp, const T* C1, const T* C2, const T* Hb, T* Ho,
                   int den_ones, int slot) {
    auto kern = hside_pass<BC, MODE, T>;
    size_t sm = smem_hside();
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    const int cs = hside_cluster();
    const T* zn = (zs_use == 2 && MODE == PM_UPDATE) ? Zgn : nullptr;
    const T* zd = (zn && bc != BC_1) ? Zgd : nullptr;
    size_t ldz_ = ldz;
    if (cs > 1) {
      // few column blocks (fp64): the rows of a block are split over a cluster of cs CTAs
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(n_hblocks * cs));
      cfg.blockDim = dim3(ST_THREADS);
      cfg.dynamicSmemBytes = sm;
      cfg.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(cs);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const T* Vc = V;
      const double* csum = colsum;
      int nb = hside_nbuf();
      const RunState* stc = st;
      CK(cudaLaunchKernelEx(&cfg, kern, Vc, ldv, F, N, K, Wp, Hp, C1, C2, Hb, Ho, csum, den_ones,
                            sc, hpart, nb, stc, slot, zn, zd, ldz_));
    } else {
      kern<<<n_hblocks, ST_THREADS, sm, stream>>>(V, ldv, F, N, K, Wp, Hp, C1, C2, Hb, Ho, colsum,
                                                  den_ones, sc, hpart, hside_nbuf(), st, slot, zn,
                                                  zd, ldz_);
    }
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  template <int BC>
  int launch_obj(const T* W, const T* H, int slot) {
    auto kern = objective_partials<BC, T>;
    size_t sm = smem_obj();
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    dim3 grid((F + ST_TF - 1) / ST_TF, S_obj);
    kern<<<grid, ST_THREADS, sm, stream>>>(V, ldv, F, N, K, W, H, seg_cols_obj, sc, opart, st, slot);
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  int wside(int mode, const T* Wp, const T* Hp, const T* C1, const T* C2, int slot) {
#define WS(B)                                                              \
  case B:                                                                  \
    return mode == PM_KKT ? launch_wside<B, PM_KKT>(Wp, Hp, C1, C2, slot)  \
                          : launch_wside<B, PM_UPDATE>(Wp, Hp, C1, C2, slot);
    switch (bc) { WS(BC_GEN) WS(BC_0) WS(BC_1) WS(BC_2) }
#undef WS
    return fail(BNMF_E_ARG, "beta class");
  }
  int hside(int mode, const T* Wp, const T* Hp, const T* C1, const T* C2, const T* Hb, T* Ho,
            int den_ones, int slot) {
#define HS(B)                                                                        \
  case B:                                                                            \
    return mode == PM_KKT                                                            \
               ? launch_hside<B, PM_KKT>(Wp, Hp, C1, C2, Hb, Ho, den_ones, slot)     \
               : launch_hside<B, PM_UPDATE>(Wp, Hp, C1, C2, Hb, Ho, den_ones, slot);
    switch (bc) { HS(BC_GEN) HS(BC_0) HS(BC_1) HS(BC_2) }
#undef HS
    return fail(BNMF_E_ARG, "beta class");
  }
  int objective(const T* W, const T* H, int slot) {
    switch (bc) {
      case BC_GEN: return launch_obj<BC_GEN>(W, H, slot);
      case BC_0: return launch_obj<BC_0>(W, H, slot);
      case BC_1: return launch_obj<BC_1>(W, H, slot);
      case BC_2: return launch_obj<BC_2>(W, H, slot);
    }
    return fail(BNMF_E_ARG, "beta class");
  }

  int allreduce(double* buf, size_t count) {
    if (nranks > 1) {
      CKN(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_nccl, stream));
      launches += 1;
    }
    return 0;
  }

  // W-side: partials -> segment reduction -> (allreduce) -> update
  // c1o / c2o (optional): chi maps of the new W against `base` (the JMM H-side factors)
  int w_update(const T* Wp, const T* Hp, const T* C1, const T* C2, const T* base, T* out,
               int slot, T* c1o = nullptr, T* c2o = nullptr) {
    size_t fk = size_t(F) * K;
    if (int rc = wside(PM_UPDATE, Wp, Hp, C1, C2, slot)) return rc;
    if (nranks == 1) {
      // one rank: segment reduction, update and chi maps in one launch
      reduce_update_w<T><<<grid_for(fk, 64), 64, 0, stream>>>(wpart, 2 * fk, S, base, F, K, out, c1o,
                                                          c2o, comm, sc, st, slot);
      CK(cudaGetLastError());
      launches += 1;
      return 0;
    }
    reduce_segments<<<grid_for(2 * fk), 256, 0, stream>>>(wpart, 2 * fk, S, 2 * fk, comm, st,
                                                           slot);
    CK(cudaGetLastError());
    launches += 1;
    if (int rc = allreduce(comm, 2 * fk)) return rc;
    update_w<T><<<grid_for(fk), 256, 0, stream>>>(base, comm, comm + fk, 0, F, K, out, sc, st,
                                                   slot);
    CK(cudaGetLastError());
    launches += 1;
    if (c1o) return chi(out, base, c1o, c2o, fk, slot);
    return 0;
  }

  int chi(const T* M, const T* Mt, T* o1, T* o2, size_t count, int slot) {
    chi_maps<T><<<grid_for(count), 256, 0, stream>>>(M, Mt, o1, o2, count, sc, st, slot);
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  int colsums(const T* M, int slot) {
    // fp64: hside_pass adds the columns of its C2 operand itself (same row order)
    if (std::is_same<T, double>::value) return 0;
    // K <= 128 (the engine's rank cap) < CS_THREADS
    const size_t row_bytes = size_t(K) * sizeof(T);
    const int rows = int(std::max<size_t>(1, std::min<size_t>(size_t(F), CS_SMEM_MAX / row_bytes)));
    const size_t smem = size_t(rows) * row_bytes;
    static bool attr_set = false;
    if (!attr_set) {
      CK(cudaFuncSetAttribute(col_sums<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              int(CS_SMEM_MAX)));
      attr_set = true;
    }
    col_sums<T><<<1, CS_THREADS, smem, stream>>>(M, F, K, colsum, rows, st, slot);
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  // One outer iteration in reference order (solver.py:239-280, 301-319).
  int enqueue_reference_iteration(int slot) {
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    int den_ones = (bc == BC_1) ? 1 : 0;
    begin_iter<<<1, 1, 0, stream>>>(st, slot);
    CK(cudaGetLastError());
    launches += 1;
    int rc;
    if (p.algorithm == BNMF_JMM) {
      for (int l = 0; l < L; ++l) {
        // chi maps of the moving H against the anchor (updates.py:217-218)
        // (at l == 0 they are chi(H~, H~), written by scale_h_chi of the previous iteration
        // or by step() before the first one)
        if (l > 0 && (rc = chi(Hc, Ht, C1h, C2h, nk, slot))) return rc;
        // fp64: the W-side pass leaves Z (same anchor for both updates of a JMM iteration) in
        // global memory for the H-side pass
        zs_use = Zgn ? 1 : 0;
        rc = w_update(Wt, Ht, C1h, C2h, Wt, Wc, slot, C1w, C2w);
        zs_use = 0;
        if (rc) return rc;
        if (den_ones && (rc = colsums(C2w, slot))) return rc;
        if (l == 0 && (rc = prof_mark(true, slot))) return rc;
        zs_use = Zgn ? 2 : 0;
        rc = hside(PM_UPDATE, Wt, Ht, C1w, C2w, Ht, Hc, den_ones, slot);
        zs_use = 0;
        if (rc) return rc;
        if (l == 0 && (rc = prof_mark(false, slot))) return rc;
      }
    } else {
      for (int l = 0; l < Lw; ++l) {
        const T* wcur = l == 0 ? Wt : Wc;
        if ((rc = w_update(wcur, Ht, Ht, Ht, wcur, Wc, slot))) return rc;
      }
      for (int l = 0; l < Lh; ++l) {
        const T* hcur = l == 0 ? Ht : Hc;
        if (den_ones && (rc = colsums(Wc, slot))) return rc;
        if (l == 0 && (rc = prof_mark(true, slot))) return rc;
        if ((rc = hside(PM_UPDATE, Wc, hcur, Wc, Wc, hcur, Hc, den_ones, slot))) return rc;
        if (l == 0 && (rc = prof_mark(false, slot))) return rc;
      }
    }
    // objective of the unnormalised new iterate (solver.py:304-309)
    if ((rc = objective(Wc, Hc, slot))) return rc;
    double* obj = comm + 2 * fk;
    if (nranks > 1) {
      sum_small<<<1, 1024, 0, stream>>>(opart, n_oblocks, obj, st, slot);
      CK(cudaGetLastError());
      launches += 1;
      if ((rc = allreduce(obj, 1))) return rc;
    }
    // normalise (solver.py:311, 167-171)
    normalize_w<T><<<K, NW_THREADS, 0, stream>>>(Wc, F, K, Wt, norms, st, slot);
    CK(cudaGetLastError());
    if (p.algorithm == BNMF_JMM)
      scale_h_chi<T><<<grid_for(nk), 256, 0, stream>>>(Hc, size_t(N), K, norms, Ht, C1h, C2h, sc,
                                                      st, slot);
    else
      scale_h<T><<<grid_for(nk), 256, 0, stream>>>(Hc, size_t(N), K, norms, Ht, st, slot);
    CK(cudaGetLastError());
    if (nranks > 1)
      finish_iter<<<1, 1, 0, stream>>>(st, slot, obj, tr_obj, tr_sec, sc.tol);
    else
      finish_iter_sum<<<1, 1024, 0, stream>>>(st, slot, opart, n_oblocks, obj, tr_obj, tr_sec,
                                              sc.tol);
    CK(cudaGetLastError());
    launches += 3;
    if (p.compute_kkt) {
      if ((rc = enqueue_kkt(slot))) return rc;
    }
    return 0;
  }

  // KKT residuals of the normalised iterate (diagnostics.py:46-59), untimed.
  int enqueue_kkt(int slot) {
    size_t fk = size_t(F) * K;
    int rc;
    if ((rc = wside(PM_KKT, Wt, Ht, Ht, Ht, slot))) return rc;
    reduce_segments<<<grid_for(fk), 256, 0, stream>>>(wpart, 2 * fk, S, fk, comm, st, slot);
    CK(cudaGetLastError());
    if ((rc = hside(PM_KKT, Wt, Ht, Wt, Wt, Ht, nullptr, 0, slot))) return rc;
    double* resh = comm + fk;
    sum_small<<<1, 1024, 0, stream>>>(hpart, n_hblocks, resh, st, slot);
    CK(cudaGetLastError());
    launches += 2;
    if ((rc = allreduce(comm, fk + 1))) return rc;
    kkt_w_residual<T><<<1, 1024, 0, stream>>>(Wt, comm, F, K, resh, size_t(K) * n_global, tr_kkt,
                                              st, slot);
    CK(cudaGetLastError());
    launches += 1;
    return 0;
  }

  FusedIO io() {
    FusedIO o;
    if constexpr (std::is_same<T, float>::value) {
      o.F = F; o.N = N; o.K = K; o.ldv = ldv;
      o.V = V; o.Wt = Wt; o.Wc = Wc; o.Ht = Ht; o.Hc = Hc;
      o.comm = comm; o.norms = norms;
      o.tr_obj = tr_obj; o.tr_sec = tr_sec; o.tr_kkt = tr_kkt;
      o.st = st; o.stream = stream; o.sc = sc; o.algorithm = p.algorithm;
      o.compute_kkt = p.compute_kkt; o.nranks = nranks; o.nccl = comm_nccl;
      o.n_global = n_global; o.launches = &launches;
    }
    return o;
  }

  int enqueue_iteration(int slot) {
    if (fused_active) {
      FusedIO o = io();
      if (prof && slot < kChunk) { o.ev_a = ev_a[slot]; o.ev_b = ev_b[slot]; prof_slots = std::max(prof_slots, slot + 1); }
      // KKT residuals (p.compute_kkt) are part of the fused slot: res_W from the reduced
      // W-side sums, res_H from an H-side-only pass (fused_tc.cu, enqueue_kkt)
      if (fused_enqueue_iteration(fused, o, slot, err)) return fail(BNMF_E_CUDA, err);
      return 0;
    }
    return enqueue_reference_iteration(slot);
  }

  // ------------------------------------------------------------------------

  int begin(const bnmf_params* pp, int64_t max_iters) override {
    if (!V || !Wt) return fail(BNMF_E_STATE, "data and factors must be set before begin");
    if (max_iters < 1) return fail(BNMF_E_ARG, "max_iters must be positive");
    if (pp->sub_iters < 1 || pp->sub_iters_w < 0 || pp->sub_iters_h < 0)
      return fail(BNMF_E_ARG, "sub-iteration counts must be positive");
    if (!(pp->floor > 0.0)) return fail(BNMF_E_ARG, "denominator_floor must be positive");
    CK(cudaSetDevice(device));
    CK(cudaStreamSynchronize(stream));
    p = *pp;
    sc.beta = p.beta; sc.gamma = p.gamma; sc.kappa = p.kappa; sc.floor = p.floor; sc.tol = p.tol;
    bc = beta_class(p.beta);
    L = p.sub_iters;
    Lw = p.sub_iters_w > 0 ? p.sub_iters_w : p.sub_iters;
    Lh = p.sub_iters_h > 0 ? p.sub_iters_h : p.sub_iters;
    if (nranks == 1) n_global = N;
    // schedule choice
    bool fused_ok = fused_supported(dtype, F, K, p.algorithm, L, Lw, Lh, p.beta);
    int sched = p.schedule;
    if (sched == BNMF_SCHED_AUTO) sched = fused_ok ? BNMF_SCHED_FUSED : BNMF_SCHED_REFERENCE;
    if (sched == BNMF_SCHED_FUSED && !fused_ok)
      return fail(BNMF_E_UNSUPPORTED, "fused schedule needs fp32, sub_iters == 1 and a supported rank");
    if (sched == BNMF_SCHED_REFERENCE && K > ST_KMAX)
      return fail(BNMF_E_UNSUPPORTED, "rank above 128 is not supported by the reference-order kernels");
    active_schedule = sched;
    // trace buffers
    if (tr_cap < max_iters) {
      double** dp[] = {&tr_obj, &tr_sec, &tr_kkt};
      for (double** q : dp) if (*q) { CK(cudaFree(*q)); *q = nullptr; }
      CK(cudaMalloc(&tr_obj, size_t(max_iters) * sizeof(double)));
      CK(cudaMalloc(&tr_sec, size_t(max_iters) * sizeof(double)));
      CK(cudaMalloc(&tr_kkt, size_t(max_iters) * 2 * sizeof(double)));
      tr_cap = max_iters;
    }
    CK(cudaMemsetAsync(tr_kkt, 0xff, size_t(max_iters) * 2 * sizeof(double), stream));  // NaN
    RunState h{};
    h.base = 1;
    h.stop_iter = LLONG_MAX;
    h.max_iter = max_iters;
    *st_host = h;
    CK(cudaMemcpyAsync(st, st_host, sizeof(RunState), cudaMemcpyHostToDevice, stream));
    if (gexec) { CK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    fused_active = (sched == BNMF_SCHED_FUSED);
    if (fused_active) {
      if (fused && !fused_shape_matches(fused, F, N, K)) { fused_destroy(fused); fused = nullptr; }
      if (!fused && fused_create(&fused, io(), err)) return fail(BNMF_E_CUDA, err);
      if (fused_begin(fused, io(), err)) return fail(BNMF_E_CUDA, err);
    }
    // count the launches of one iteration (dry pass against a throwaway
    // capture, so the graph and the direct path agree)
    CK(cudaStreamSynchronize(stream));
    begun = true;
    chi_h_valid = false;
    return 0;
  }

  int capture(int chunk) {
    if (gexec && gchunk == chunk) return 0;
    if (gexec) { CK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    int l0 = launches;
    int rc = 0;
    for (int j = 0; j < chunk && rc == 0; ++j) rc = enqueue_iteration(j);
    if (rc == 0) {
      advance_base<<<1, 1, 0, stream>>>(st, chunk);
      rc = cudaGetLastError() == cudaSuccess ? 0 : BNMF_E_CUDA;
    }
    cudaError_t ec = cudaStreamEndCapture(stream, &g);
    if (rc) return rc;
    if (ec != cudaSuccess) return fail(BNMF_E_CUDA, std::string("capture: ") + cudaGetErrorString(ec));
    launches_per_iter = (launches - l0) / chunk;
    CK(cudaGraphInstantiate(&gexec, g, 0));
    CK(cudaGraphDestroy(g));
    gchunk = chunk;
    return 0;
  }

  int prepare(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    CK(cudaSetDevice(device));
    if (n >= kChunk) return capture(kChunk);
    return 0;
  }

  int step(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    CK(cudaSetDevice(device));
    if (!fused_active && p.algorithm == BNMF_JMM && !chi_h_valid) {
      // W-side factors chi(H~, H~) of the first iteration; later ones come from scale_h_chi
      if (int rc = chi(Ht, Ht, C1h, C2h, size_t(N) * K, 0)) return rc;
      chi_h_valid = true;
    }
    const int chunk = kChunk;
    int64_t full = n / chunk, rest = n % chunk;
    if (full > 0) {
      if (int rc = capture(chunk)) return rc;
      for (int64_t i = 0; i < full; ++i) CK(cudaGraphLaunch(gexec, stream));
    }
    for (int64_t i = 0; i < rest; ++i) {
      int l0 = launches;
      if (int rc = enqueue_iteration(0)) return rc;
      launches_per_iter = launches - l0;
      advance_base<<<1, 1, 0, stream>>>(st, 1);
      CK(cudaGetLastError());
    }
    return 0;
  }

  int sync(int64_t* done, int* conv) override {
    CK(cudaSetDevice(device));
    CK(cudaMemcpyAsync(st_host, st, sizeof(RunState), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (done) *done = st_host->iters_done;
    if (conv) *conv = st_host->converged;
    return 0;
  }

  int read_trace(double* obj, double* sec, double* kkt, int64_t n) override {
    if (n > tr_cap) return fail(BNMF_E_ARG, "trace request exceeds max_iters");
    CK(cudaSetDevice(device));
    if (obj) CK(cudaMemcpyAsync(obj, tr_obj, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (sec) CK(cudaMemcpyAsync(sec, tr_sec, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (kkt) CK(cudaMemcpyAsync(kkt, tr_kkt, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    return 0;
  }

  int set_profiling(int on) override {
    CK(cudaSetDevice(device));
    if (on && !ev_a[0]) {
      for (int i = 0; i < kChunk; ++i) {
        CK(cudaEventCreate(&ev_a[i]));
        CK(cudaEventCreate(&ev_b[i]));
      }
    }
    prof = on != 0;
    prof_slots = 0;
    if (gexec) { CK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    return 0;
  }

  void pass_info(int* out4) override {
    if (fused_active && fused) fused_info(fused, out4);
    else out4[0] = out4[1] = out4[2] = out4[3] = 0;
  }

  int pass_time(float* ms_avg, int* samples) override {
    CK(cudaStreamSynchronize(stream));
    double tot = 0.0;
    int n = 0;
    for (int i = 0; i < prof_slots; ++i) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev_a[i], ev_b[i]) == cudaSuccess) { tot += t; ++n; }
    }
    cudaGetLastError();
    *ms_avg = n ? float(tot / n) : 0.f;
    *samples = n;
    return 0;
  }

  // One update kernel / diagnostic of the reference's lower-level API (bnmf.h: bnmf_kernel)
  // on the reference-order kernels: slot 0 of a one-iteration run state.
  int kernel_op(int op, const bnmf_params* pp, const double* cur, double* out) override {
    if (!V || !Wt) return fail(BNMF_E_STATE, "data and factors must be set first");
    if (!out) return fail(BNMF_E_ARG, "null output");
    bnmf_params q = *pp;
    q.schedule = BNMF_SCHED_REFERENCE;
    q.compute_kkt = op == BNMF_OP_KKT ? 1 : 0;
    if (int rc = begin(&q, 1)) return rc;
    const size_t fk = size_t(F) * K, nk = size_t(N) * K;
    const int den_ones = (bc == BC_1) ? 1 : 0;
    if (int rc = ensure_staging(std::max(fk, nk) * sizeof(double))) return rc;
    double* stg = reinterpret_cast<double*>(staging);
    if (op == BNMF_OP_JMM_W || op == BNMF_OP_JMM_H) {
      if (!cur) return fail(BNMF_E_ARG, "the joint kernels need the current factor");
      if (op == BNMF_OP_JMM_W) {   // h_current -> Hc (N x K)
        if (int rc = h2d_bounce(stg, cur, nk * sizeof(double))) return rc;
        transpose_in<T><<<grid_for(nk), 256, 0, stream>>>(stg, K, size_t(N), Hc);
      } else {                     // w_current -> Wc
        if (int rc = h2d_bounce(stg, cur, fk * sizeof(double))) return rc;
        from_double<T><<<grid_for(fk), 256, 0, stream>>>(stg, fk, Wc);
      }
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(stream));
    }
    int rc = 0;
    bool w_out = false, h_out = false;
    switch (op) {
      case BNMF_OP_OBJECTIVE: {
        if ((rc = objective(Wt, Ht, 0))) return rc;
        sum_small<<<1, 1024, 0, stream>>>(opart, n_oblocks, comm + 2 * fk, st, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, comm + 2 * fk, sizeof(double), cudaMemcpyDeviceToHost, stream));
        break;
      }
      case BNMF_OP_KKT: {
        if ((rc = enqueue_kkt(0))) return rc;
        CK(cudaMemcpyAsync(out, tr_kkt, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        break;
      }
      case BNMF_OP_BMM_W:
        if ((rc = w_update(Wt, Ht, Ht, Ht, Wt, Wc, 0))) return rc;
        w_out = true;
        break;
      case BNMF_OP_BMM_H:
        if (den_ones && (rc = colsums(Wt, 0))) return rc;
        if ((rc = hside(PM_UPDATE, Wt, Ht, Wt, Wt, Ht, Hc, den_ones, 0))) return rc;
        h_out = true;
        break;
      case BNMF_OP_JMM_W:
        chi_h_valid = false;
        if ((rc = chi(Hc, Ht, C1h, C2h, nk, 0))) return rc;
        if ((rc = w_update(Wt, Ht, C1h, C2h, Wt, Wc, 0))) return rc;
        w_out = true;
        break;
      case BNMF_OP_JMM_H:
        if ((rc = chi(Wc, Wt, C1w, C2w, fk, 0))) return rc;
        if (den_ones && (rc = colsums(C2w, 0))) return rc;
        if ((rc = hside(PM_UPDATE, Wt, Ht, C1w, C2w, Ht, Hc, den_ones, 0))) return rc;
        h_out = true;
        break;
      default:
        return fail(BNMF_E_ARG, "unknown kernel operation");
    }
    if (w_out) {
      to_double<T><<<grid_for(fk), 256, 0, stream>>>(Wc, fk, stg);
      CK(cudaGetLastError());
      if ((rc = d2h_bounce(out, stg, fk * sizeof(double)))) return rc;
    } else if (h_out) {
      transpose_out<T><<<grid_for(nk), 256, 0, stream>>>(Hc, K, size_t(N), stg);
      CK(cudaGetLastError());
      if ((rc = d2h_bounce(out, stg, nk * sizeof(double)))) return rc;
    }
    CK(cudaStreamSynchronize(stream));
    begun = false;
    return 0;
  }

  int init_comm(int r, int nr, const void* id, int64_t ng) override {
    CK(cudaSetDevice(device));
    rank = r; nranks = nr; n_global = ng;
    if (nr > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      CKN(ncclCommInitRank(&comm_nccl, nr, uid, r));
    }
    return 0;
  }
};

}  // namespace bnmf

// ----------------------------------------------------------------------------
// C ABI

struct bnmf_ctx {
  std::unique_ptr<EngineBase> eng;
  bool sparse = false;
};

static int set_err(const std::string& m, int code) {
  g_err = m;
  return code;
}

extern "C" {

int bnmf_abi_version(void) { return BNMF_ABI_VERSION; }

int bnmf_device_count(int* count) {
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) { *count = 0; return set_err(cudaGetErrorString(e), BNMF_E_CUDA); }
  return 0;
}

int bnmf_ctx_create(bnmf_ctx** out, int device, int dtype) {
  if (!out) return set_err("null out", BNMF_E_ARG);
  *out = nullptr;
  if (dtype != BNMF_FP64 && dtype != BNMF_FP32) return set_err("dtype", BNMF_E_ARG);
  std::unique_ptr<bnmf_ctx> c(new bnmf_ctx);
  if (dtype == BNMF_FP64) c->eng.reset(new Engine<double>(device, dtype));
  else c->eng.reset(new Engine<float>(device, dtype));
  int rc = (dtype == BNMF_FP64) ? static_cast<Engine<double>*>(c->eng.get())->init()
                                : static_cast<Engine<float>*>(c->eng.get())->init();
  if (rc) return rc;
  *out = c.release();
  return 0;
}

void bnmf_ctx_destroy(bnmf_ctx* ctx) { delete ctx; }

const char* bnmf_last_error(const bnmf_ctx* ctx) {
  if (ctx && ctx->eng && !ctx->eng->err.empty()) return ctx->eng->err.c_str();
  return g_err.c_str();
}

int bnmf_nccl_unique_id(void* id128) {
  ncclUniqueId uid;
  ncclResult_t r = ncclGetUniqueId(&uid);
  if (r != ncclSuccess) return set_err(ncclGetErrorString(r), BNMF_E_NCCL);
  std::memcpy(id128, &uid, sizeof(uid));
  return 0;
}

#define CTX_CHECK(ctx) \
  if (!(ctx) || !(ctx)->eng) return set_err("null context", BNMF_E_ARG)

int bnmf_ctx_init_comm(bnmf_ctx* ctx, int rank, int nranks, const void* id128, int64_t n_global) {
  CTX_CHECK(ctx);
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_err("bad rank", BNMF_E_ARG);
  return ctx->eng->init_comm(rank, nranks, id128, n_global);
}

int bnmf_set_dense(bnmf_ctx* ctx, const void* v, int src_dtype, int src_on_device, int64_t F,
                   int64_t N, int64_t ld, double kappa) {
  CTX_CHECK(ctx);
  if (!v) return set_err("null data", BNMF_E_ARG);
  return ctx->eng->set_dense(v, src_dtype, src_on_device, F, N, ld, kappa);
}

int bnmf_kernel(bnmf_ctx* ctx, int op, const bnmf_params* p, const double* cur, double* out) {
  CTX_CHECK(ctx);
  if (!p) return set_err("null params", BNMF_E_ARG);
  return ctx->eng->kernel_op(op, p, cur, out);
}

int bnmf_data_stats(bnmf_ctx* ctx, double* out) {
  CTX_CHECK(ctx);
  if (!out) return set_err("null output", BNMF_E_ARG);
  int rc = ctx->eng->data_stats(out);
  if (rc < 0) return set_err("data statistics need dense data", BNMF_E_STATE);
  return rc;
}

int bnmf_set_csr(bnmf_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                 const float* values, const int64_t* colptr, const int32_t* rowidx,
                 const int32_t* perm, int64_t F, int64_t N, int64_t nnz, int src_on_device) {
  CTX_CHECK(ctx);
  if (ctx->eng->dtype != BNMF_FP32) return set_err("sparse path computes in fp32", BNMF_E_UNSUPPORTED);
  if (!indptr || !colptr || (nnz > 0 && (!indices || !values || !rowidx || !perm)))
    return set_err("null sparse arrays", BNMF_E_ARG);
  if (!ctx->sparse) {
    int dev = ctx->eng->device;
    cudaSetDevice(dev);
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
      return set_err("stream create", BNMF_E_CUDA);
    std::unique_ptr<EngineBase> sp(make_sparse_engine(dev, s));
    // a communicator attached before the switch moves to the sparse engine
    // (the dense engine's destructor would otherwise destroy it)
    sp->rank = ctx->eng->rank;
    sp->nranks = ctx->eng->nranks;
    sp->n_global = ctx->eng->n_global;
    sp->comm_nccl = ctx->eng->comm_nccl;
    ctx->eng->comm_nccl = nullptr;
    ctx->eng = std::move(sp);
    ctx->sparse = true;
  }
  if (nnz >= int64_t(INT32_MAX))
    return set_err("the sparse path takes fewer than 2^31 - 1 nonzeros", BNMF_E_UNSUPPORTED);
  return sparse_set_csr(ctx->eng.get(), reinterpret_cast<const long long*>(indptr), indices,
                        values, reinterpret_cast<const long long*>(colptr), rowidx, perm, F, N,
                        nnz, src_on_device);
}

int bnmf_set_factors(bnmf_ctx* ctx, const double* w, const double* h, int64_t K,
                     int src_on_device) {
  CTX_CHECK(ctx);
  if (!w || !h) return set_err("null factors", BNMF_E_ARG);
  return ctx->eng->set_factors(w, h, K, src_on_device);
}

int bnmf_begin(bnmf_ctx* ctx, const bnmf_params* p, int64_t max_iters) {
  CTX_CHECK(ctx);
  if (!p) return set_err("null params", BNMF_E_ARG);
  return ctx->eng->begin(p, max_iters);
}

int bnmf_step(bnmf_ctx* ctx, int64_t n) {
  CTX_CHECK(ctx);
  return ctx->eng->step(n);
}

int bnmf_step_timed(bnmf_ctx* ctx, int64_t n, float* ms) {
  CTX_CHECK(ctx);
  EngineBase* e = ctx->eng.get();
  cudaEvent_t a, b;
  cudaSetDevice(e->device);
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess)
    return set_err("event create", BNMF_E_CUDA);
  if (int rc0 = e->prepare(n)) return rc0;
  cudaEventRecord(a, e->stream);
  int rc = e->step(n);
  cudaEventRecord(b, e->stream);
  cudaError_t s = cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (rc) return rc;
  if (s != cudaSuccess) return set_err(cudaGetErrorString(s), BNMF_E_CUDA);
  if (ms) *ms = t;
  return 0;
}

int bnmf_sync(bnmf_ctx* ctx, int64_t* iters_done, int* converged) {
  CTX_CHECK(ctx);
  return ctx->eng->sync(iters_done, converged);
}

int bnmf_read_trace(bnmf_ctx* ctx, double* obj, double* seconds, double* kkt, int64_t n) {
  CTX_CHECK(ctx);
  return ctx->eng->read_trace(obj, seconds, kkt, n);
}

int bnmf_get_factors(bnmf_ctx* ctx, double* w, double* h) {
  CTX_CHECK(ctx);
  if (!w || !h) return set_err("null output", BNMF_E_ARG);
  return ctx->eng->get_factors(w, h);
}

int bnmf_run(bnmf_ctx* ctx, const bnmf_params* p, int64_t max_iters, int64_t* iters_done,
             int* converged) {
  CTX_CHECK(ctx);
  int rc = bnmf_begin(ctx, p, max_iters);
  if (rc) return rc;
  int64_t done = 0;
  int conv = 0;
  // chunks of 64 iterations between host checks of the device stop flag
  while (done < max_iters && !conv) {
    int64_t n = std::min<int64_t>(64, max_iters - done);
    if ((rc = bnmf_step(ctx, n))) return rc;
    if ((rc = bnmf_sync(ctx, &done, &conv))) return rc;
  }
  if (iters_done) *iters_done = done;
  if (converged) *converged = conv;
  return 0;
}

int bnmf_launches_per_iter(bnmf_ctx* ctx, int* launches) {
  CTX_CHECK(ctx);
  *launches = ctx->eng->launches_per_iter;
  return 0;
}

int bnmf_set_profiling(bnmf_ctx* ctx, int on) {
  CTX_CHECK(ctx);
  return ctx->eng->set_profiling(on);
}

int bnmf_pass_time(bnmf_ctx* ctx, float* ms_avg, int* samples) {
  CTX_CHECK(ctx);
  if (!ms_avg || !samples) return set_err("null output", BNMF_E_ARG);
  return ctx->eng->pass_time(ms_avg, samples);
}

int bnmf_active_schedule(bnmf_ctx* ctx, int* schedule) {
  CTX_CHECK(ctx);
  *schedule = ctx->eng->active_schedule;
  return 0;
}

int bnmf_pass_info(bnmf_ctx* ctx, int* out4) {
  CTX_CHECK(ctx);
  if (!out4) return set_err("null output", BNMF_E_ARG);
  ctx->eng->pass_info(out4);
  return 0;
}

void* bnmf_stream(bnmf_ctx* ctx) {
  if (!ctx || !ctx->eng) return nullptr;
  return ctx->eng->stream;
}

}  // extern "C"
