// Sparse KL (beta = 1) path: V in CSR (plus a CSC view for the column sums),
// fp32 factors, fp64 reductions, deterministic (no float atomics).
//
// Restates the dense beta = 1 updates at the nonzeros (the reference has no
// sparse kernel: it densifies, matrixio.py:115-128):
//   W_p = W~ * ((V/Vt) H~^T) / rowsum(H~)          updates.py:301-303
//   H_p = H~ * (W^T (V/Vt)) / colsum(W_p)            updates.py:325-327
//         (JMM: W^T with W = W~ and Vt = W~H~; BMM: W = W_p, Vt = W_p H~)
//   D(V | WH) = sum_nnz [x log(x/y) - x] + (1^T W)(H 1)   core.py:101 at x=0
// Per outer iteration (solver.py:301-319), rows of V are local to the rank:
//   pass A (CSR, warp per row)   y, z = x/y at the nonzeros, W_p row update,
//                                per-block colsum / sum-of-squares of W_p
//   reduce (+ allreduce)         DenH = colsum(W_p), norms = ||W_p[:,k]||
//   pass B (CSC, warp per column) H_p = H~ * num/DenH, H~_p = H_p * norms,
//                                per-block rowsum of H~_p (next DenW)
//   pass C (CSR, warp per row)   W~_p = W_p / norms, objective at nonzeros
//   finish                       objective + dense term, stop rule
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <string>

#include "engine.h"
#include "small_kernels.cuh"

namespace bnmf {

constexpr int SP_THREADS = 256;
constexpr int SP_WARPS = SP_THREADS / 32;
constexpr int SP_KMAX = 128;   // 4 k per lane

// warp sum (butterfly => every lane holds the identical result)
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct SpArgs {
  int F, N, K, KL;             // KL = K rounded up to a multiple of 32 (lanes x per-lane)
  const long long* indptr;
  const int* indices;
  const float* vals;
  const long long* colptr;
  const int* rowidx;
  const int* perm;             // CSC position -> CSR position
  float* z;                    // per nonzero (CSR order)
  float* Wt;                   // W~ (F x K)
  float* Wp;                   // W_p (F x K)
  float* Ht;                   // H~ (N x K)
  float* Hn;                   // H~_p (N x K)
  const double* denw;          // rowsum(H~) (K)
  const double* denh;          // colsum(W_p) (K)
  const double* norms;         // ||W_p[:,k]|| (K)
  double* pa;                  // pass A partials [blocks][2K]: colsum, sumsq
  double* pb;                  // pass B partials [blocks][K]: rowsum(H~_p)
  double* pc;                  // pass C partials [blocks]: sum_nnz x log(x/y) - x
  int algorithm;
  Scalars sc;
};

// ---- pass A: rows --------------------------------------------------------
__global__ void __launch_bounds__(SP_THREADS) sp_pass_a(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = a.K, per = a.KL / 32;
  double cs[SP_KMAX / 32], sq[SP_KMAX / 32];
  for (int i = 0; i < per; ++i) { cs[i] = 0.0; sq[i] = 0.0; }
  __shared__ double red[SP_WARPS][2 * SP_KMAX];
  for (int f = blockIdx.x * SP_WARPS + warp; f < a.F; f += gridDim.x * SP_WARPS) {
    float w[SP_KMAX / 32], num[SP_KMAX / 32];
    for (int i = 0; i < per; ++i) {
      const int k = lane + 32 * i;
      w[i] = k < K ? a.Wt[size_t(f) * K + k] : 0.f;
      num[i] = 0.f;
    }
    const long long j0 = a.indptr[f], j1 = a.indptr[f + 1];
    for (long long j = j0; j < j1; ++j) {
      const int n = a.indices[j];
      const float x = a.vals[j];
      float h[SP_KMAX / 32], p = 0.f;
      for (int i = 0; i < per; ++i) {
        const int k = lane + 32 * i;
        h[i] = k < K ? a.Ht[size_t(n) * K + k] : 0.f;
        p = fmaf(w[i], h[i], p);
      }
      const float y = warp_sum(p);
      const float zz = x / y;
      if (lane == 0) a.z[j] = zz;
      for (int i = 0; i < per; ++i) num[i] = fmaf(zz, h[i], num[i]);
    }
    for (int i = 0; i < per; ++i) {
      const int k = lane + 32 * i;
      if (k < K) {
        const double r = double(num[i]) / fmax(a.denw[k], a.sc.floor);
        const float wn = float(double(w[i]) * apply_exponent<double>(r, a.sc.gamma));
        a.Wp[size_t(f) * K + k] = wn;
        cs[i] += double(wn);
        sq[i] += double(wn) * double(wn);
      }
    }
  }
  for (int i = 0; i < per; ++i) {
    red[warp][lane + 32 * i] = cs[i];
    red[warp][SP_KMAX + lane + 32 * i] = sq[i];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < SP_WARPS; ++w) { s0 += red[w][k]; s1 += red[w][SP_KMAX + k]; }
    a.pa[size_t(blockIdx.x) * 2 * K + k] = s0;
    a.pa[size_t(blockIdx.x) * 2 * K + K + k] = s1;
  }
}

// ---- pass B: columns -----------------------------------------------------
__global__ void __launch_bounds__(SP_THREADS) sp_pass_b(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = a.K, per = a.KL / 32;
  double rs[SP_KMAX / 32];
  for (int i = 0; i < per; ++i) rs[i] = 0.0;
  __shared__ double red[SP_WARPS][SP_KMAX];
  const bool bmm = a.algorithm == BNMF_BMM;
  for (int n = blockIdx.x * SP_WARPS + warp; n < a.N; n += gridDim.x * SP_WARPS) {
    float h[SP_KMAX / 32], num[SP_KMAX / 32];
    for (int i = 0; i < per; ++i) {
      const int k = lane + 32 * i;
      h[i] = k < K ? a.Ht[size_t(n) * K + k] : 0.f;
      num[i] = 0.f;
    }
    const long long j0 = a.colptr[n], j1 = a.colptr[n + 1];
    for (long long j = j0; j < j1; ++j) {
      const int f = a.rowidx[j];
      float w[SP_KMAX / 32];
      const float* W = bmm ? a.Wp : a.Wt;
      for (int i = 0; i < per; ++i) {
        const int k = lane + 32 * i;
        w[i] = k < K ? W[size_t(f) * K + k] : 0.f;
      }
      float zz;
      if (bmm) {   // block update: Vt2 = W_p H~ at this nonzero (updates.py:173-181)
        float p = 0.f;
        for (int i = 0; i < per; ++i) p = fmaf(w[i], h[i], p);
        zz = a.vals[a.perm[j]] / warp_sum(p);
      } else {     // joint update: the anchor's Z from pass A
        zz = a.z[a.perm[j]];
      }
      for (int i = 0; i < per; ++i) num[i] = fmaf(zz, w[i], num[i]);
    }
    for (int i = 0; i < per; ++i) {
      const int k = lane + 32 * i;
      if (k < K) {
        const double r = double(num[i]) / fmax(a.denh[k], a.sc.floor);
        const double hp = double(h[i]) * apply_exponent<double>(r, a.sc.gamma);
        const float hn = float(hp * a.norms[k]);
        a.Hn[size_t(n) * K + k] = hn;
        rs[i] += double(hn);
      }
    }
  }
  for (int i = 0; i < per; ++i) red[warp][lane + 32 * i] = rs[i];
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < SP_WARPS; ++w) s += red[w][k];
    a.pb[size_t(blockIdx.x) * K + k] = s;
  }
}

// ---- pass C: normalise W, objective at the nonzeros ------------------------
__global__ void __launch_bounds__(SP_THREADS) sp_pass_c(SpArgs a, const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = a.K, per = a.KL / 32;
  double acc = 0.0;
  __shared__ double red[SP_WARPS];
  for (int f = blockIdx.x * SP_WARPS + warp; f < a.F; f += gridDim.x * SP_WARPS) {
    float w[SP_KMAX / 32];
    for (int i = 0; i < per; ++i) {
      const int k = lane + 32 * i;
      w[i] = 0.f;
      if (k < K) {
        w[i] = float(double(a.Wp[size_t(f) * K + k]) / a.norms[k]);
        a.Wt[size_t(f) * K + k] = w[i];
      }
    }
    const long long j0 = a.indptr[f], j1 = a.indptr[f + 1];
    double rowacc = 0.0;
    for (long long j = j0; j < j1; ++j) {
      const int n = a.indices[j];
      float p = 0.f;
      for (int i = 0; i < per; ++i) {
        const int k = lane + 32 * i;
        if (k < K) p = fmaf(w[i], a.Hn[size_t(n) * K + k], p);
      }
      const double y = double(warp_sum(p));
      const double x = double(a.vals[j]);
      if (x != 0.0) rowacc += x * log(x / y) - x;
    }
    acc += rowacc;   // identical on every lane
  }
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < SP_WARPS; ++w) s += red[w];
    a.pc[blockIdx.x] = s;
  }
}

// fixed-order reduction of the pass-A partials -> comm[0:2K] (colsum, sumsq)
__global__ void sp_reduce_a(const double* pa, int G, int K, double* comm, const RunState* st,
                            int slot) {
  if (!iter_active(st, slot)) return;
  for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += pa[size_t(g) * 2 * K + i];
    comm[i] = s;
  }
}
// DenH = colsum(W_p), norms = sqrt(sum_f W_p^2)  (after the allreduce)
__global__ void sp_post_a(const double* comm, int K, double* denh, double* norms,
                          const RunState* st, int slot) {
  if (!iter_active(st, slot)) return;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    denh[k] = comm[k];
    norms[k] = sqrt(comm[K + k]);
  }
}
// rowsum(H~_p) -> denw (next iteration); objective = sum_nnz + sum_k colsum(W~_p) rowsum(H~_p)
// colsum(W~_p) = colsum(W_p) / norms
__global__ void sp_finish(const double* pb, int GB, const double* pc, int GC, int K,
                          const double* comm_a, const double* norms, double* denw,
                          double* comm_obj, RunState* st, int slot, double* tr_obj,
                          double* tr_sec, double tol, int nranks_obj_done) {
  (void)nranks_obj_done;
  if (!iter_active(st, slot)) return;
  if (threadIdx.x == 0) {
    double dense = 0.0;
    for (int k = 0; k < K; ++k) {
      double rs = 0.0;
      for (int g = 0; g < GB; ++g) rs += pb[size_t(g) * K + k];
      denw[k] = rs;
      dense += (comm_a[k] / norms[k]) * rs;
    }
    double s = 0.0;
    for (int g = 0; g < GC; ++g) s += pc[g];
    comm_obj[0] = s;       // local nonzero part (allreduced by the host before finish)
    comm_obj[1] = dense;   // global dense part (every rank holds all of H~)
  }
}
__global__ void sp_rowsum_init(const float* Ht, int N, int K, double* denw) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int n = 0; n < N; ++n) s += double(Ht[size_t(n) * K + k]);
    denw[k] = s;
  }
}
__global__ void sp_total_obj(double* comm_obj, int nranks_parts) {
  (void)nranks_parts;
  comm_obj[2] = comm_obj[0] + comm_obj[1];
}

#define SCK(call)                                                                   \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      return fail(BNMF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    }                                                                               \
  } while (0)

struct SparseEngine : EngineBase {
  int F = 0, N = 0, K = 0, KL = 32;
  long long nnz = 0;
  long long* indptr = nullptr;
  int* indices = nullptr;
  float* vals = nullptr;
  long long* colptr = nullptr;
  int* rowidx = nullptr;
  int* perm = nullptr;
  float *z = nullptr, *Wt = nullptr, *Wp = nullptr, *Ht = nullptr, *Hn = nullptr;
  double *denw = nullptr, *denh = nullptr, *norms = nullptr, *pa = nullptr, *pb = nullptr,
         *pc = nullptr, *comm = nullptr;
  double *tr_obj = nullptr, *tr_sec = nullptr, *tr_kkt = nullptr;
  int64_t tr_cap = 0;
  RunState* st = nullptr;
  RunState* st_host = nullptr;
  int GA = 1, GB = 1;
  bnmf_params p{};
  Scalars sc{};
  bool begun = false;
  cudaGraphExec_t gexec = nullptr;
  int gchunk = 0;
  int launches = 0;

  SparseEngine(int dev, cudaStream_t s) { device = dev; dtype = BNMF_FP32; stream = s; }
  ~SparseEngine() override {
    if (gexec) cudaGraphExecDestroy(gexec);
    void* ptrs[] = {indptr, indices, vals, colptr, rowidx, perm, z, Wt, Wp, Ht, Hn, denw, denh,
                    norms, pa, pb, pc, comm, tr_obj, tr_sec, tr_kkt, st};
    for (void* q : ptrs) if (q) cudaFree(q);
    if (st_host) cudaFreeHost(st_host);
    if (comm_nccl) ncclCommDestroy(comm_nccl);
    if (stream) cudaStreamDestroy(stream);
  }

  int set_dense(const void*, int, int, int64_t, int64_t, int64_t, double) override {
    return fail(BNMF_E_STATE, "context holds a sparse matrix");
  }

  template <typename Tp>
  int upload(Tp** dst, const void* src, size_t count, int on_dev) {
    if (*dst) SCK(cudaFree(*dst));
    SCK(cudaMalloc(dst, std::max<size_t>(count, 1) * sizeof(Tp)));
    if (count)
      SCK(cudaMemcpyAsync(*dst, src, count * sizeof(Tp),
                          on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    return 0;
  }

  int set_csr(const long long* ip, const int* ix, const float* v, const long long* cp,
              const int* ri, const int* pm, int64_t F_, int64_t N_, int64_t nnz_, int on_dev) {
    SCK(cudaSetDevice(device));
    if (F_ < 1 || N_ < 1 || nnz_ < 0 || F_ > INT_MAX || N_ > INT_MAX)
      return fail(BNMF_E_ARG, "bad sparse shape");
    F = int(F_); N = int(N_); nnz = nnz_;
    int rc;
    if ((rc = upload(&indptr, ip, size_t(F) + 1, on_dev))) return rc;
    if ((rc = upload(&indices, ix, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&vals, v, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&colptr, cp, size_t(N) + 1, on_dev))) return rc;
    if ((rc = upload(&rowidx, ri, size_t(nnz), on_dev))) return rc;
    if ((rc = upload(&perm, pm, size_t(nnz), on_dev))) return rc;
    if (z) SCK(cudaFree(z));
    SCK(cudaMalloc(&z, std::max<size_t>(nnz, 1) * sizeof(float)));
    if (!st) {
      SCK(cudaMalloc(&st, sizeof(RunState)));
      SCK(cudaMallocHost(&st_host, sizeof(RunState)));
    }
    SCK(cudaStreamSynchronize(stream));
    K = 0;
    begun = false;
    return 0;
  }

  int set_factors(const double* w, const double* h, int64_t K_, int on_dev) override {
    if (!indptr) return fail(BNMF_E_STATE, "set_csr must precede set_factors");
    if (K_ < 1 || K_ > SP_KMAX) return fail(BNMF_E_UNSUPPORTED, "sparse path supports rank 1..128");
    SCK(cudaSetDevice(device));
    if (K != K_) {
      float** fp[] = {&Wt, &Wp, &Ht, &Hn};
      for (float** q : fp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      double** dp[] = {&denw, &denh, &norms, &pa, &pb, &pc, &comm};
      for (double** q : dp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      K = int(K_);
      KL = (K + 31) / 32 * 32;
      SCK(cudaMalloc(&Wt, size_t(F) * K * sizeof(float)));
      SCK(cudaMalloc(&Wp, size_t(F) * K * sizeof(float)));
      SCK(cudaMalloc(&Ht, size_t(N) * K * sizeof(float)));
      SCK(cudaMalloc(&Hn, size_t(N) * K * sizeof(float)));
      GA = std::max(1, std::min((F + SP_WARPS - 1) / SP_WARPS, 148 * 8));
      GB = std::max(1, std::min((N + SP_WARPS - 1) / SP_WARPS, 148 * 8));
      SCK(cudaMalloc(&denw, K * sizeof(double)));
      SCK(cudaMalloc(&denh, K * sizeof(double)));
      SCK(cudaMalloc(&norms, K * sizeof(double)));
      SCK(cudaMalloc(&pa, size_t(GA) * 2 * K * sizeof(double)));
      SCK(cudaMalloc(&pb, size_t(GB) * K * sizeof(double)));
      SCK(cudaMalloc(&pc, size_t(GA) * sizeof(double)));
      SCK(cudaMalloc(&comm, (2 * K + 8) * sizeof(double)));
    }
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    double* stg;
    SCK(cudaMalloc(&stg, std::max(fk, nk) * sizeof(double)));
    SCK(cudaMemcpyAsync(stg, w, fk * sizeof(double),
                        on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    from_double<float><<<int(std::min<size_t>((fk + 255) / 256, 1184)), 256, 0, stream>>>(stg, fk, Wt);
    SCK(cudaMemcpyAsync(stg, h, nk * sizeof(double),
                        on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream));
    transpose_in<float><<<int(std::min<size_t>((nk + 255) / 256, 1184)), 256, 0, stream>>>(stg, K, size_t(N), Ht);
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(stream));
    SCK(cudaFree(stg));
    begun = false;
    return 0;
  }

  SpArgs args() {
    SpArgs a;
    a.F = F; a.N = N; a.K = K; a.KL = KL;
    a.indptr = indptr; a.indices = indices; a.vals = vals;
    a.colptr = colptr; a.rowidx = rowidx; a.perm = perm; a.z = z;
    a.Wt = Wt; a.Wp = Wp; a.Ht = Ht; a.Hn = Hn;
    a.denw = denw; a.denh = denh; a.norms = norms;
    a.pa = pa; a.pb = pb; a.pc = pc;
    a.algorithm = p.algorithm; a.sc = sc;
    return a;
  }

  int begin(const bnmf_params* pp, int64_t max_iters) override {
    if (!Wt) return fail(BNMF_E_STATE, "factors must be set before begin");
    if (pp->beta != 1.0) return fail(BNMF_E_UNSUPPORTED, "sparse path implements beta = 1 (KL)");
    if (pp->kappa != 0.0) return fail(BNMF_E_UNSUPPORTED, "sparse path needs kappa = 0");
    if (pp->sub_iters != 1 || pp->sub_iters_w > 1 || pp->sub_iters_h > 1)
      return fail(BNMF_E_UNSUPPORTED, "sparse path implements one sub-iteration");
    SCK(cudaSetDevice(device));
    p = *pp;
    sc.beta = p.beta; sc.gamma = p.gamma; sc.kappa = 0.0; sc.floor = p.floor; sc.tol = p.tol;
    active_schedule = BNMF_SCHED_REFERENCE;
    if (tr_cap < max_iters) {
      double** dp[] = {&tr_obj, &tr_sec, &tr_kkt};
      for (double** q : dp) if (*q) { SCK(cudaFree(*q)); *q = nullptr; }
      SCK(cudaMalloc(&tr_obj, size_t(max_iters) * sizeof(double)));
      SCK(cudaMalloc(&tr_sec, size_t(max_iters) * sizeof(double)));
      SCK(cudaMalloc(&tr_kkt, size_t(max_iters) * 2 * sizeof(double)));
      tr_cap = max_iters;
    }
    SCK(cudaMemsetAsync(tr_kkt, 0xff, size_t(max_iters) * 2 * sizeof(double), stream));
    RunState h{};
    h.base = 1;
    h.stop_iter = LLONG_MAX;
    h.max_iter = max_iters;
    *st_host = h;
    SCK(cudaMemcpyAsync(st, st_host, sizeof(RunState), cudaMemcpyHostToDevice, stream));
    sp_rowsum_init<<<1, 128, 0, stream>>>(Ht, N, K, denw);
    SCK(cudaGetLastError());
    if (gexec) { SCK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    SCK(cudaStreamSynchronize(stream));
    begun = true;
    return 0;
  }

  int allreduce(double* buf, size_t count) {
    if (nranks > 1) {
      ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_nccl, stream);
      if (r != ncclSuccess) return fail(BNMF_E_NCCL, ncclGetErrorString(r));
      launches += 1;
    }
    return 0;
  }

  int enqueue_iteration(int slot) {
    SpArgs a = args();
    begin_iter<<<1, 1, 0, stream>>>(st, slot);
    sp_pass_a<<<GA, SP_THREADS, 0, stream>>>(a, st, slot);
    sp_reduce_a<<<1, 256, 0, stream>>>(pa, GA, K, comm, st, slot);
    SCK(cudaGetLastError());
    launches += 3;
    if (int rc = allreduce(comm, 2 * K)) return rc;
    sp_post_a<<<1, 128, 0, stream>>>(comm, K, denh, norms, st, slot);
    if (nranks > 1) {
      // the column pass needs every rank's nonzeros: rows are sharded, so the
      // H numerator would need a K x N allreduce (not implemented: see DESIGN.md)
      return fail(BNMF_E_UNSUPPORTED, "multi-GPU sparse path not implemented");
    }
    sp_pass_b<<<GB, SP_THREADS, 0, stream>>>(a, st, slot);
    sp_pass_c<<<GA, SP_THREADS, 0, stream>>>(a, st, slot);
    double* cobj = comm + 2 * K;
    sp_finish<<<1, 32, 0, stream>>>(pb, GB, pc, GA, K, comm, norms, denw, cobj, st, slot, tr_obj,
                                    tr_sec, sc.tol, nranks);
    sp_total_obj<<<1, 1, 0, stream>>>(cobj, nranks);
    finish_iter<<<1, 1, 0, stream>>>(st, slot, cobj + 2, tr_obj, tr_sec, sc.tol);
    // H~_p becomes the next iterate
    SCK(cudaMemcpyAsync(Ht, Hn, size_t(N) * K * sizeof(float), cudaMemcpyDeviceToDevice, stream));
    SCK(cudaGetLastError());
    launches += 7;
    return 0;
  }

  int capture(int chunk) {
    if (gexec && gchunk == chunk) return 0;
    if (gexec) { SCK(cudaGraphExecDestroy(gexec)); gexec = nullptr; }
    cudaGraph_t g;
    SCK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    int l0 = launches, rc = 0;
    for (int j = 0; j < chunk && rc == 0; ++j) rc = enqueue_iteration(j);
    if (rc == 0) advance_base<<<1, 1, 0, stream>>>(st, chunk);
    cudaError_t ec = cudaStreamEndCapture(stream, &g);
    if (rc) return rc;
    if (ec != cudaSuccess) return fail(BNMF_E_CUDA, cudaGetErrorString(ec));
    launches_per_iter = (launches - l0) / chunk;
    SCK(cudaGraphInstantiate(&gexec, g, 0));
    SCK(cudaGraphDestroy(g));
    gchunk = chunk;
    return 0;
  }

  int prepare(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    SCK(cudaSetDevice(device));
    return n >= 16 ? capture(16) : 0;
  }

  int step(int64_t n) override {
    if (!begun) return fail(BNMF_E_STATE, "begin must precede step");
    SCK(cudaSetDevice(device));
    const int chunk = 16;
    for (int64_t i = 0; i < n / chunk; ++i) {
      if (int rc = capture(chunk)) return rc;
      SCK(cudaGraphLaunch(gexec, stream));
    }
    for (int64_t i = 0; i < n % chunk; ++i) {
      int l0 = launches;
      if (int rc = enqueue_iteration(0)) return rc;
      launches_per_iter = launches - l0;
      advance_base<<<1, 1, 0, stream>>>(st, 1);
      SCK(cudaGetLastError());
    }
    return 0;
  }

  int sync(int64_t* done, int* conv) override {
    SCK(cudaSetDevice(device));
    SCK(cudaMemcpyAsync(st_host, st, sizeof(RunState), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    if (done) *done = st_host->iters_done;
    if (conv) *conv = st_host->converged;
    return 0;
  }

  int read_trace(double* obj, double* sec, double* kkt, int64_t n) override {
    if (n > tr_cap) return fail(BNMF_E_ARG, "trace request exceeds max_iters");
    if (obj) SCK(cudaMemcpyAsync(obj, tr_obj, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (sec) SCK(cudaMemcpyAsync(sec, tr_sec, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    if (kkt) SCK(cudaMemcpyAsync(kkt, tr_kkt, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    return 0;
  }

  int get_factors(double* w, double* h) override {
    size_t fk = size_t(F) * K, nk = size_t(N) * K;
    double* stg;
    SCK(cudaMalloc(&stg, std::max(fk, nk) * sizeof(double)));
    to_double<float><<<int(std::min<size_t>((fk + 255) / 256, 1184)), 256, 0, stream>>>(Wt, fk, stg);
    SCK(cudaMemcpyAsync(w, stg, fk * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    transpose_out<float><<<int(std::min<size_t>((nk + 255) / 256, 1184)), 256, 0, stream>>>(Ht, K, size_t(N), stg);
    SCK(cudaMemcpyAsync(h, stg, nk * sizeof(double), cudaMemcpyDeviceToHost, stream));
    SCK(cudaStreamSynchronize(stream));
    SCK(cudaFree(stg));
    return 0;
  }

  int init_comm(int r, int nr, const void* id, int64_t ng) override {
    (void)ng;
    rank = r; nranks = nr;
    if (nr > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof(uid));
      ncclResult_t rr = ncclCommInitRank(&comm_nccl, nr, uid, r);
      if (rr != ncclSuccess) return fail(BNMF_E_NCCL, ncclGetErrorString(rr));
    }
    return 0;
  }
  int set_profiling(int) override { return 0; }
  int pass_time(float* ms, int* n) override { *ms = 0.f; *n = 0; return 0; }
};

EngineBase* make_sparse_engine(int device, cudaStream_t stream) {
  return new SparseEngine(device, stream);
}

int sparse_set_csr(EngineBase* e, const long long* ip, const int* ix, const float* v,
                   const long long* cp, const int* ri, const int* pm, int64_t F, int64_t N,
                   int64_t nnz, int on_dev) {
  return static_cast<SparseEngine*>(e)->set_csr(ip, ix, v, cp, ri, pm, F, N, nnz, on_dev);
}

}  // namespace bnmf
