// Host-side engine interface shared by engine.cu and the fused tensor-core
// pass (fused_tc.cu).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>

#include "../../include/bnmf.h"
#include "bnmf_common.cuh"

namespace bnmf {

struct EngineBase {
  int device = 0, dtype = 0;
  std::string err;
  cudaStream_t stream = nullptr;
  ncclComm_t comm_nccl = nullptr;
  int rank = 0, nranks = 1;
  int64_t n_global = 0;
  int launches_per_iter = 0;
  int active_schedule = 0;
  bool fused_active = false;

  virtual ~EngineBase() {}
  int fail(int code, const std::string& msg);
  // [min, max, sum, non-finite count, count] of the values passed to the
  // last set_dense (before the kappa shift)
  virtual int data_stats(double* out5) { (void)out5; return -1; }
  virtual int set_dense(const void* v, int src_dtype, int on_dev, int64_t F, int64_t N,
                        int64_t ld, double kappa) = 0;
  virtual int set_factors(const double* w, const double* h, int64_t K, int on_dev) = 0;
  virtual int get_factors(double* w, double* h) = 0;
  virtual int begin(const bnmf_params* p, int64_t max_iters) = 0;
  virtual int step(int64_t n) = 0;
  // build whatever step(n) will replay (CUDA graph) without running it, so a
  // timed step does not include graph capture / instantiation
  virtual int prepare(int64_t n) { (void)n; return 0; }
  virtual int sync(int64_t* done, int* conv) = 0;
  virtual int read_trace(double* obj, double* sec, double* kkt, int64_t n) = 0;
  virtual int init_comm(int rank, int nranks, const void* id, int64_t n_global) = 0;
  virtual int set_profiling(int on) = 0;
  virtual int kernel_op(int op, const bnmf_params* p, const double* cur, double* out) {
    (void)op; (void)p; (void)cur; (void)out;
    return fail(BNMF_E_UNSUPPORTED, "kernel operations need dense data");
  }
  virtual int pass_time(float* ms_avg, int* samples) = 0;
  // [kind (0 none, 1 SIMT pair, 2 tcgen05), grid CTAs, cluster size, rows of cluster rank 0]
  // of the fused pass the last begin() selected
  virtual void pass_info(int* out4) { out4[0] = out4[1] = out4[2] = out4[3] = 0; }
};

// What the fused fp32 pass needs from the engine (device pointers are owned by
// the engine; Wt / Ht hold the normalised iterate in the standard layouts:
// W F x K row-major, H transposed N x K row-major).
struct FusedIO {
  int F = 0, N = 0, K = 0;
  size_t ldv = 0;
  const float* V = nullptr;
  float *Wt = nullptr, *Wc = nullptr, *Ht = nullptr, *Hc = nullptr;
  double* comm = nullptr;   // >= 2*F*K + 8 doubles, reduced / allreduced sums
  double* norms = nullptr;  // K
  double *tr_obj = nullptr, *tr_sec = nullptr, *tr_kkt = nullptr;
  RunState* st = nullptr;
  cudaStream_t stream = nullptr;
  Scalars sc{};
  int algorithm = 0;
  int compute_kkt = 0;
  int nranks = 1;
  ncclComm_t nccl = nullptr;
  int64_t n_global = 0;
  int* launches = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // optional, around the pass kernel
};

// Record an event so that it also works inside stream capture (external
// event node); outside capture a plain record.
inline cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  return cudaEventRecord(ev, s);
}

EngineBase* make_sparse_engine(int device, cudaStream_t stream);
int sparse_set_csr(EngineBase* e, const long long* ip, const int* ix, const float* v,
                   const long long* cp, const int* ri, const int* pm, int64_t F, int64_t N,
                   int64_t nnz, int on_dev);

struct FusedState;
bool fused_supported(int dtype, int F, int K, int algorithm, int L, int Lw, int Lh, double beta);
int fused_create(FusedState** out, const FusedIO& io, std::string& err);
int fused_begin(FusedState* fs, const FusedIO& io, std::string& err);
int fused_enqueue_iteration(FusedState* fs, const FusedIO& io, int slot, std::string& err);
int fused_export(FusedState* fs, const FusedIO& io, std::string& err);
int fused_select(FusedState* fs, const FusedIO& io, std::string& err);  // async, no sync
void fused_destroy(FusedState* fs);
bool fused_shape_matches(const FusedState* fs, int F, int N, int K);
void fused_info(const FusedState* fs, int* out4);

}  // namespace bnmf
