/*
 * bnmf.h -- C ABI of the B200-native beta-NMF iteration library (libbnmf.so).
 *
 * The reference (betanmf, arXiv 2106.15214) is a pure-Python package with no
 * FFI of its own; its hot path is the solver loop
 *     fit / run_jmm / run_bmm(data, config)      solver.py:224-289
 *     _outer_loop (init, step, objective, stop)  solver.py:292-326
 *     step: anchor + joint bases + updates       solver.py:239-280, majorizer.py:53-62,
 *                                                updates.py:157-235, 281-331
 * Each entry point below names the reference interface it replaces.  A ctypes
 * binding (paper_2106_15214_b200/_native.py) is what the
 * reference's fit() would call instead of its numpy loop.
 *
 * Conventions: plain pointers and sizes, no torch types.  Every function
 * returns 0 on success or a negative BNMF_E* code; bnmf_last_error() gives
 * the message.  All device work is enqueued on the context's own stream;
 * results are bitwise reproducible for a fixed device count.
 */
#ifndef BNMF_H_
#define BNMF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BNMF_ABI_VERSION 1

enum { BNMF_FP64 = 0, BNMF_FP32 = 1 };
enum { BNMF_JMM = 0, BNMF_BMM = 1 };
/* schedule: 0 = auto, 1 = reference order (SIMT, any L), 2 = fused single-read
 * pipelined pass (fp32, L = 1, tensor cores) */
enum { BNMF_SCHED_AUTO = 0, BNMF_SCHED_REFERENCE = 1, BNMF_SCHED_FUSED = 2 };

enum {
  BNMF_OK = 0,
  BNMF_E_ARG = -1,
  BNMF_E_CUDA = -2,
  BNMF_E_NCCL = -3,
  BNMF_E_STATE = -4,
  BNMF_E_UNSUPPORTED = -5
};

/* Mirrors SolverConfig (solver.py:62-114) after resolution of kappa and gamma. */
typedef struct bnmf_params {
  int algorithm;        /* BNMF_JMM / BNMF_BMM            (config.algorithm)   */
  int sub_iters;        /* L for JMM                      (config.sub_iters)   */
  int sub_iters_w;      /* L_W for BMM (0 -> sub_iters)   (config.sub_iters_w) */
  int sub_iters_h;      /* L_H for BMM (0 -> sub_iters)   (config.sub_iters_h) */
  double beta;          /* config.beta                                          */
  double gamma;         /* config.gamma (solver.py:107-109)                     */
  double kappa;         /* resolved shift (solver.py:205-221)                   */
  double floor;         /* config.denominator_floor                             */
  double tol;           /* config.tol (solver.py:174-180)                       */
  int compute_kkt;      /* per-iteration KKT residuals (solver.py:313)          */
  int schedule;         /* BNMF_SCHED_*                                         */
} bnmf_params;

typedef struct bnmf_ctx bnmf_ctx;

int bnmf_abi_version(void);
int bnmf_device_count(int* count);

/* Context on CUDA device `device` computing in `dtype` (BNMF_FP64/BNMF_FP32).
 * Replaces the implicit numpy state of solver._outer_loop. */
int bnmf_ctx_create(bnmf_ctx** out, int device, int dtype);
void bnmf_ctx_destroy(bnmf_ctx* ctx);
const char* bnmf_last_error(const bnmf_ctx* ctx); /* ctx may be NULL */

/* N-column sharding across ranks (one process per GPU).  Rank 0 creates the
 * 128-byte NCCL unique id, the host layer broadcasts it.  No reference
 * counterpart (the reference is single-process). */
int bnmf_nccl_unique_id(void* id128);
int bnmf_ctx_init_comm(bnmf_ctx* ctx, int rank, int nranks, const void* id128,
                       int64_t n_global);

/* Data: the local column block V[:, n0:n0+N] (F x N, row stride ld elements),
 * src_dtype BNMF_FP64/BNMF_FP32, host or device memory.  kappa is added on the
 * device (DataMatrix.shifted, core.py:216-220). */
int bnmf_set_dense(bnmf_ctx* ctx, const void* v, int src_dtype, int src_on_device,
                   int64_t F, int64_t N, int64_t ld, double kappa);

/* Statistics of the values passed to the last bnmf_set_dense (before the
 * kappa shift), computed on the device during the upload: out[0] min and
 * out[1] max of the finite entries, out[2] their sum (fp64), out[3] the number
 * of non-finite entries, out[4] the entry count.  They replace the host scans
 * of DataMatrix.__post_init__ / check_domain (core.py:188-228) and
 * default_kappa (core.py:176-185, solver.py:205-221), so the Python layer can
 * raise the reference's errors without reading V on the host. */
int bnmf_data_stats(bnmf_ctx* ctx, double* out);

/* Sparse data (beta = 1 only): the local rows of V in CSR (indptr F+1,
 * int32 column indices, fp32 values) plus its CSC view (colptr N+1, int32 row
 * indices, perm[j] = CSR position of CSC entry j) used for the deterministic
 * column sums.  The reference densifies sparse input (matrixio.py:115-128);
 * this replaces DataMatrix for config 5.  Switches the context to the sparse
 * engine (fp32 contexts only). */
int bnmf_set_csr(bnmf_ctx* ctx, const int64_t* indptr, const int32_t* indices,
                 const float* values, const int64_t* colptr, const int32_t* rowidx,
                 const int32_t* perm, int64_t F, int64_t N, int64_t nnz, int src_on_device);

/* Factors: W (F x K) and the local H block (K x N), fp64 row-major host or
 * device memory (init_factors, solver.py:137-153, or an injected init).
 * Applies the reference FactorPair checks (core.py FactorPair.__post_init__)
 * to the device copy: BNMF_E_ARG with "factor entries must be finite" or
 * "factor entries must be strictly positive" (the reference's messages). */
int bnmf_set_factors(bnmf_ctx* ctx, const double* w, const double* h, int64_t K,
                     int src_on_device);

/* Start a fit: validates params, resets the trace (TraceRow list) and the
 * stop state; max_iters = config.max_outer_iters. */
int bnmf_begin(bnmf_ctx* ctx, const bnmf_params* p, int64_t max_iters);
/* Enqueue n outer iterations (solver.py:301-319) asynchronously.  Iterations
 * after a stop (should_stop) or past max_iters are no-ops on the device. */
int bnmf_step(bnmf_ctx* ctx, int64_t n);
/* Same, bracketed by CUDA events on the context stream; *ms = device time. */
int bnmf_step_timed(bnmf_ctx* ctx, int64_t n, float* ms);
/* Wait for the stream; report finished iterations and convergence. */
int bnmf_sync(bnmf_ctx* ctx, int64_t* iters_done, int* converged);
/* Trace rows 1..n: objective, cumulative loop seconds, kkt (2 per row, may be
 * NULL).  TraceRow of solver.py:54-59. */
int bnmf_read_trace(bnmf_ctx* ctx, double* obj, double* seconds, double* kkt, int64_t n);
/* Normalised factors W (F x K) and local H (K x N), fp64 host. */
int bnmf_get_factors(bnmf_ctx* ctx, double* w, double* h);

/* Whole fit: begin + steps until stop or max_iters (fit, solver.py:285-289). */
int bnmf_run(bnmf_ctx* ctx, const bnmf_params* p, int64_t max_iters,
             int64_t* iters_done, int* converged);

/* Introspection for the bench / tests. */
int bnmf_launches_per_iter(bnmf_ctx* ctx, int* launches);
int bnmf_active_schedule(bnmf_ctx* ctx, int* schedule);
/* CUDA events around the dominant V-pass kernel of every iteration slot;
 * bnmf_pass_time returns its average device time over the last chunk. */
int bnmf_set_profiling(bnmf_ctx* ctx, int on);
int bnmf_pass_time(bnmf_ctx* ctx, float* ms_avg, int* samples);
/* Which fused pass kernel the last begin() selected: out[0] = 0 (none: reference
 * schedule), 1 (SIMT pair) or 2 (tcgen05); out[1] = grid CTAs; out[2] = CTAs per
 * cluster; out[3] = rows owned by cluster rank 0.  Diagnostics for the parity
 * tests (BNMF_TC_MAX_CLUSTERS caps the tcgen05 grid). */
int bnmf_pass_info(bnmf_ctx* ctx, int* out4);
void* bnmf_stream(bnmf_ctx* ctx);

/* One kernel of the reference's lower-level public API on the data (bnmf_set_dense: the
 * already-shifted V + kappa, passed with kappa = 0) and the factor pair (bnmf_set_factors:
 * (w, h), or the anchor (w~, h~) of the joint kernels) the context holds.  p carries beta,
 * gamma, kappa (the shift of the model product), floor.
 *   BNMF_OP_OBJECTIVE  out[0] = D_beta(V | W H + kappa)            core.objective, core.py:275-306
 *   BNMF_OP_KKT        out[0..1] = res_W, res_H                   diagnostics.py:46-59
 *   BNMF_OP_BMM_W      out = F x K  bmm_update_w(v, w, h)          updates.py:157-170
 *   BNMF_OP_BMM_H      out = K x N  bmm_update_h(v, w, h)          updates.py:173-181
 *   BNMF_OP_JMM_W      out = F x K  jmm_update_w(v, anchor, cur = h_current (K x N))   :203-220
 *   BNMF_OP_JMM_H      out = K x N  jmm_update_h(v, anchor, cur = w_current (F x K))   :223-235
 * cur and out are fp64 row-major host arrays (cur is NULL where unused). */
enum { BNMF_OP_OBJECTIVE = 0, BNMF_OP_KKT = 1, BNMF_OP_BMM_W = 2, BNMF_OP_BMM_H = 3,
       BNMF_OP_JMM_W = 4, BNMF_OP_JMM_H = 5 };
int bnmf_kernel(bnmf_ctx* ctx, int op, const bnmf_params* p, const double* cur, double* out);

#ifdef __cplusplus
}
#endif

#endif /* BNMF_H_ */
