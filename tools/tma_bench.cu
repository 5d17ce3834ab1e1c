// TMA ring streaming bandwidth for the fused pass's box shapes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

constexpr int NEPI = 16;
// mode 0: H boxes [32 rows x 128 cols] only; 1: W boxes [128 x 32] swizzled only;
// 2: per block 8 H + 8 W (the fused pass order); 3: like 2 with an L2 prefetch 2 blocks ahead
__global__ void __launch_bounds__(32 * (1 + NEPI), 1)
ring(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mw, int nblocks,
     int nstage, int mode, float* sink) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NEPI); }
    mbar_fence_init();
  }
  __syncthreads();
  const int per = (mode == 0 || mode == 1) ? 16 : 16;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0; uint32_t ph = 0;
      for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
        if (mode == 3) {
          int bp = b + 2 * gridDim.x;
          if (bp < nblocks) for (int t = 0; t < 2; ++t) for (int u = 0; u < 4; ++u) tma_prefetch_l2_2d(&mw, bp * 128 + 32 * u, 128 * t);
        }
        for (int i = 0; i < per; ++i) {
          mbar_wait(&empty[stage], ph ^ 1);
          mbar_expect_tx(&full[stage], 16384);
          bool h = (mode == 0) || ((mode >= 2) && i < 8);
          if (h) tma_load_2d(sm + stage * 16384, &mh, &full[stage], b * 128, 32 * (i & 7));
          else tma_load_2d(sm + stage * 16384, &mw, &full[stage], b * 128 + 32 * (i & 3), 128 * ((i >> 2) & 1));
          if (++stage == nstage) { stage = 0; ph ^= 1; }
        }
      }
    }
  } else {
    int stage = 0; uint32_t ph = 0; float acc = 0.f;
    const uint32_t base = smem_u32(sm);
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
      for (int i = 0; i < per; ++i) {
        mbar_wait(&full[stage], ph);
        acc += lds_f32(base + stage * 16384 + ((threadIdx.x - 32) * 4 % 16384));
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == nstage) { stage = 0; ph ^= 1; }
      }
    }
    if (acc == 12345.f) sink[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
int main() {
  const long F = 256, N = 4194304;
  float* v; cudaMalloc(&v, F * N * 4); cudaMemset(v, 0, F * N * 4);
  float* sink; cudaMalloc(&sink, 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap mh, mw;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)F}, strides[1] = {(cuuint64_t)N * 4};
  cuuint32_t bh[2] = {128, 32}, bw[2] = {32, 128}, es[2] = {1, 1};
  enc(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, v, dims, strides, bh, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, v, dims, strides, bw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int nblocks = N / 128;
  for (int mode = 0; mode < 4; ++mode)
    for (int ns : {3, 5, 8, 12}) {
      ring<<<148, 32 * (1 + NEPI), 200 * 1024>>>(mh, mw, nblocks, ns, mode, sink);
      cudaEventRecord(a);
      ring<<<148, 32 * (1 + NEPI), 200 * 1024>>>(mh, mw, nblocks, ns, mode, sink);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = double(nblocks) * 16 * 16384;
      printf("mode %d nstage %2d: %.3f ms  %.0f GB/s smem-delivered (%s)\n", mode, ns, ms, bytes / ms / 1e6, cudaGetErrorString(e));
    }
  return 0;
}
