// Measured tensor peaks of this B200 for the roofline denominators of configs 1-3
// (BASELINE.md section 3 asks for P_tensor measured on the box):
//   1. tcgen05.mma kind::tf32, M128 N256 K8, operands in shared memory, one issuing thread per
//      SM, all 148 SMs -> dense TF32 TFLOP/s (the 3xTF32 products of the passes run at a third)
//   2. the same with N = 32 (the width of the passes' side products): issue-bound rate
//   3. mma.sync.m8n8k4.f64 (DMMA), 8 warps x 8 independent accumulators per SM, 4 CTAs per SM
//      -> FP64 tensor TFLOP/s (the fp64 reference-order kernels)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tensor_peaks tensor_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

template <int N>
__global__ void __launch_bounds__(128, 1) tf32_peak(int iters, int per_commit) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(dyn)[i] = 0.5f;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  if ((threadIdx.x >> 5) == 0) {
    // A: 128 rows x 8 tf32 (core matrices of 8 rows x 16 B), B: N rows x 8 tf32, both K-major
    const uint64_t da = sdesc(smem_u32(dyn), 128, 256);
    const uint64_t db = sdesc(smem_u32(dyn) + 16384, 128, 256);
    constexpr uint32_t id = idesc_tf32(128, N, 0, 0);
    for (int it = 0; it < iters; ++it) {
      if (it >= 2) { mbar_wait(&bar[it & 1], ((it - 2) >> 1) & 1); tc_fence_after(); }
      if (elect_one()) {
        for (int s = 0; s < per_commit; ++s) mma_ss(t + (s & 1) * 256, da, db, id, 1u);
        mma_commit(&bar[it & 1]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc<512>(t);
}

__global__ void __launch_bounds__(256) dmma_peak(int iters, double* sink) {
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[0] = s;
}

template <typename F>
static float time_ms(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  printf("%s, %d SMs\n", p.name, sms);
  double* sink; cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(tf32_peak<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66560);
  cudaFuncSetAttribute(tf32_peak<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66560);
  {
    const int iters = 2000, pc = 16;
    float ms = time_ms([&] { tf32_peak<256><<<sms, 128, 66560>>>(iters, pc); }, 5);
    double fl = 2.0 * 128 * 256 * 8 * double(iters) * pc * sms;
    printf("tcgen05 kind::tf32 M128 N256 K8 (SS), %d SMs: %.3f ms, %.1f TFLOP/s dense TF32; 3xTF32 effective %.1f TFLOP/s\n",
           sms, ms, fl / ms * 1e-9, fl / ms * 1e-9 / 3.0);
    ms = time_ms([&] { tf32_peak<32><<<sms, 128, 66560>>>(iters, pc); }, 5);
    fl = 2.0 * 128 * 32 * 8 * double(iters) * pc * sms;
    printf("tcgen05 kind::tf32 M128 N32  K8 (SS), %d SMs: %.3f ms, %.1f TFLOP/s (one issuing thread per SM, issue-bound)\n",
           sms, ms, fl / ms * 1e-9);
  }
  {
    const int iters = 20000;
    float ms = time_ms([&] { dmma_peak<<<sms * 4, 256>>>(iters, sink); }, 5);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * double(iters) * 8 * (sms * 4);
    printf("mma.sync.m8n8k4.f64 (DMMA), %d CTAs x 8 warps x 8 accumulators: %.3f ms, %.2f TFLOP/s FP64\n",
           sms * 4, ms, fl / ms * 1e-9);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
