// Throughput of the tcgen05 kind::tf32 shapes the fused pass issues.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench mma_bench.cu
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

template <int MODE>  // 0: TS M128 N16, 1: SS M128 N32, 2: TS M128 N32, 3: SS M128 N16, 4: TS M128 N64
__global__ void __launch_bounds__(128) bench(long long* out, int iters) {
  __shared__ __align__(1024) float sB[64 * 64];
  __shared__ __align__(1024) float sA[128 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 64 * 64; i += 128) sB[i] = 0.5f;
  for (int i = threadIdx.x; i < 128 * 16; i += 128) sA[i] = 0.25f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<256>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  long long t0 = clock64();
  if ((threadIdx.x >> 5) == 0) {
    const uint64_t db = sdesc(smem_u32(sB), 128, 512);
    const uint64_t da = sdesc(smem_u32(sA), 128, 512);
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          if (MODE == 0) mma_ts(t + 0, t + 128 + 8 * (s & 3), db + 16 * s, idesc_tf32(128, 16, 0, 0), 1u);
          if (MODE == 1) mma_ss(t + 0, da + 16 * (s & 1), db + 16 * s, idesc_tf32(128, 32, 0, 0), 1u);
          if (MODE == 2) mma_ts(t + 0, t + 128 + 8 * (s & 3), db + 16 * s, idesc_tf32(128, 32, 0, 0), 1u);
          if (MODE == 3) mma_ss(t + 0, da + 16 * (s & 1), db + 16 * s, idesc_tf32(128, 16, 0, 0), 1u);
          if (MODE == 4) mma_ts(t + 0, t + 128 + 8 * (s & 3), db + 16 * s, idesc_tf32(128, 64, 0, 0), 1u);
        }
        mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, it & 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc<256>(t);
}

template <int MODE>
__global__ void __launch_bounds__(128) bench_nowait(long long* out, int iters) {
  __shared__ __align__(1024) float sB[64 * 64];
  __shared__ __align__(1024) float sA[128 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  for (int i = threadIdx.x; i < 64 * 64; i += 128) sB[i] = 0.5f;
  for (int i = threadIdx.x; i < 128 * 16; i += 128) sA[i] = 0.25f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<256>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  long long t0 = clock64();
  if ((threadIdx.x >> 5) == 0) {
    const uint64_t db = sdesc(smem_u32(sB), 128, 512);
    const uint64_t da = sdesc(smem_u32(sA), 128, 512);
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          if (MODE == 0) mma_ts(t + 0, t + 128 + 8 * (s & 3), db + 16 * s, idesc_tf32(128, 16, 0, 0), 1u);
          if (MODE == 1) mma_ss(t + 0, da + 16 * (s & 1), db + 16 * s, idesc_tf32(128, 32, 0, 0), 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 0) tmem_dealloc<256>(t);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  long long h[148];
  const int iters = 2000;
  auto run = [&](auto kern, const char* name, int nmma) {
    kern<<<148, 128>>>(d, 10);
    kern<<<148, 128>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-28s %s  cycles/MMA = %.1f\n", name, cudaGetErrorString(e), double(h[0]) / (iters * nmma));
  };
  run(bench<0>, "TS M128 N16 (sync/8)", 8);
  run(bench<1>, "SS M128 N32 (sync/8)", 8);
  run(bench<2>, "TS M128 N32 (sync/8)", 8);
  run(bench<3>, "SS M128 N16 (sync/8)", 8);
  run(bench<4>, "TS M128 N64 (sync/8)", 8);
  run(bench_nowait<0>, "TS M128 N16 stream", 8);
  run(bench_nowait<1>, "SS M128 N32 stream", 8);
  return 0;
}
