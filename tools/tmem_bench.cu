// TMEM load/store throughput per SM (tcgen05.ld / tcgen05.st, 32x32b shapes).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

__global__ void __launch_bounds__(32 * 17, 1) bench(int mode, int nw, int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  unsigned long long t0 = 0, t1 = 0;
  if (warp >= 1 && warp <= nw) {
    const int e = warp - 1, q = warp & 3, g = e >> 2;
    const uint32_t base = tmem + (uint32_t(32 * q) << 16);
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane + i;
    __syncwarp();
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
        float y[8];
        tmem_ld8(base + 8 * g + 32 * (it & 7), y);
        acc += y[0] + y[7];
      } else if (mode == 1) {
        tmem_ld16(base + 16 * (g & 1) + 32 * (it & 7), v);
        acc += v[0] + v[15];
      } else if (mode == 2) {
        v[0] += 1.f;
        tmem_st8(base + 8 * g + 32 * (it & 7), v);
        tmem_st_wait();
      } else if (mode == 3) {
        v[0] += 1.f;
        tmem_st32(base + 32 * g + 128 * (it & 1), v);
        tmem_st_wait();
      } else if (mode == 4) {
        float y[8];
        tmem_ld8(base + 8 * g + 32 * (it & 1), y);
        v[0] += y[3];
        tmem_st32(base + 64 + 32 * g + 128 * (it & 1), v);
        tmem_st_wait();
      } else if (mode == 5) {   // 4 x st8 (the current kernel's Z store)
        v[0] += 1.f;
        tmem_st8(base + 128 + 8 * g, v);
        tmem_st8(base + 160 + 8 * g, v + 8);
        tmem_st8(base + 192 + 8 * g, v + 16);
        tmem_st8(base + 224 + 8 * g, v + 24);
        tmem_st_wait();
      } else if (mode == 6) {   // st32 without per-iteration wait
        v[0] += 1.f;
        tmem_st32(base + 32 * g + 128 * (it & 1), v);
        if ((it & 7) == 7) tmem_st_wait();
      }
    }
    tmem_st_wait();
    t1 = clock64();
    if (lane == 0) out[blockIdx.x * 32 + e] = t1 - t0;
    for (int i = 0; i < 32; ++i) acc += v[i];
  }
  if (acc == 1234.5f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 32 * 8);
  float* sink; cudaMalloc(&sink, 4);
  unsigned long long h[148 * 32];
  const char* names[] = {"ld x8", "ld x16", "st x8", "st x32", "ld x8 + st x32", "4 x st x8", "st x32 (wait/8)"};
  const int bytes[] = {1024, 2048, 1024, 4096, 5120, 4096, 4096};
  for (int mode = 0; mode < 7; ++mode)
    for (int nw : {4, 8, 16}) {
      const int iters = 4096;
      bench<<<148, 32 * 17>>>(mode, nw, iters, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bpc = double(bytes[mode]) * nw * iters / mx;
      printf("%-18s warps %2d: %7.1f cyc/iter/warp  %6.1f B/cyc/SM (%s)\n", names[mode], nw,
             double(mx) / iters, bpc, cudaGetErrorString(e));
    }
  return 0;
}
