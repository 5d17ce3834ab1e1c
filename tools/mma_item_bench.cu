// Tensor-pipe time of one fused-pass item: 6 Vt MMAs (TS M128 N32) + 2 x
// (4 x [TS N32 + TS N16]) side MMAs, exactly as fused_tc_kernel.cuh issues
// them; streaming (commit per item, wait two items behind).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_item_bench mma_item_bench.cu
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/fused_tc_kernel.cuh"
using namespace bnmf::ftc;
using namespace bnmf::tc;

__global__ void __launch_bounds__(32 * 18, 1) bench(int iters, int mode, long long* out, float* sink) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  const uint32_t sb = smem_u32(dyn);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<float*>(dyn)[i] = 0.5f;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); stop = 0; }
  if ((threadIdx.x >> 5) == 1) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t id32 = idesc_tf32(128, 32, 0, 0), id16 = idesc_tf32(128, 16, 0, 0);
  const uint64_t d_wa = sdesc(sb, 128, 512);
  const uint64_t d_c1 = sdesc(sb + 16384, 128, 4096);
  const uint64_t d_c2 = sdesc(sb + 32768, 128, 4096);
  if (warp == 1) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (it >= 2) { mbar_wait(&bar[it & 1], ((it - 2) >> 1) & 1); tc_fence_after(); }
      if (mode == 4) tc_fence_after();
      if (mode == 5) { tc_fence_after(); tc_fence_after(); tc_fence_after(); }
      const int idx = it & 3;
      const uint32_t zb = tmem + TM_Z + 128 * (it & 1);
      if (elect_one()) {
        if (mode != 2 && mode != 6) issue_vt(tmem + TM_D + 32 * (it & 1), tmem + TM_HP, tmem + TM_HP + 16,
                                dplus(d_wa, idx * 2048), dplus(d_wa, idx * 2048 + HILO), id32);
        if (mode != 1) {
          issue_side(tmem + TM_ACCH, zb, dplus(d_c1, idx * 1024), id32, id16, idx == 0);
          issue_side(tmem + TM_ACCH + 32, zb + 16, dplus(d_c2, idx * 1024), id32, id16, idx == 0);
        }
        mma_commit(&bar[it & 1]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (warp >= 2 && mode == 3) {
    // epilogue-like TMEM traffic: ld x8 + st x32 per "item"
    const int q = warp & 3, g = (warp - 2) >> 2;
    const uint32_t base = tmem + (uint32_t(32 * q) << 16);
    float z[32];
    for (int i = 0; i < 32; ++i) z[i] = lane * 0.1f + i;
    while (!stop) {
      float y[8];
      tmem_ld8(base + TM_D + 8 * g, y);
      z[0] += y[2];
      tmem_st32(base + TM_Z + 128 + 32 * g, z);   // buffer 1 region (harmless)
      tmem_st_wait();
    }
    if (z[0] == 1.5f) sink[0] = z[0];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * 8);
  float* sink; cudaMalloc(&sink, 4);
  long long h[148];
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  const char* nm[] = {"Vt + side", "Vt only", "side only", "Vt + side + epilogue TMEM load",
                      "+1 fence::after_thread_sync", "+3 fences", "side only (2 acc)"};
  for (int mode = 0; mode < 6; ++mode) {
    const int iters = 4000;
    bench<<<148, 32 * 18, 98304>>>(50, mode, d, sink);
    bench<<<148, 32 * 18, 98304>>>(iters, mode, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s %7.1f cycles/item (%s)\n", nm[mode], double(h[0]) / iters, cudaGetErrorString(e));
  }
  return 0;
}
