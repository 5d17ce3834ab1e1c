// tcgen05 kind::tf32 streaming cost per MMA vs N, SS vs TS, number of
// independent accumulators, alone and with concurrent epilogue TMEM stores.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench2 mma_bench2.cu
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

template <int TS, int N, int NACC>
__global__ void __launch_bounds__(32 * 17, 1)
bench(int bg, int iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  float* sB = reinterpret_cast<float*>(dyn);
  float* sA = reinterpret_cast<float*>(dyn + 65536);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sB[i] = 0.5f;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sA[i] = 0.25f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); stop = 0; }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const uint64_t db = sdesc(smem_u32(sB), 128, 512);
    const uint64_t da = sdesc(smem_u32(sA), 128, 512);
    constexpr uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t dc = t + (s % NACC) * (256 / NACC);
          if (TS) mma_ts(dc, t + 256 + 8 * (s & 3), db + 16 * s, id, 1u);
          else mma_ss(dc, da + 16 * (s & 3), db + 16 * s, id, 1u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (bg) {
    const int q = warp & 3, g = (warp - 1) >> 2;
    const uint32_t base = t + (uint32_t(32 * q) << 16) + 384 + 32 * g;
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane + i;
    while (!stop) { tmem_st32(base, v); tmem_st_wait(); v[0] += 1.f; }
    if (v[0] == 1.5f) sink[0] = v[0];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(t);
}

long long* d; float* sink;
template <int TS, int N, int NACC>
void run(int bg) {
  long long h[148];
  const int iters = 2000;
  cudaFuncSetAttribute(bench<TS, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  bench<TS, N, NACC><<<148, 32 * 17, 96 * 1024>>>(bg, 50, d, sink);
  bench<TS, N, NACC><<<148, 32 * 17, 96 * 1024>>>(bg, iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s acc%d %s M128 N%-3d K8: %6.1f cyc/MMA (floor %d) %s\n", bg ? "+st" : "   ", NACC,
         TS ? "TS" : "SS", N, double(h[0]) / (iters * 8), N / 2, cudaGetErrorString(e));
}
template <int TS, int NACC>
void runN(int bg) { run<TS, 16, NACC>(bg); run<TS, 32, NACC>(bg); run<TS, 64, NACC>(bg); if (NACC <= 2) run<TS, 128, NACC>(bg); }

int main() {
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  for (int bg = 0; bg < 2; ++bg) {
    runN<1, 1>(bg); runN<1, 2>(bg); runN<1, 4>(bg);
    runN<0, 1>(bg); runN<0, 2>(bg); runN<0, 4>(bg);
  }
  return 0;
}
