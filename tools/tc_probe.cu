// Probe of the tcgen05 / TMA conventions used by the fused pass (run once on a
// B200):  nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu -lcuda
//   test 1: D = A * B^T, A and B K-major core-tiled in smem (SS)
//   test 2: D = A * B, A in TMEM, B MN-major core-tiled in smem (TS)
//   test 3: TMA boxes [32 x 128] (no swizzle) and [128 x 32] (128B swizzle)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"

using namespace bnmf::tc;

__device__ float A1(int m, int k) { return float((m + 2 * k) % 7 - 3); }
__device__ float B1(int n, int k) { return float((3 * n + k) % 5 - 2); }
__device__ float A2(int m, int k) { return float((5 * m + k) % 9 - 4); }
__device__ float B2(int k, int n) { return float((k + 7 * n) % 6 - 2) * 0.5f; }

__global__ void __launch_bounds__(128) probe(float* d1, float* d2, float* d3, float* d4, float* tma_h, float* tma_w,
                                             const __grid_constant__ CUtensorMap mh,
                                             const __grid_constant__ CUtensorMap mw) {
  __shared__ __align__(1024) float sA[128 * 16];
  __shared__ __align__(1024) float sB[32 * 16];
  __shared__ __align__(1024) float sB2[32 * 16];
  __shared__ __align__(1024) float sA2[128 * 32];
  __shared__ __align__(1024) float sB2k[16 * 32];
  extern __shared__ __align__(1024) float dyn[];
  float* sTh = dyn;
  float* sTw = dyn + 32 * 128;
  __shared__ __align__(8) uint64_t bar[3];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  char* cA = reinterpret_cast<char*>(sA);
  char* cB = reinterpret_cast<char*>(sB);
  char* cB2 = reinterpret_cast<char*>(sB2);
  for (int i = t; i < 128 * 16; i += 128) {
    int m = i / 16, k = i % 16;
    *reinterpret_cast<float*>(cA + core_off(m, k)) = A1(m, k);
  }
  for (int i = t; i < 32 * 16; i += 128) {
    int n = i / 16, k = i % 16;
    *reinterpret_cast<float*>(cB + core_off(n, k)) = B1(n, k);
    int kk = i / 16, nn = i % 16;  // B2 rows = K-dim (32), cols = N (16)
    *reinterpret_cast<float*>(cB2 + core_off(kk, nn)) = B2(kk, nn);
  }
  // A2 K-major core-tiled [128 x 32] (4 groups of 16 k -> 2 tiles of 16 wide each)
  char* cA2 = reinterpret_cast<char*>(sA2);
  char* cB2k = reinterpret_cast<char*>(sB2k);
  for (int i = t; i < 128 * 32; i += 128) {
    int m = i / 32, k = i % 32;
    // k-tile kt (16 wide) stored as separate [128 x 16] core-tiled blocks of 8 KB
    *reinterpret_cast<float*>(cA2 + (k / 16) * 8192 + core_off(m, k % 16)) = A2(m, k);
  }
  for (int i = t; i < 16 * 32; i += 128) {
    int n = i / 32, k = i % 32;
    *reinterpret_cast<float*>(cB2k + (k / 16) * 1024 + core_off(n, k % 16)) = B2(k, n);
  }
  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<128>(&tbase);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  // A2 into TMEM columns [64, 96)
  {
    float v[16];
    for (int half = 0; half < 2; ++half) {
      for (int j = 0; j < 16; ++j) v[j] = A2(t, 16 * half + j);
      tmem_st16(tb + ((warp * 32) << 16) + 64 + 16 * half, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    const uint32_t id1 = idesc_tf32(128, 32, 0, 0);
    for (int s = 0; s < 2; ++s)
      mma_ss(tb + 0, sdesc(smem_u32(cA) + 256 * s, 128, 512), sdesc(smem_u32(cB) + 256 * s, 128, 512),
             id1, s);
    const uint32_t id2 = idesc_tf32(128, 16, 0, 1);
    for (int s = 0; s < 4; ++s)
      mma_ts(tb + 32, tb + 64 + 8 * s, sdesc(smem_u32(cB2) + 512 * s, 512, 128), id2, s);
    // (b) SS: A2 smem K-major, B2 MN-major  -> cols 48..63
    for (int s = 0; s < 4; ++s)
      mma_ss(tb + 48, sdesc(smem_u32(cA2) + (s / 2) * 8192 + 256 * (s % 2), 128, 512),
             sdesc(smem_u32(cB2) + 512 * s, 512, 128), id2, s);
    for (int s = 0; s < 4; ++s)
      mma_ts(tb + 112, tb + 64 + 8 * s, sdesc(smem_u32(cB2) + 512 * s, 128, 512), id2, s);
    // (a) TS: A2 in TMEM, B2 K-major -> cols 96..111
    const uint32_t id3 = idesc_tf32(128, 16, 0, 0);
    for (int s = 0; s < 4; ++s)
      mma_ts(tb + 96, tb + 64 + 8 * s, sdesc(smem_u32(cB2k) + (s / 2) * 1024 + 256 * (s % 2), 128, 512), id3, s);
    mma_commit(&bar[0]);
    // TMA
    mbar_expect_tx(&bar[1], 32 * 128 * 4);
    tma_load_2d(sTh, &mh, &bar[1], 64, 32);
    mbar_expect_tx(&bar[2], 128 * 32 * 4);
    tma_load_2d(sTw, &mw, &bar[2], 160, 0);
  }
  mbar_wait(&bar[0], 0);
  tc_fence_after();
  {
    float v[16];
    for (int c = 0; c < 2; ++c) {
      tmem_ld16(tb + ((warp * 32) << 16) + 16 * c, v);
      for (int j = 0; j < 16; ++j) d1[t * 32 + 16 * c + j] = v[j];
    }
    tmem_ld16(tb + ((warp * 32) << 16) + 32, v);
    for (int j = 0; j < 16; ++j) d2[t * 16 + j] = v[j];
    tmem_ld16(tb + ((warp * 32) << 16) + 48, v);
    for (int j = 0; j < 16; ++j) d3[t * 16 + j] = v[j];
    tmem_ld16(tb + ((warp * 32) << 16) + 96, v);
    for (int j = 0; j < 16; ++j) d4[t * 16 + j] = v[j];
    tmem_ld16(tb + ((warp * 32) << 16) + 112, v);
    for (int j = 0; j < 16; ++j) d2[t * 16 + j] = v[j];
    tmem_ld16(tb + ((warp * 32) << 16) + 64, v);
    if (t == 5) printf("A2 tmem readback lane5: %g %g %g (want %g %g %g)\n", v[0], v[1], v[2], A2(5,0), A2(5,1), A2(5,2));
  }
  mbar_wait(&bar[1], 0);
  mbar_wait(&bar[2], 0);
  for (int i = t; i < 32 * 128; i += 128) tma_h[i] = sTh[i];
  for (int i = t; i < 128 * 32; i += 128) tma_w[i] = sTw[i];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<128>(tb);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  const int F = 64, N = 200;
  std::vector<float> hv(F * N);
  for (int i = 0; i < F * N; ++i) hv[i] = float(i);
  float *dv, *d1, *d2, *d3, *d4, *th, *tw;
  cudaMalloc(&d3, 128 * 16 * 4);
  cudaMalloc(&d4, 128 * 16 * 4);
  cudaMalloc(&dv, F * N * 4);
  cudaMemcpy(dv, hv.data(), F * N * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&d1, 128 * 32 * 4);
  cudaMalloc(&d2, 128 * 16 * 4);
  cudaMalloc(&th, 32 * 128 * 4);
  cudaMalloc(&tw, 128 * 32 * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap mh, mw;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)F};
  cuuint64_t strides[1] = {(cuuint64_t)N * 4};
  cuuint32_t boxh[2] = {128, 32}, boxw[2] = {32, 128}, es[2] = {1, 1};
  CUresult r1 = enc(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dv, dims, strides, boxh, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dv, dims, strides, boxw, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", int(r1), int(r2));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(d1, d2, d3, d4, th, tw, mh, mw);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> h1(128 * 32), h2(128 * 16), hh(32 * 128), hw(128 * 32);
  cudaMemcpy(h1.data(), d1, h1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), d2, h2.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<float> h3(128 * 16), h4(128 * 16);
  cudaMemcpy(h3.data(), d3, h3.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h4.data(), d4, h4.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hh.data(), th, hh.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hw.data(), tw, hw.size() * 4, cudaMemcpyDeviceToHost);
  auto a1 = [](int m, int k) { return float((m + 2 * k) % 7 - 3); };
  auto b1 = [](int n, int k) { return float((3 * n + k) % 5 - 2); };
  auto a2 = [](int m, int k) { return float((5 * m + k) % 9 - 4); };
  auto b2 = [](int k, int n) { return float((k + 7 * n) % 6 - 2) * 0.5f; };
  int bad1 = 0, bad2 = 0, badh = 0, badw = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      float s = 0;
      for (int k = 0; k < 16; ++k) s += a1(m, k) * b1(n, k);
      if (h1[m * 32 + n] != s) { if (bad1 < 5) printf("t1 m%d n%d got %g want %g\n", m, n, h1[m * 32 + n], s); ++bad1; }
    }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      float s = 0;
      for (int k = 0; k < 32; ++k) s += a2(m, k) * b2(k, n);
      if (h2[m * 16 + n] != s) { if (bad2 < 5) printf("t2 m%d n%d got %g want %g\n", m, n, h2[m * 16 + n], s); ++bad2; }
    }
  int bad3 = 0, bad4 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      float s = 0;
      for (int k = 0; k < 32; ++k) s += a2(m, k) * b2(k, n);
      if (h3[m * 16 + n] != s) { if (bad3 < 3) printf("t3 m%d n%d got %g want %g\n", m, n, h3[m * 16 + n], s); ++bad3; }
      if (h4[m * 16 + n] != s) { if (bad4 < 3) printf("t4 m%d n%d got %g want %g\n", m, n, h4[m * 16 + n], s); ++bad4; }
    }
  printf("bad3 (SS, B MN-major)=%d bad4 (TS, B K-major)=%d\n", bad3, bad4);
  for (int r = 0; r < 32; ++r)
    for (int c = 0; c < 128; ++c) {
      float want = hv[(32 + r) * N + 64 + c];
      if (hh[r * 128 + c] != want) { if (badh < 5) printf("th r%d c%d got %g want %g\n", r, c, hh[r * 128 + c], want); ++badh; }
    }
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 32; ++c) {
      int chunk = c / 4, phys = chunk ^ (r & 7);
      float got = hw[r * 32 + phys * 4 + (c & 3)];
      float want = (r < F && 160 + c < N) ? hv[r * N + 160 + c] : 0.f;
      if (got != want) { if (badw < 5) printf("tw r%d c%d got %g want %g\n", r, c, got, want); ++badw; }
    }
  printf("bad: t1=%d t2=%d tma_h=%d tma_w=%d\n", bad1, bad2, badh, badw);
  return (bad1 || bad2 || badh || badw) ? 2 : 0;
}
