// tcgen05 issue / pipe cost probes for the fused pass (round 2):
//   A  one issuing thread: cycles per MMA for kind::tf32 (K = 8) and kind::f16 (bf16, K = 16),
//      A operand in TMEM, N = 16 .. 128
//   B  two issuing threads (different warps, different accumulators): does the rate double?
//      (tells whether small-N MMAs are bound by the issuing thread or by the tensor pipe)
//   C  item mixes of the fused pass (Vt + side products), one issuer vs two issuers
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o mma_bench3 mma_bench3.cu
#include <cstdio>
#include "../paper_2106_15214_b200/csrc/tc_primitives.cuh"
using namespace bnmf::tc;

__device__ __forceinline__ void mma_ts_bf16(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

struct Step { int kind; uint32_t idesc; };   // kind 0 = tf32, 1 = bf16

// one issuing warp runs `prog` (nsteps MMAs per item); commit per item, wait two items behind
__device__ void issue_loop(uint32_t t, uint32_t acc0, uint64_t db, const Step* prog, int nsteps,
                           int iters, uint64_t* bar2) {
  for (int it = 0; it < iters; ++it) {
    if (it >= 2) { mbar_wait(&bar2[it & 1], ((it - 2) >> 1) & 1); tc_fence_after(); }
    if (elect_one()) {
      for (int s = 0; s < nsteps; ++s) {
        const uint32_t dc = t + acc0 + (s & 1) * 96;
        if (prog[s].kind == 0)
          mma_ts(dc, t + 384 + 8 * (s & 7), db + 16 * (s & 7), prog[s].idesc, 1u);
        else
          mma_ts_bf16(dc, t + 384 + 8 * (s & 7), db + 16 * (s & 7), prog[s].idesc, 1u);
      }
      mma_commit(&bar2[it & 1]);
    }
    __syncwarp();
  }
  mbar_wait(&bar2[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
}

// straight-line variants (compile-time program) to take the loop overhead out
template <int KIND, int N, int CNT>
__device__ void issue_fixed(uint32_t t, uint32_t acc0, uint64_t db, int iters, uint64_t* bar2) {
  constexpr uint32_t id = KIND == 0 ? idesc_tf32(128, N, 0, 0) : idesc_bf16(128, N);
  for (int it = 0; it < iters; ++it) {
    if (it >= 2) { mbar_wait(&bar2[it & 1], ((it - 2) >> 1) & 1); tc_fence_after(); }
    if (elect_one()) {
#pragma unroll
      for (int s = 0; s < CNT; ++s) {
        const uint32_t dc = t + acc0 + (s & 1) * (N < 64 ? 64 : N);
        if (KIND == 0) mma_ts(dc, t + 384 + 8 * (s & 7), db + 16 * (s & 7), id, 1u);
        else mma_ts_bf16(dc, t + 384 + 8 * (s & 7), db + 16 * (s & 7), id, 1u);
      }
      mma_commit(&bar2[it & 1]);
    }
    __syncwarp();
  }
  mbar_wait(&bar2[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
}

template <int KIND, int N>
__global__ void __launch_bounds__(32 * 12, 1)
benchA(int nissuers, int bg, int iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(dyn)[i] = 0.5f;
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); mbar_fence_init(); stop = 0; }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t db = sdesc(smem_u32(dyn), 128, 512);
  if (warp < nissuers) {
    long long t0 = clock64();
    issue_fixed<KIND, N, 8>(t, warp * 2 * (N < 64 ? 64 : N), db, iters, &bar[2 * warp]);
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x * 2 + warp] = t1 - t0; if (warp == 0) stop = 1; }
  } else if (bg && warp >= 4) {
    const int q = warp & 3, g = (warp - 4) >> 2;
    const uint32_t base = t + (uint32_t(32 * q) << 16) + 448 + 32 * g;
    float v[32];
    for (int i = 0; i < 32; ++i) v[i] = lane + i;
    while (!stop) {
      float y[32];
      tmem_ld16(t + (uint32_t(32 * q) << 16) + 256 + 16 * g, y);
      v[0] += y[1];
      tmem_st32(base, v);
      tmem_st_wait();
    }
    if (v[0] == 1.5f) sink[0] = v[0];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(t);
}

// item mixes: prog0 on warp 0 (Vt-like), prog1 on warp 1 (side-like); split = 0 runs both
// programs back to back on warp 0
__global__ void __launch_bounds__(32 * 12, 1)
benchC(const Step* p0, int n0, const Step* p1, int n1, int split, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tb;
  __shared__ Step prog[2][64];
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(dyn)[i] = 0.5f;
  if (threadIdx.x < n0) prog[0][threadIdx.x] = p0[threadIdx.x];
  if (threadIdx.x < n1) prog[split ? 1 : 0][(split ? 0 : n0) + threadIdx.x] = p1[threadIdx.x];
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); mbar_fence_init(); }
  if ((threadIdx.x >> 5) == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t db = sdesc(smem_u32(dyn), 128, 512);
  if (warp == 0 || (warp == 1 && split)) {
    long long t0 = clock64();
    issue_loop(t, warp * 192, db, prog[warp], split ? (warp ? n1 : n0) : n0 + n1, iters, &bar[2 * warp]);
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 2 + warp] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(t);
}

long long* d;
float* sink;
Step* dprog;

template <int KIND, int N>
void runA(int nissuers, int bg) {
  long long h[296];
  const int iters = 1500;
  cudaFuncSetAttribute(benchA<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  benchA<KIND, N><<<148, 32 * 12, 65536>>>(nissuers, bg, 50, d, sink);
  benchA<KIND, N><<<148, 32 * 12, 65536>>>(nissuers, bg, iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("A issuers=%d %s %s M128 N%-3d: %6.1f cyc/MMA per issuer (math floor %d) %s\n", nissuers,
         bg ? "+ld/st" : "      ", KIND ? "bf16 K16" : "tf32 K8 ", N, double(h[0]) / (iters * 8), N / 2,
         cudaGetErrorString(e));
}

void runC(const char* name, const Step* p0, int n0, const Step* p1, int n1) {
  long long h[296];
  const int iters = 1500;
  cudaMemcpy(dprog, p0, n0 * sizeof(Step), cudaMemcpyHostToDevice);
  cudaMemcpy(dprog + 64, p1, n1 * sizeof(Step), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(benchC, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int split = 0; split < 2; ++split) {
    benchC<<<148, 32 * 12, 65536>>>(dprog, n0, dprog + 64, n1, split, 50, d);
    benchC<<<148, 32 * 12, 65536>>>(dprog, n0, dprog + 64, n1, split, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("C %-44s %s: %7.1f cyc/item (%d + %d MMAs) %s\n", name, split ? "two issuers" : "one issuer ",
           double(split ? (h[0] > h[1] ? h[0] : h[1]) : h[0]) / iters, n0, n1, cudaGetErrorString(e));
  }
}

int main() {
  cudaMalloc(&d, 296 * 8);
  cudaMalloc(&sink, 4);
  cudaMalloc(&dprog, 128 * sizeof(Step));
  for (int bg = 0; bg < 2; ++bg)
    for (int ni = 1; ni <= 2; ++ni) {
      runA<0, 16>(ni, bg); runA<0, 32>(ni, bg); runA<0, 48>(ni, bg); runA<0, 64>(ni, bg);
      if (ni == 1) runA<0, 128>(ni, bg);
      runA<1, 16>(ni, bg); runA<1, 32>(ni, bg); runA<1, 48>(ni, bg); runA<1, 64>(ni, bg);
      runA<1, 96>(ni, bg);
    }
  auto T = [](int n) { return Step{0, idesc_tf32(128, n, 0, 0)}; };
  auto B = [](int n) { return Step{1, idesc_bf16(128, n)}; };
  const Step T32 = T(32), T16 = T(16), T64 = T(64), B16 = B(16), B32 = B(32), B48 = B(48), B64 = B(64),
             B96 = B(96);
  {  // current item: Vt 6 x tf32 N32; side 2 x 4 x (tf32 N32 + tf32 N16)
    Step vt[6] = {T32, T32, T32, T32, T32, T32};
    Step sd[16] = {T32, T16, T32, T16, T32, T16, T32, T16, T32, T16, T32, T16, T32, T16, T32, T16};
    runC("3xTF32 (current)", vt, 6, sd, 16);
    Step sd1[8] = {T32, T32, T32, T32, T32, T32, T32, T32};
    runC("3xTF32 Vt, single-TF32 Z side", vt, 6, sd1, 8);
    Step sd2[12] = {T32, T32, T32, T32, T32, T32, T32, T32, B16, B16, B16, B16};
    runC("3xTF32 Vt, Z lo terms in bf16", vt, 6, sd2, 12);
    Step vt2[4] = {T32, T32, B32, B32};
    runC("Vt cross terms bf16, Z lo terms bf16", vt2, 4, sd2, 12);
    Step vt3[3] = {B96, B64, B32};
    Step sd3[8] = {B48, B48, B32, B32, B48, B48, B32, B32};
    runC("all bf16: Vt 3x3 pieces, Z 2 pieces x B 3", vt3, 3, sd3, 8);
    Step sd4[12] = {B48, B48, B32, B32, B16, B16, B48, B48, B32, B32, B16, B16};
    runC("all bf16: Vt 3x3 pieces, Z 3 pieces x B 3", vt3, 3, sd4, 12);
    Step vt12[12] = {T32, T32, T32, T32, T32, T32, T32, T32, T32, T32, T32, T32};
    Step sd5[16] = {T64, T32, T64, T32, T64, T32, T64, T32, T64, T32, T64, T32, T64, T32, T64, T32};
    runC("rank 32: Vt 12 x N32, side 2 x 4 x (N64 + N32)", vt12, 12, sd5, 16);
  }
  return 0;
}
