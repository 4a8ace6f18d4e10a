// TMEM read bandwidth per SM: W warps (lane quarter w % 4) repeatedly load
// six 32x32b.x4 column groups (the gather epilogue's tmem_ld4x6_wait) and
// wait; optionally with one thread issuing the gather's UMMA pass pattern
// concurrently (A from TMEM, B from shared memory).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_probe tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2407_06834_b200/csrc/nld_umma.cuh"

using namespace nld::umma;

__global__ void __launch_bounds__(640, 1) k_ld(int warps, int iters, int mma, long long* cyc,
                                              unsigned* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  for (int e = threadIdx.x; e < 64 * 1024; e += blockDim.x) sm[e] = (uint8_t)(e * 7 + 3);
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long t0 = clock64();
  if (warp < warps) {
    unsigned acc = 0;
    const uint32_t tl = t + ((uint32_t)((warp & 3) * 32) << 16);
    for (int i = 0; i < iters; ++i) {
      uint32_t d[6][4];
      tmem_ld4x6_wait(tl + (uint32_t)(((i + warp) & 7) * 8 % 192), 32, d);
#pragma unroll
      for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc ^= d[a][b];
    }
    if (acc == 0x12345) sink[threadIdx.x] = acc;
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = clock64() - t0;
  } else if (warp == warps && mma && lane == 0) {
    const uint32_t bB = smem_u32(sm);
    const int passes = 4 * mma;
    for (int g = 0; g < passes; ++g) {
#pragma unroll
      for (int p = 0; p < 6; ++p)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          mma_i8_ta(t + 256 + p * 32 - 256 + 0 * g, t + 384 + p * 16 + ks * 8,
                    make_sdesc(bB + ((g * 6) & 15) * 2048 + ks * 256, 128, 512),
                    idesc_i8(128, (6 - p) * 32), (p > 0 || ks > 0));
    }
    commit(&mbar);
    mbar_wait(&mbar, 0);
    cyc[blockIdx.x * 32 + 31] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

int main() {
  long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, sizeof(long long) * 148 * 32);
  cudaMalloc(&sink, sizeof(unsigned) * 640);
  cudaFuncSetAttribute(k_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  long long h[148 * 32];
  for (int mma = 0; mma <= 1; ++mma)
    for (int w : {1, 4, 8, 16}) {
      const int iters = 2000;
      const int mm = mma ? 500 : 0;   // 500 tiles' worth of passes
      for (int rep = 0; rep < 2; ++rep)
        k_ld<<<148, 640, 64 * 1024>>>(w, iters, mm, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int k = 0; k < w; ++k) mx = h[k] > mx ? h[k] : mx;
      const double bytes = (double)w * iters * 6 * 32 * 4 * 4;   // per CTA
      printf("mma=%d warps=%2d: %lld cycles, TMEM read %.1f B/clk/SM; UMMA thread %lld cycles "
             "(%.0f per 4-pass tile)\n", mma, w, mx, bytes / mx, mma ? h[31] : 0LL,
             mma ? (double)h[31] / 500 : 0.0);
    }
  return 0;
}
