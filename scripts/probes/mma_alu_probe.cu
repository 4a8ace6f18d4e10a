// Does CUDA-core work slow down while the tensor core runs?  W warps run the
// gather epilogue's combine arithmetic on register data (no TMEM, no shared
// memory, no global memory) for a fixed number of iterations, with and
// without one thread issuing the gather's UMMA pass pattern back to back on
// the same SM.  Reported: cycles of the arithmetic warps and of the UMMA
// thread, each alone and together.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_alu_probe mma_alu_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2407_06834_b200/csrc/nld_umma.cuh"

using namespace nld::umma;

__global__ void __launch_bounds__(640, 1) k(int warps, int iters, int tiles, int kind,
                                            long long* cyc, double* sink) {
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
  if (warp >= 4 && warp < 4 + warps) {
    int d[4][6];
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 6; ++q) d[i][q] = (int)(threadIdx.x * 31 + i * 7 + q);
    double s[4] = {0, 0, 0, 0};
    const double a = 1.0 + lane * 1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (kind == 0) {   // the int64 combine + I2F + DFMA
          const int x01 = d[i][0] * 256 + d[i][1], x23 = d[i][2] * 256 + d[i][3],
                    x45 = d[i][4] * 256 + d[i][5];
          const long long T = (long long)x23 * 65536 + (long long)x45 + ((long long)x01 << 32);
          s[i] = fma((double)T, a, s[i]);
        } else if (kind == 1) {   // integer only
          d[i][1] = d[i][0] * 256 + d[i][1];
          d[i][3] = d[i][2] * 256 + d[i][3];
          d[i][5] = (d[i][4] * 256 + d[i][5]) ^ d[i][1];
        } else {                  // fp64 only
          s[i] = fma(s[i], a, 0.25);
          s[i] = fma(s[i], a, 0.5);
        }
        d[i][0] += it;
        d[i][4] ^= it;
      }
    }
    if (s[0] + s[1] + s[2] + s[3] + d[0][1] + d[1][3] + d[2][5] + d[3][1] == 12345.678)
      sink[threadIdx.x] = s[0];
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = clock64() - t0;
  } else if (warp == 0 && tiles && lane == 0) {
    const uint32_t bB = smem_u32(sm);
    for (int g = 0; g < 4 * tiles; ++g) {
#pragma unroll
      for (int p = 0; p < 6; ++p)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
          mma_i8_ta(t + p * 32, t + 384 + p * 16 + ks * 8,
                    make_sdesc(bB + ((g * 6) & 15) * 2048 + ks * 256, 128, 512),
                    idesc_i8(128, (6 - p) * 32), (p > 0 || ks > 0));
    }
    commit(&mbar);
    mbar_wait(&mbar, 0);
    cyc[blockIdx.x * 32 + 0] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

int main() {
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, sizeof(long long) * 148 * 32);
  cudaMalloc(&sink, sizeof(double) * 640);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  long long h[148 * 32];
  const char* names[3] = {"combine (IMAD, IMAD.WIDE, I2F.S64, DFMA)", "integer only", "fp64 only"};
  for (int kind = 0; kind < 3; ++kind)
    for (int w : {8, 12}) {
      const int iters = 20000;
      long long alu[2] = {0, 0}, mma[2] = {0, 0};
      for (int tiles : {0, 2000}) {
        for (int rep = 0; rep < 2; ++rep) k<<<148, 640, 64 * 1024>>>(w, iters, tiles, kind, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int q = 4; q < 4 + w; ++q) mx = h[q] > mx ? h[q] : mx;
        alu[tiles ? 1 : 0] = mx;
        mma[tiles ? 1 : 0] = tiles ? h[0] : 0;
      }
      for (int rep = 0; rep < 2; ++rep) k<<<148, 640, 64 * 1024>>>(0, iters, 2000, kind, cyc, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%-42s %2d warps: arithmetic alone %lld cycles, beside UMMAs %lld (x%.2f); "
             "UMMA 2000 tiles alone %lld, beside the arithmetic %lld (x%.2f)\n",
             names[kind], w, alu[0], alu[1], (double)alu[1] / alu[0], h[0], mma[1],
             (double)mma[1] / h[0]);
    }
  return 0;
}
