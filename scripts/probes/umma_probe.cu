// (1) Throughput of the gather's UMMA issue patterns, A from TMEM, B from
//     shared memory, one CTA per SM, issuer only: cycles per 128-node tile for
//     4-rhs passes (4 x 12 UMMAs, N = (6 - p) 32) and 2-rhs passes
//     (8 x 12 UMMAs, N = (6 - p) 16).
// (2) WAR hazard: does a tcgen05.cp into TMEM columns that earlier UMMAs of the
//     same thread read as their A operand wait for those UMMAs?  D must equal
//     the product with the OLD A contents.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_probe umma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "../../paper_2407_06834_b200/csrc/nld_umma.cuh"

using namespace nld::umma;

__device__ __forceinline__ int canon64(int row, int k) {
  return (row >> 3) * 512 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

__global__ void __launch_bounds__(128, 1) k_rate(int rhs_per_pass, int tiles, long long* cyc) {
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
  if (threadIdx.x == 0) {
    const uint32_t bB = smem_u32(sm);
    const int passes = 16 / rhs_per_pass;
    const int rows = rhs_per_pass * 8;           // N per digit slice
    const int acc = 6 * rows;
    const long long t0 = clock64();
    for (int g = 0; g < tiles; ++g) {
      for (int ps = 0; ps < passes; ++ps) {
        const uint32_t dcol = t + (uint32_t)(((g * passes + ps) & 1) * acc);
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            mma_i8_ta(dcol + p * rows, t + 384 + p * 16 + ks * 8,
                      make_sdesc(bB + ((ps * 6) & 15) * 2048 + ks * 256, 128, 512),
                      idesc_i8(128, (6 - p) * rows), (p > 0 || ks > 0));
      }
    }
    commit(&mbar);
    mbar_wait(&mbar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

// WAR test: A (128 x 32 int8) copied to TMEM cols [384,392) from smem buffer 0,
// a long chain of UMMAs reads it, then a cp of buffer 1 into the same columns,
// commit; D = sum over the chain of A0 B (B = 1s) must be reps * rowsum(A0).
__global__ void __launch_bounds__(128, 1) k_war(int reps, int32_t* out, int use_fence) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  // buffer 0: A0[m][k] = (m + k) % 5 - 2 ; buffer 1: A1 = 100 ; B = 1 (256 x 32)
  uint8_t* a0 = sm;
  uint8_t* a1 = sm + 4096;
  uint8_t* b = sm + 8192;
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    a0[canon64(m, k) % 4096 + 0] = 0;  // placeholder, rewritten below
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    const int off = (m >> 3) * 256 + (k >> 4) * 128 + (m & 7) * 16 + (k & 15);
    a0[off] = (uint8_t)(int8_t)((m + k) % 5 - 2);
    a1[off] = (uint8_t)100;
  }
  for (int e = threadIdx.x; e < 256 * 32; e += blockDim.x) b[e] = 1;
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  if (threadIdx.x == 0) {
    tmem_cp_128x256b(t + 384, make_sdesc(smem_u32(a0), 128, 256));
    for (int r = 0; r < reps; ++r)
      mma_i8_ta(t, t + 384, make_sdesc(smem_u32(b), 128, 256), idesc_i8(128, 256), r > 0);
    if (use_fence) {
      commit(&mbar);
      mbar_wait(&mbar, 0);
    }
    tmem_cp_128x256b(t + 384, make_sdesc(smem_u32(a1), 128, 256));
    commit(&mbar);
    mbar_wait(&mbar, use_fence ? 1 : 0);
  }
  fence_before();
  __syncthreads();
  fence_after();
  // read D column 0 for each lane: warp w reads lanes 32w..32w+31
  const int w = threadIdx.x >> 5;
  uint32_t v[4];
  tmem_ld4(t + ((uint32_t)(w * 32) << 16), v);
  tmem_wait_ld();
  out[blockIdx.x * 128 + threadIdx.x] = (int32_t)v[0];
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int rpp : {4, 2}) {
    const int tiles = 200;
    k_rate<<<148, 128, 64 * 1024>>>(rpp, tiles, cyc);
    k_rate<<<148, 128, 64 * 1024>>>(rpp, tiles, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> h(148);
    cudaMemcpy(h.data(), cyc, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto x : h) avg += x;
    avg /= 148;
    const double macs = 128.0 * 128 * 64 * 21;   // per tile
    printf("rhs/pass %d: %s  %.0f cycles per 128-node tile  (%.0f MAC/clk/SM)\n", rpp,
           cudaGetErrorString(e), avg / tiles, macs / (avg / tiles));
  }
  int32_t* out;
  cudaMalloc(&out, 148 * 128 * sizeof(int32_t));
  cudaFuncSetAttribute(k_war, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
  for (int fence : {0, 1}) {
    for (int reps : {1, 8, 64}) {
      int bad = 0;
      for (int trial = 0; trial < 20; ++trial) {
        k_war<<<148, 128, 16 * 1024>>>(reps, out, fence);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        std::vector<int32_t> h(148 * 128);
        cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost);
        for (int i = 0; i < 148 * 128; ++i) {
          const int m = i % 128;
          int rs = 0;
          for (int k = 0; k < 32; ++k) rs += (m + k) % 5 - 2;
          if (h[i] != reps * rs) ++bad;
        }
      }
      printf("WAR fence=%d reps=%d: %d wrong lanes of %d\n", fence, reps, bad, 20 * 148 * 128);
    }
  }
  return 0;
}
