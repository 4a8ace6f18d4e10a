// Experimental probe: cost of the sliced gather's UMMA issue pattern per
// 32-node tile (12 kind::i8 UMMAs, M = 128, K = 32, N = (6 - p) * 32 with the
// D window shifted by 32 p) against variants, one CTA per SM, issuer only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared
//        -Xcompiler -fPIC -o probe_pattern.so probe_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2407_06834_b200/csrc/nld_umma.cuh"

using namespace nld::umma;

constexpr int kGA = 128 * 64;     // one G digit slice (128 rows x K 64)
constexpr int kGB = 32 * 64;      // one Y digit slice (32 nodes x K 64)

__global__ void __launch_bounds__(128, 1) k_pat(int variant, int tiles, int32_t* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  const int bytes = 6 * kGA + 6 * 8 * kGB;
  for (int e = threadIdx.x; e < bytes; e += blockDim.x) sm[e] = (uint8_t)(e * 7 + 3);
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) {
    mbar_init(&mbar, 1);
    mbar_fence_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  if (threadIdx.x == 0) {
    const uint32_t aB = smem_u32(sm);
    for (int g = 0; g < tiles; ++g) {
      const uint32_t bB = smem_u32(sm + 6 * kGA + (g & 7) * 6 * kGB);
      const uint32_t dcol = t + (uint32_t)((g & 1) * 192);
      if (variant == 0 || variant == 3) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            const uint64_t db = make_sdesc(bB + ks * 256, 128, 512);
            if (variant == 0) {
              const uint64_t da = make_sdesc(aB + p * kGA + ks * 256, 128, 512);
              mma_i8(dcol + p * 32, da, db, idesc_i8(128, (6 - p) * 32), (ks > 0 || p > 0));
            } else {
              mma_i8_ta(dcol + p * 32, t + 384 + p * 16 + ks * 8, db, idesc_i8(128, (6 - p) * 32),
                        (ks > 0 || p > 0));
            }
          }
      } else if (variant == 1) {   // 12 x N = 32, disjoint D per p
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            const uint64_t da = make_sdesc(aB + p * kGA + ks * 256, 128, 512);
            const uint64_t db = make_sdesc(bB + ks * 256, 128, 512);
            mma_i8(dcol + p * 32, da, db, idesc_i8(128, 32), ks > 0);
          }
      } else if (variant == 2) {   // 12 x N = 192, same D
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            const uint64_t da = make_sdesc(aB + p * kGA + ks * 256, 128, 512);
            const uint64_t db = make_sdesc(bB + ks * 256, 128, 512);
            mma_i8(dcol, da, db, idesc_i8(128, 192), (ks > 0 || p > 0));
          }
      } else if (variant == 4) {   // 12 x N = 256, same D (floor reference)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            const uint64_t da = make_sdesc(aB + p * kGA + ks * 256, 128, 512);
            const uint64_t db = make_sdesc(bB + ks * 256, 128, 512);
            mma_i8(t + (uint32_t)((g & 1) * 256), da, db, idesc_i8(128, 256), (ks > 0 || p > 0));
          }
      } else if (variant == 5) {   // 4 x N = 256 (same MACs as 8 x N = 128)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t da = make_sdesc(aB + q * kGA, 128, 512);
          const uint64_t db = make_sdesc(bB, 128, 512);
          mma_i8(t + (uint32_t)((g & 1) * 256), da, db, idesc_i8(128, 256), q > 0);
        }
      } else if (variant == 7 || variant == 8) {
        // spread pattern per 32-node chunk: A = X digit p (128 x 32), B = the
        // stacked Y slices [e_q0 .. e_q0+nq-1] (64 rows each), D shifted by 64 (p + q0);
        // variant 8 issues each UMMA for two chunks back to back (same D window)
        const int reps = variant == 8 ? 2 : 1;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
          for (int q0 = 0; q0 < 6 - p; q0 += 4) {
            const int nq = (6 - p - q0) < 4 ? (6 - p - q0) : 4;
            for (int rr = 0; rr < reps; ++rr) {
              const uint64_t da = make_sdesc(aB + p * 4096 + rr * 24576, 128, 256);
              const uint64_t db = make_sdesc(smem_u32(sm + 6 * kGA) + q0 * 2048 + rr * 12288, 128, 256);
              mma_i8(t + (uint32_t)((p + q0) * 64), da, db, idesc_i8(128, nq * 64), 1u);
            }
          }
      } else if (variant == 6) {   // gather pattern, K = 64 per instruction impossible for i8:
        // same as 0 but ks-outer order swapped (p outer): consecutive UMMAs on the same D window
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint64_t da = make_sdesc(aB + p * kGA + ks * 256, 128, 512);
            const uint64_t db = make_sdesc(bB + ks * 256, 128, 512);
            mma_i8(dcol + p * 32, da, db, idesc_i8(128, (6 - p) * 32), (ks > 0 || p > 0));
          }
      }
    }
    commit(&mbar);
  }
  __syncwarp();
  // wait for everything: poll the final phase count via a blocking loop on all commits
  mbar_wait(&mbar, 0);
  __syncthreads();
  fence_after();
  uint32_t r[16];
  tmem_ld16(t + ((uint32_t)((threadIdx.x >> 5) * 32) << 16), r);
  tmem_wait_ld();
  if (r[0] == 0x12345678u) sink[0] = (int32_t)r[1];
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

extern "C" int pattern_rate(int variant, int tiles, int blocks, double* cyc_per_tile) {
  int32_t* sink;
  cudaMalloc(&sink, 4);
  const int smem = 6 * kGA + 6 * 8 * kGB;
  cudaFuncSetAttribute(k_pat, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pat<<<blocks, 128, smem>>>(variant, 64, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_pat<<<blocks, 128, smem>>>(variant, tiles, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  *cyc_per_tile = ms * 1e-3 * clk * 1e3 / tiles;
  cudaFree(sink);
  if (e != cudaSuccess) {
    printf("err %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

// TMEM read throughput: every warp loads 32 lanes x 8 columns (1 KB) per
// tcgen05.ld 32x32b.x8 from its lane quarter, `iters` times (x6 per wait)
__global__ void k_tld(int iters, int32_t* sink) {
  __shared__ uint32_t taddr;
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr + ((uint32_t)(((threadIdx.x >> 5) & 3) * 32) << 16);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[6][8];
#pragma unroll
    for (int q = 0; q < 6; ++q) tmem_ld8(t + (uint32_t)(((it * 6 + q) * 8) & 511), r[q]);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += r[q][i];
  }
  if (acc == 0x12345678u) sink[0] = (int32_t)acc;
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(taddr);
}

extern "C" int tld_rate(int warps, int iters, int blocks, double* bytes_per_cyc) {
  int32_t* sink;
  cudaMalloc(&sink, 4);
  k_tld<<<blocks, 32 * warps>>>(16, sink);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_tld<<<blocks, 32 * warps>>>(iters, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  *bytes_per_cyc = (double)warps * iters * 6 * 1024 / cyc;   // per SM (one CTA per SM)
  cudaFree(sink);
  return e != cudaSuccess;
}

// commit round trip: lane 0 of warp 0 issues (optionally one UMMA and) a
// tcgen05.commit to bar_a; warp 1 waits on bar_a and arrives on bar_b;
// warp 0 waits on bar_b -- cycles per iteration
__global__ void __launch_bounds__(64, 1) k_commit_rt(int iters, int with_mma, long long* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t bar_a, bar_b;
  __shared__ uint32_t taddr;
  for (int e = threadIdx.x; e < 128 * 32 + 32 * 32; e += blockDim.x) sm[e] = (uint8_t)e;
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) {
    mbar_init(&bar_a, 1);
    mbar_init(&bar_b, 1);
    mbar_fence_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  const long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int it = 0; it < iters; ++it) {
      if (threadIdx.x == 0) {
        if (with_mma) {
          const uint64_t da = make_sdesc(smem_u32(sm), 128, 256);
          const uint64_t db = make_sdesc(smem_u32(sm + 4096), 128, 256);
          mma_i8(t, da, db, idesc_i8(128, 32), 1u);
        }
        commit(&bar_a);
      }
      __syncwarp();
      mbar_wait(&bar_b, it & 1);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&bar_a, it & 1);
      if (threadIdx.x == 32) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar_b)) : "memory");
      __syncwarp();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

extern "C" int commit_rt(int iters, int with_mma, int blocks, double* cyc) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  k_commit_rt<<<blocks, 64, 8192>>>(iters, with_mma, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * (blocks < 256 ? blocks : 256), cudaMemcpyDeviceToHost);
  *cyc = (double)h[0] / iters;
  cudaFree(d);
  return e != cudaSuccess;
}
