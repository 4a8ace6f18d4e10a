// Experimental probe: tcgen05 kind::i8 UMMA correctness (descriptor layout)
// and throughput for the tile shapes of the sliced spread / gather.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2407_06834_b200/csrc/nld_umma.cuh"

using namespace nld::umma;

// element (r, k) of an R x K K-major operand at byte offset in the canonical layout
__device__ __forceinline__ int canon_off(int r, int k, int K, int variant) {
  if (variant == 0) return ((r >> 3) * (K >> 4) + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
  // variant 1: K-blocks outermost
  return ((k >> 4) * 16 + (r >> 3)) * 128 + (r & 7) * 16 + (k & 15);
}

template <int NCOLS>
__global__ void k_check(const int8_t* A, const int8_t* B, int M, int N, int K, int32_t* D,
                        int variant, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  uint8_t* sa = sm;
  uint8_t* sb = sm + M * K;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x)
    sa[canon_off(e / K, e % K, K, variant)] = (uint8_t)A[e];
  for (int e = threadIdx.x; e < N * K; e += blockDim.x)
    sb[canon_off(e / K, e % K, K, variant)] = (uint8_t)B[e];
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<NCOLS>(&taddr);
  if (threadIdx.x == 32) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(M, N);
    uint32_t lboA, sboA, lboB, sboB;
    if (variant == 0) { lboA = 128; sboA = (K / 16) * 128; lboB = 128; sboB = (K / 16) * 128; }
    else { lboA = 128 * (M / 8); sboA = 128; lboB = 128 * 16; sboB = 128; }
    if (swap) { uint32_t x = lboA; lboA = sboA; sboA = x; x = lboB; lboB = sboB; sboB = x; }
    for (int kc = 0; kc < K / 32; ++kc) {
      const uint32_t stepA = variant == 0 ? 256 : 2 * 128 * (M / 8);
      const uint32_t stepB = variant == 0 ? 256 : 2 * 128 * 16;
      const uint64_t da = make_sdesc(smem_u32(sa) + kc * stepA, lboA, sboA);
      const uint64_t db = make_sdesc(smem_u32(sb) + kc * stepB, lboB, sboB);
      mma_i8(t, da, db, idesc, kc > 0);
    }
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    if (row < M)
      for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int32_t)r[j];
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<NCOLS>(t);
}

template <int NCOLS>
__global__ void k_rate(int M, int N, int K, int iters, int32_t* sink, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  for (int e = threadIdx.x; e < (M + N) * K; e += blockDim.x) sm[e] = (uint8_t)(e * 7 + 3);
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<NCOLS>(&taddr);
  if (threadIdx.x == 32) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(M, N);
    const uint32_t sboA = (K / 16) * 128;
    for (int it = 0; it < iters; ++it)
      for (int kc = 0; kc < K / 32; ++kc) {
        const uint64_t da = make_sdesc(smem_u32(sm) + kc * 256, 128, sboA);
        const uint64_t db = make_sdesc(smem_u32(sm + M * K) + kc * 256, 128, sboA);
        mma_i8(t + (it % nacc) * N, da, db, idesc, 1);
      }
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after();
  uint32_t r[16];
  const int warp = threadIdx.x >> 5;
  tmem_ld16(t + ((uint32_t)(warp * 32) << 16), r);
  tmem_wait_ld();
  if (r[0] == 0x12345678) sink[0] = r[1];
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<NCOLS>(t);
}

extern "C" int umma_check(const int8_t* A, const int8_t* B, int M, int N, int K, int32_t* D,
                          int variant, int swap) {
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A, M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, N * K, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  const int smem = (M + N) * K;
  cudaFuncSetAttribute(k_check<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_check<256><<<1, 128, smem>>>(dA, dB, M, N, K, dD, variant, swap);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D, dD, M * N * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}

extern "C" int umma_rate(int M, int N, int K, int iters, int blocks, double* tops, int nacc) {
  int32_t* sink;
  cudaMalloc(&sink, 4);
  const int smem = (M + N) * K;
  cudaFuncSetAttribute(k_rate<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<512><<<blocks, 128, smem>>>(M, N, K, 2, sink, nacc);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_rate<512><<<blocks, 128, smem>>>(M, N, K, iters, sink, nacc);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  *tops = 2.0 * M * N * (double)K * iters * blocks / (ms * 1e-3) / 1e12;
  cudaFree(sink);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}

// ---- slicing check (copies of the nld_ozaki.cu helpers) ----
namespace slc {
constexpr double kMagic = 4503599627370496.0 + 141289400074368.0;
__device__ __forceinline__ uint32_t digit_word(uint32_t l0, uint32_t l1, uint32_t l2, uint32_t l3,
                                               uint32_t h0, uint32_t h1, uint32_t h2, uint32_t h3,
                                               int p) {
  const int byte = 5 - p;
  const bool top = byte >= 4;
  const uint32_t s0 = top ? h0 : l0, s1 = top ? h1 : l1, s2 = top ? h2 : l2, s3 = top ? h3 : l3;
  const uint32_t k = byte & 3;
  const uint32_t sel = k | ((k + 4) << 4);
  const uint32_t w01 = __byte_perm(s0, s1, sel);
  const uint32_t w23 = __byte_perm(s2, s3, sel);
  return __byte_perm(w01, w23, 0x5410) ^ 0x80808080u;
}
__global__ void k_slice(const double* x, const double* y, int n, uint32_t* out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 >= n) return;
  uint32_t lo[4], hi[4];
  for (int e = 0; e < 4; ++e) {
    const long long u = __double_as_longlong(fma(x[i + e], y[i + e], kMagic));
    lo[e] = (uint32_t)u;
    hi[e] = (uint32_t)(u >> 32);
  }
  for (int p = 0; p < 6; ++p)
    out[(i / 4) * 6 + p] = digit_word(lo[0], lo[1], lo[2], lo[3], hi[0], hi[1], hi[2], hi[3], p);
}
}  // namespace slc

extern "C" int slice_check(const double* x, const double* y, int n, uint32_t* out) {
  double *dx, *dy;
  uint32_t* dout;
  cudaMalloc(&dx, n * 8); cudaMalloc(&dy, n * 8); cudaMalloc(&dout, n / 4 * 6 * 4);
  cudaMemcpy(dx, x, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y, n * 8, cudaMemcpyHostToDevice);
  slc::k_slice<<<(n / 4 + 127) / 128, 128>>>(dx, dy, n, dout);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(out, dout, n / 4 * 6 * 4, cudaMemcpyDeviceToHost);
  cudaFree(dx); cudaFree(dy); cudaFree(dout);
  return e != cudaSuccess;
}

// ---- A operand from TMEM (written with tcgen05.st) ----
__global__ void k_check_tmemA(const int8_t* A, const int8_t* B, int N, int32_t* D) {
  // M = 128, K = 32: A row m in TMEM lane m, 8 columns of 4 int8 (k = 4 c + byte)
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  const int K = 32;
  for (int e = threadIdx.x; e < N * K; e += blockDim.x)
    sm[((e / K) >> 3) * 256 + ((e % K) >> 4) * 128 + ((e / K) & 7) * 16 + ((e % K) & 15)] =
        (uint8_t)B[e];
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) { mbar_init(&mbar, 1); mbar_fence_init(); }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t t = taddr;
  // D at columns [0, N), A at columns [256, 264)
  {
    const int row = threadIdx.x;   // 128 threads = 4 warps = 128 lanes
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) v |= (uint32_t)(uint8_t)A[row * K + 4 * c + b] << (8 * b);
      w[c] = v;
    }
    const uint32_t ta = t + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + 256;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                 "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(128, N);
    const uint64_t db = make_sdesc(smem_u32(sm), 128, 256);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(t),
        "r"(t + 256), "l"(db), "r"(idesc), "r"(0));
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(t + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c0 + j] = (int32_t)r[j];
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_free<512>(t);
}

extern "C" int umma_check_tmemA(const int8_t* A, const int8_t* B, int N, int32_t* D) {
  int8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, 128 * 32); cudaMalloc(&dB, N * 32); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, A, 128 * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, N * 32, cudaMemcpyHostToDevice);
  k_check_tmemA<<<1, 128, N * 32>>>(dA, dB, N, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
