// fp64 FMA throughput probe: the roofline denominator for the spread/gather
// kernels, which are fp64-FMA bound (SURVEY.md §7 hard part 1).
// MEASURED_PEAKS.json carries HBM and bf16 only, so bench.py measures the
// sustained DFMA rate on the same box, in the same run.
#include "nld_internal.cuh"
#include "nld_umma.cuh"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dfma(double* out, int64_t iters, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

constexpr int kMmaChains = 8;

// fp64 tensor-core path (DMMA): mma.sync m8n8k4, 256 FMA per warp-instruction
__global__ void __launch_bounds__(256) k_dmma(double* out, int64_t iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[kMmaChains][2];
#pragma unroll
  for (int k = 0; k < kMmaChains; ++k) c[k][0] = c[k][1] = k * 1e-3;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kMmaChains; ++k)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[k][0]), "+d"(c[k][1])
          : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kMmaChains; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// half the warps run DMMA, half run DFMA: tells whether the two fp64 paths
// share execution resources (combined ~= max) or not (combined ~= sum)
__global__ void __launch_bounds__(256) k_mixed(double* out, int64_t iters_mma, int64_t iters_fma) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp & 1) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-7 + c;
    for (int64_t i = 0; i < iters_fma; ++i) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], 0.999999, 1e-9);
    }
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
  } else {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double c[kMmaChains][2];
#pragma unroll
    for (int k = 0; k < kMmaChains; ++k) c[k][0] = c[k][1] = k * 1e-3;
    for (int64_t i = 0; i < iters_mma; ++i) {
#pragma unroll
      for (int k = 0; k < kMmaChains; ++k)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
            : "+d"(c[k][0]), "+d"(c[k][1])
            : "d"(a), "d"(b));
    }
#pragma unroll
    for (int k = 0; k < kMmaChains; ++k) s += c[k][0] + c[k][1];
  }
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" NLD_API int nld_probe_mixed(int64_t iters_mma, int64_t iters_fma, double* tflops,
                                       double* ms, void* stream) {
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* out = nullptr;
    NLD_CUDA(cudaMallocAsync(&out, sizeof(double), st));
    cudaEvent_t e0, e1;
    NLD_CUDA(cudaEventCreate(&e0));
    NLD_CUDA(cudaEventCreate(&e1));
    const int blocks = 148 * 4;
    k_mixed<<<blocks, 256, 0, st>>>(out, iters_mma / 8, iters_fma / 8);
    NLD_CUDA(cudaEventRecord(e0, st));
    k_mixed<<<blocks, 256, 0, st>>>(out, iters_mma, iters_fma);
    NLD_CUDA(cudaEventRecord(e1, st));
    NLD_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    // 4 DMMA warps and 4 DFMA warps per block
    const double fl = 4.0 * blocks * (512.0 * kMmaChains * iters_mma +
                                      32.0 * 2.0 * kChains * iters_fma);
    *ms = t;
    *tflops = fl / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(out, st);
    return NLD_OK;
  } catch (const nld::Error& e) {
    return nld::fail(e.code, e.msg);
  }
}

extern "C" NLD_API int nld_probe_dmma(int64_t iters, int32_t blocks, double* tflops,
                                      double* ms, void* stream) {
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0;
    NLD_CUDA(cudaGetDevice(&dev));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocks <= 0) blocks = sms * 8;
    double* out = nullptr;
    NLD_CUDA(cudaMallocAsync(&out, sizeof(double), st));
    cudaEvent_t e0, e1;
    NLD_CUDA(cudaEventCreate(&e0));
    NLD_CUDA(cudaEventCreate(&e1));
    k_dmma<<<blocks, 256, 0, st>>>(out, iters / 8);
    NLD_CUDA(cudaEventRecord(e0, st));
    k_dmma<<<blocks, 256, 0, st>>>(out, iters);
    NLD_CUDA(cudaEventRecord(e1, st));
    NLD_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    // per warp-instruction: 8x8x4 FMA = 512 flop
    const double flops = 512.0 * kMmaChains * (double)iters * blocks * (256 / 32);
    *ms = t;
    *tflops = flops / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(out, st);
    return NLD_OK;
  } catch (const nld::Error& e) {
    return nld::fail(e.code, e.msg);
  }
}

extern "C" NLD_API int nld_probe_fp64(int64_t iters, int32_t blocks, double* tflops,
                                      double* ms, void* stream) {
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0;
    NLD_CUDA(cudaGetDevice(&dev));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocks <= 0) blocks = sms * 8;
    double* out = nullptr;
    NLD_CUDA(cudaMallocAsync(&out, sizeof(double), st));
    cudaEvent_t e0, e1;
    NLD_CUDA(cudaEventCreate(&e0));
    NLD_CUDA(cudaEventCreate(&e1));
    k_dfma<<<blocks, 256, 0, st>>>(out, iters / 8, 0.999999, 1e-9);  // warm-up
    NLD_CUDA(cudaEventRecord(e0, st));
    k_dfma<<<blocks, 256, 0, st>>>(out, iters, 0.999999, 1e-9);
    NLD_CUDA(cudaEventRecord(e1, st));
    NLD_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    const double flops = 2.0 * kChains * (double)iters * blocks * 256.0;
    *ms = t;
    *tflops = flops / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(out, st);
    return NLD_OK;
  } catch (const nld::Error& e) {
    return nld::fail(e.code, e.msg);
  }
}

// int8 tensor-core (tcgen05 UMMA kind::i8) peak: one CTA per SM issues
// M = 128, N = 256, K = 32 MMAs back to back from shared memory into TMEM --
// the roofline denominator of the integer-sliced spread / gather
__global__ void __launch_bounds__(128, 1) k_imma(int iters, int32_t* sink) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t taddr;
  for (int e = threadIdx.x; e < (128 + 256) * 32; e += blockDim.x) sm[e] = (uint8_t)(e * 7 + 3);
  nld::umma::fence_async_smem();
  if (threadIdx.x < 32) nld::umma::tmem_alloc<512>(&taddr);
  if (threadIdx.x == 32) {
    nld::umma::mbar_init(&mbar, 1);
    nld::umma::mbar_fence_init();
  }
  nld::umma::fence_before();
  __syncthreads();
  nld::umma::fence_after();
  const uint32_t t = taddr;
  if (threadIdx.x == 0) {
    const uint32_t base = nld::umma::smem_u32(sm);
    const uint64_t da = nld::umma::make_sdesc(base, 128, 256);
    const uint64_t db = nld::umma::make_sdesc(base + 128 * 32, 128, 256);
    const uint32_t idesc = nld::umma::idesc_i8(128, 256);
    for (int it = 0; it < iters; ++it) nld::umma::mma_i8(t + (it & 1) * 256, da, db, idesc, 1);
    nld::umma::commit(&mbar);
  }
  nld::umma::mbar_wait(&mbar, 0);
  nld::umma::fence_after();
  uint32_t r[16];
  nld::umma::tmem_ld16(t + ((uint32_t)((threadIdx.x >> 5) * 32) << 16), r);
  nld::umma::tmem_wait_ld();
  if (r[0] == 0x12345678u) sink[0] = (int32_t)r[1];
  nld::umma::fence_before();
  __syncthreads();
  if (threadIdx.x < 32) nld::umma::tmem_free<512>(t);
}

extern "C" NLD_API int nld_probe_imma(int64_t iters, int32_t blocks, double* tops, double* ms,
                                      void* stream) {
  try {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int dev = 0;
    NLD_CUDA(cudaGetDevice(&dev));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocks <= 0) blocks = sms;
    int32_t* sink = nullptr;
    NLD_CUDA(cudaMallocAsync(&sink, sizeof(int32_t), st));
    const int smem = (128 + 256) * 32;
    cudaEvent_t e0, e1;
    NLD_CUDA(cudaEventCreate(&e0));
    NLD_CUDA(cudaEventCreate(&e1));
    k_imma<<<blocks, 128, smem, st>>>((int)(iters / 8), sink);
    NLD_CUDA(cudaEventRecord(e0, st));
    k_imma<<<blocks, 128, smem, st>>>((int)iters, sink);
    NLD_CUDA(cudaEventRecord(e1, st));
    NLD_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t;
    *tops = 2.0 * 128 * 256 * 32 * (double)iters * blocks / (t * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(sink, st);
    return NLD_OK;
  } catch (const nld::Error& e) {
    return nld::fail(e.code, e.msg);
  }
}
