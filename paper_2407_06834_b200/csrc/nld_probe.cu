// fp64 FMA throughput probe: the roofline denominator for the spread/gather
// kernels, which are fp64-FMA bound (SURVEY.md §7 hard part 1).
// MEASURED_PEAKS.json carries HBM and bf16 only, so bench.py measures the
// sustained DFMA rate on the same box, in the same run.
#include "nld_internal.cuh"

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
