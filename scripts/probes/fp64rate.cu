// fp64 issue-rate probe: independent DFMA / DMUL chains (8 per thread), runtime
// operands so nothing folds; 148 x 4 blocks of 512 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64rate fp64rate.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 4096;
template <int K>
__global__ void k(const double* in, double m, double* out) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = in[(threadIdx.x + i) & 255];
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) a[i] = fma(a[i], m, 0.25);
      if (K == 1) a[i] = a[i] * m;
      if (K == 2) a[i] = a[i] + m;
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K>
void run(const char* n, double* in, double* out) {
  k<K><<<148 * 4, 512>>>(in, 0.999999, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<K><<<148 * 4, 512>>>(in, 0.999999, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ops = 148.0 * 4 * 512 * IT * 8;
  printf("%s: %.3f ms, %.1f ops/clk/SM at 1.95 GHz, %.1f TFLOP/s-equiv\n", n, ms,
         ops / (ms * 1e-3) / 148 / 1.95e9, ops * (K == 0 ? 2 : 1) / (ms * 1e-3) / 1e12);
}
int main() {
  double *in, *out;
  cudaMalloc(&in, 256 * 8); cudaMemset(in, 0, 256 * 8);
  cudaMalloc(&out, 148 * 4 * 512 * 8);
  run<0>("DFMA", in, out); run<1>("DMUL", in, out); run<2>("DADD", in, out);
  return 0;
}
