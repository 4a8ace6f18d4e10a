// Issue-rate probe for the epilogue's conversion options on this GPU:
// DADD, DFMA, I2F.F64.S32, I2F.F64.S64, the magic-number int32->fp64 and IMAD.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int K>
__global__ void k_probe(const int* in, double* out) {
  int x[8];
  double acc[8];
  for (int i = 0; i < 8; ++i) { x[i] = in[threadIdx.x + i]; acc[i] = 0.0; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (K == 0) acc[i] = acc[i] + 1.000000001;                         // DADD
      if (K == 1) acc[i] = fma(acc[i], 1.0000001, 0.5);                   // DFMA
      if (K == 2) { acc[i] += (double)x[i]; x[i] += 3; }                  // I2F.F64.S32 + DADD + IADD
      if (K == 3) { acc[i] += (double)(long long)x[i]; x[i] += 3; }       // I2F.F64.S64
      if (K == 4) { acc[i] += __hiloint2double(0x43300000, x[i] ^ 0x80000000) - 4503601774854144.0; x[i] += 3; }
      if (K == 5) { x[i] = x[i] * 257 + 3; }                               // IMAD
      if (K == 6) { acc[i] += (double)(float)x[i]; x[i] += 3; }           // I2F.F32 + F2F.F64
      if (K == 7) acc[i] = acc[i] * 1.0000001;                            // DMUL
      if (K == 8) { x[i] = __byte_perm(x[i], x[i + 1 & 7], 0x5140) ^ 0x80808080; }  // PRMT+LOP
    }
  }
  double s = 0.0;
  for (int i = 0; i < 8; ++i) s += acc[i] + x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(const char* name, int ops_per_iter) {
  int* in; double* out;
  cudaMalloc(&in, 4096 * sizeof(int));
  cudaMemset(in, 0, 4096 * sizeof(int));
  const int blocks = 148 * 4, threads = 512;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  k_probe<K><<<blocks, threads>>>(in, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_probe<K><<<blocks, threads>>>(in, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double thr_ops = (double)blocks * threads * ITERS * 8 * ops_per_iter;
  const double per_clk_sm = thr_ops / (ms * 1e-3) / 148 / (clk * 1e3);
  printf("%-28s %8.3f ms  %7.1f thread-ops/clk/SM (at %d MHz nominal)\n", name, ms, per_clk_sm, clk / 1000);
  cudaFree(in); cudaFree(out);
}

int main() {
  run<0>("DADD", 1);
  run<1>("DFMA", 1);
  run<2>("I2F.F64.S32 (+DADD)", 1);
  run<3>("I2F.F64.S64 (+DADD)", 1);
  run<4>("magic i2d (LOP,MOV,DADD x2)", 1);
  run<5>("IMAD", 1);
  run<6>("I2F.F32+F2F.F64 (+DADD)", 1);
  run<7>("DMUL", 1);
  run<8>("PRMT+LOP", 2);
  return 0;
}
