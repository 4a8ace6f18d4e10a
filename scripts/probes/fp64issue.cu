// fp64 issue behaviour with FEW warps per SM sub-partition (the sliced
// gather's epilogue has two): cycles per DFMA for W warps per sub-partition
// with C independent chains per thread, a dependent chain (latency), and the
// epilogue's combine mix (3 IMAD, 2 LEA-like, I2F, DADD, 2 DFMA per value).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64issue fp64issue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int IT = 2048;
template <int C>
__global__ void k_dfma(const double* in, double m, double* out, long long* cyc) {
  double a[C];
  for (int i = 0; i < C; ++i) a[i] = in[(threadIdx.x + i) & 255];
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) a[i] = fma(a[i], m, 0.25);
  }
  const long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < C; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_combine(const int* in, const double* av, double* out, long long* cyc) {
  int d[6][4];
  for (int t = 0; t < 6; ++t)
    for (int i = 0; i < 4; ++i) d[t][i] = in[(threadIdx.x + 4 * t + i) & 255];
  double a0 = av[threadIdx.x & 7], a1 = av[(threadIdx.x + 1) & 7], sh = 0, sl = 0, sh1 = 0, sl1 = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t x01 = (uint32_t)d[0][i] * 256u + (uint32_t)d[1][i];
      const int32_t x23 = (int32_t)((uint32_t)d[2][i] * 256u + (uint32_t)d[3][i]);
      const uint32_t x45b = (uint32_t)d[4][i] * 256u + ((uint32_t)d[5][i] ^ 0x80000000u);
      double r;
      asm("{\n\t.reg .b64 c;\n\tmov.b64 c, {%1, %2};\n\tmad.wide.s32 c, %3, 65536, c;\n\t"
          "mov.b64 %0, c;\n\t}" : "=d"(r) : "r"(x45b), "r"(0x43380000u), "r"(x23));
      const double lo = r - (6755399441055744.0 + 2147483648.0);
      const double hi = (double)(int32_t)x01;
      if (i & 1) { sh1 = fma(hi, a1, sh1); sl1 = fma(lo, a1, sl1); }
      else { sh = fma(hi, a0, sh); sl = fma(lo, a0, sl); }
      d[0][i] += it; d[3][i] ^= it;   // new inputs each round
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sh + sl + sh1 + sl1;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double *in, *out; long long* cyc; int* ii;
  cudaMalloc(&in, 256 * 8); cudaMemset(in, 0, 256 * 8);
  cudaMalloc(&ii, 256 * 4); cudaMemset(ii, 1, 256 * 4);
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  for (int w : {1, 2, 4, 8}) {
    k_dfma<1><<<148, 128 * w>>>(in, 0.999, out, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c1 = (double)h[0] / IT;
    k_dfma<4><<<148, 128 * w>>>(in, 0.999, out, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c4 = (double)h[0] / IT / 4;
    k_dfma<8><<<148, 128 * w>>>(in, 0.999, out, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c8 = (double)h[0] / IT / 8;
    k_combine<<<148, 128 * w>>>(ii, in, out, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double cc = (double)h[0] / IT / 4;
    printf("%d warps/SMSP: dependent DFMA %.1f cyc, 4 chains %.2f cyc/DFMA/warp, 8 chains %.2f; combine %.1f cyc per value per warp (%.1f per SMSP-value)\n",
           w, c1, c4, c8, cc, cc / w);
  }
  return 0;
}
