// Cost of the gather epilogue's diagonal combine (6 int32 -> fp64, times a
// weight, accumulated) for W warps per SM sub-partition, per variant:
//  0 hi/lo: I2F.F64.S32(x01) + IMAD.WIDE-on-magic(lo) + DADD + 2 DFMA
//  1 int64: one I2F.F64.S64 + 1 DFMA
//  2 magic: H = x01 2^16 + x23 and L = x45 by magic patterns, 2 DADD + 2 DFMA
//  3 mixed: values alternate between 1 and 2
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o combine_probe combine_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int IT = 2048;
__device__ __forceinline__ void v0(const int (&d)[6], double a, double& s0, double& s1) {
  const uint32_t x01 = (uint32_t)d[0] * 256u + (uint32_t)d[1];
  const int32_t x23 = (int32_t)((uint32_t)d[2] * 256u + (uint32_t)d[3]);
  const uint32_t x45b = (uint32_t)d[4] * 256u + ((uint32_t)d[5] ^ 0x80000000u);
  double r;
  asm("{\n\t.reg .b64 c;\n\tmov.b64 c, {%1, %2};\n\tmad.wide.s32 c, %3, 65536, c;\n\tmov.b64 %0, c;\n\t}"
      : "=d"(r) : "r"(x45b), "r"(0x43380000u), "r"(x23));
  s0 = fma((double)(int32_t)x01, a, s0);
  s1 = fma(r - (6755399441055744.0 + 2147483648.0), a, s1);
}
__device__ __forceinline__ void v1(const int (&d)[6], double a, double& s0, double&) {
  const int32_t x01 = d[0] * 256 + d[1], x23 = d[2] * 256 + d[3], x45 = d[4] * 256 + d[5];
  const long long lo = (long long)x23 * 65536 + (long long)x45;
  long long t;
  asm("{\n\t.reg .b32 l, h;\n\tmov.b64 {l, h}, %1;\n\tadd.s32 h, h, %2;\n\tmov.b64 %0, {l, h};\n\t}"
      : "=l"(t) : "l"(lo), "r"(x01));
  s0 = fma((double)t, a, s0);
}
__device__ __forceinline__ void v2(const int (&d)[6], double a, double& s0, double& s1) {
  const int32_t x01 = d[0] * 256 + d[1];
  const uint32_t x23b = (uint32_t)(d[2] * 256 + d[3]) ^ 0x80000000u;
  const uint32_t x45b = (uint32_t)(d[4] * 256 + d[5]) ^ 0x80000000u;
  double h;
  asm("{\n\t.reg .b64 c;\n\tmov.b64 c, {%1, %2};\n\tmad.wide.s32 c, %3, 65536, c;\n\tmov.b64 %0, c;\n\t}"
      : "=d"(h) : "r"(x23b), "r"(0x43380000u), "r"(x01));
  const double l = __hiloint2double(0x43300000, (int)x45b) - 4503601774854144.0;
  s0 = fma(h - (6755399441055744.0 + 2147483648.0), a, s0);
  s1 = fma(l, a, s1);
}
template <int V>
__global__ void k(const int* in, const double* av, double* out, long long* cyc) {
  int d[4][6];
  for (int i = 0; i < 4; ++i)
    for (int t = 0; t < 6; ++t) d[i][t] = in[(threadIdx.x + 4 * t + i) & 255];
  double a0 = av[threadIdx.x & 7], a1 = av[(threadIdx.x + 1) & 7];
  double s[4][2] = {};
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double a = (i & 1) ? a1 : a0;
      if (V == 0) v0(d[i], a, s[i][0], s[i][1]);
      if (V == 1) v1(d[i], a, s[i][0], s[i][1]);
      if (V == 2) v2(d[i], a, s[i][0], s[i][1]);
      if (V == 3) { if (i & 1) v2(d[i], a, s[i][0], s[i][1]); else v1(d[i], a, s[i][0], s[i][1]); }
      if (V == 4) { if (i == 3) v2(d[i], a, s[i][0], s[i][1]); else v1(d[i], a, s[i][0], s[i][1]); }
      d[i][0] += it; d[i][3] ^= it; d[i][5] += 7;
    }
  }
  const long long t1 = clock64();
  double r = 0;
  for (int i = 0; i < 4; ++i) r += s[i][0] + s[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int V>
double run(int w, int* ii, double* in, double* out, long long* cyc) {
  long long h[148];
  k<V><<<148, 128 * w>>>(ii, in, out, cyc);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  return (double)h[0] / IT / 4;
}
int main() {
  double *in, *out; long long* cyc; int* ii;
  cudaMalloc(&in, 256 * 8); cudaMemset(in, 0, 256 * 8);
  cudaMalloc(&ii, 256 * 4); cudaMemset(ii, 1, 256 * 4);
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&cyc, 148 * 8);
  for (int w : {1, 2, 3, 4}) {
    printf("%d warps/SMSP, cycles per value per warp: hi/lo %.1f  int64 %.1f  magic %.1f  mixed 1:1 %.1f  mixed 3:1 %.1f\n", w,
           run<0>(w, ii, in, out, cyc), run<1>(w, ii, in, out, cyc), run<2>(w, ii, in, out, cyc),
           run<3>(w, ii, in, out, cyc), run<4>(w, ii, in, out, cyc));
  }
  return 0;
}
