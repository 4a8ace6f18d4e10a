// Feature / window preparation on the device:
// patch features (features.py:20-36) and the plug-in mutual information of
// every patch offset with the centre (features.py:44-78), which ranks the
// offsets into ANOVA windows.  Histograms are integer counts (exact,
// order-independent); the digitisation replays numpy's operation order.
#include <algorithm>
#include <cmath>
#include <vector>

#include "nld_internal.cuh"

namespace nld {
namespace {

constexpr int kBins = 16;          // MI_BINS (features.py:16)

int nb(int64_t n, int threads = 256, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

__device__ __forceinline__ int64_t reflect_idx(int64_t i, int64_t n) {
  if (n == 1) return 0;
  while (i < 0 || i >= n) i = i < 0 ? -i : 2 * (n - 1) - i;
  return i;
}

// out[(y*w + x) * F + ch*p*p + dr*p + dc] = a * img[ch][y+dr-r][x+dc-r] + b
__global__ void k_patches(const double* __restrict__ img, int64_t h, int64_t w, int C, int p,
                          int mode, double a, double b, double* __restrict__ out) {
  const int r = p / 2;
  const int F = C * p * p;
  const int64_t total = h * w * F;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(e % F);
    const int64_t px = e / F;
    const int64_t y = px / w, x = px % w;
    const int ch = f / (p * p);
    const int dr = (f / p) % p, dc = f % p;
    int64_t yy = y + dr - r, xx = x + dc - r;
    double v;
    if (mode == 0) {
      v = (yy < 0 || yy >= h || xx < 0 || xx >= w) ? 0.0 : img[(ch * h + yy) * w + xx];
    } else {
      yy = reflect_idx(yy, h);
      xx = reflect_idx(xx, w);
      v = img[(ch * h + yy) * w + xx];
    }
    out[e] = a * (v - b);
  }
}

__global__ void k_colminmax(const double* __restrict__ f, int64_t n, int d,
                            double* __restrict__ lo, double* __restrict__ hi) {
  // one block per column, fixed-order-free (min/max are exact)
  const int j = blockIdx.x;
  __shared__ double smin[256], smax[256];
  double mn = INFINITY, mx = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = f[i * d + j];
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + off]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + off]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    lo[j] = smin[0];
    hi[j] = smax[0];
  }
}

// digitize (features.py:59-64): equal-width bins over the column's range
__device__ __forceinline__ int bin_of(double v, double lo, double hi) {
  if (hi <= lo) return 0;
  const double w = (double)kBins / __dsub_rn(hi, lo);
  const long long idx = (long long)__dmul_rn(__dsub_rn(v, lo), w);
  return (int)min(idx, (long long)(kBins - 1));
}

// joint counts[j][bj][bc] of every column j with the centre column
__global__ void k_joint_hist(const double* __restrict__ f, int64_t n, int d, int center,
                             const double* __restrict__ lo, const double* __restrict__ hi,
                             unsigned int* __restrict__ counts) {
  extern __shared__ unsigned int sh[];   // [d][256]
  for (int e = threadIdx.x; e < d * kBins * kBins; e += blockDim.x) sh[e] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int bc = bin_of(f[i * d + center], lo[center], hi[center]);
    for (int j = 0; j < d; ++j) {
      const int bj = bin_of(f[i * d + j], lo[j], hi[j]);
      atomicAdd(&sh[(j * kBins + bj) * kBins + bc], 1u);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d * kBins * kBins; e += blockDim.x)
    if (sh[e]) atomicAdd(&counts[e], sh[e]);
}

// MI (nats) from the counts (features.py:70-77), one thread per column
__global__ void k_mi(const unsigned int* __restrict__ counts, int64_t n, int d,
                     double* __restrict__ scores) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const unsigned int* c = counts + (int64_t)j * kBins * kBins;
  double pj[kBins], pc[kBins];
  for (int a = 0; a < kBins; ++a) pj[a] = pc[a] = 0.0;
  for (int a = 0; a < kBins; ++a)
    for (int b = 0; b < kBins; ++b) {
      const double p = (double)c[a * kBins + b] / (double)n;
      pj[a] += p;
      pc[b] += p;
    }
  double mi = 0.0;
  for (int a = 0; a < kBins; ++a)
    for (int b = 0; b < kBins; ++b) {
      const unsigned int cnt = c[a * kBins + b];
      if (!cnt) continue;
      const double p = (double)cnt / (double)n;
      mi += p * log(p / (pj[a] * pc[b]));
    }
  scores[j] = mi;
}

}  // namespace
}  // namespace nld

using nld::Error;

extern "C" {

int nld_extract_patches(const double* image, int64_t h, int64_t w, int32_t channels,
                        int32_t patch, int32_t mode, double a, double b, double* out,
                        void* stream) {
  try {
    if (h <= 0 || w <= 0 || channels <= 0) throw Error(NLD_ERR_VALUE, "expected a 2-d image");
    if (patch < 1 || patch % 2 == 0) throw Error(NLD_ERR_VALUE, "patch size must be odd and positive");
    if (mode != 0 && mode != 1) throw Error(NLD_ERR_VALUE, "mode must be 0 (zero) or 1 (reflect)");
    if (mode == 1 && (patch / 2 >= h || patch / 2 >= w))
      throw Error(NLD_ERR_VALUE, "reflect padding wider than the image");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t total = h * w * channels * patch * patch;
    nld::k_patches<<<nld::nb(total), 256, 0, st>>>(image, h, w, channels, patch, mode, a, b, out);
    NLD_CUDA(cudaGetLastError());
    return NLD_OK;
  } catch (const Error& e) {
    return nld::fail(e.code, e.msg);
  }
}

int nld_mi_scores(const double* features, int64_t n, int32_t d, int32_t center,
                  double* scores_host, void* stream) {
  try {
    if (n <= 0 || d <= 0) throw Error(NLD_ERR_VALUE, "empty feature matrix");
    if (center < 0 || center >= d) throw Error(NLD_ERR_VALUE, "center column out of range");
    if ((int64_t)d * nld::kBins * nld::kBins * 4 > 200 * 1024)
      throw Error(NLD_ERR_VALUE, "too many feature columns for the shared histogram");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double *lo = nullptr, *hi = nullptr, *sc = nullptr;
    unsigned int* counts = nullptr;
    NLD_CUDA(cudaMallocAsync(&lo, sizeof(double) * d, st));
    NLD_CUDA(cudaMallocAsync(&hi, sizeof(double) * d, st));
    NLD_CUDA(cudaMallocAsync(&sc, sizeof(double) * d, st));
    NLD_CUDA(cudaMallocAsync(&counts, sizeof(unsigned int) * d * 256, st));
    NLD_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned int) * d * 256, st));
    nld::k_colminmax<<<d, 256, 0, st>>>(features, n, d, lo, hi);
    const size_t smem = sizeof(unsigned int) * d * 256;
    if (smem > 48 * 1024)
      NLD_CUDA(cudaFuncSetAttribute(nld::k_joint_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    nld::k_joint_hist<<<nld::nb(n, 256, 148 * 2), 256, smem, st>>>(features, n, d, center, lo,
                                                                    hi, counts);
    nld::k_mi<<<(d + 63) / 64, 64, 0, st>>>(counts, n, d, sc);
    NLD_CUDA(cudaGetLastError());
    NLD_CUDA(cudaMemcpyAsync(scores_host, sc, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(lo, st);
    cudaFreeAsync(hi, st);
    cudaFreeAsync(sc, st);
    cudaFreeAsync(counts, st);
    return NLD_OK;
  } catch (const Error& e) {
    return nld::fail(e.code, e.msg);
  }
}

}  // extern "C"
