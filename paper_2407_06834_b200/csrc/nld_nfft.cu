// The general transform API: NFFT, adjoint NFFT, exact
// NDFT / adjoint and direct Gauss sums, plus the FastsumPlan geometry and
// Gaussian coefficients -- transform.py:74-333.
//
// An NFFT plan is an nld_operator in raw-torus mode (one window of d
// dimensions, nodes used as given after an optional affine map).  It reuses
// the operator's node tables and its spread / gather stages with the complex
// values as two right-hand sides: the pixel-major [N][2] layout of the stages
// is exactly interleaved complex.  Between the support box of the grid and
// the M^d centred frequencies sit d pruned separable DFT passes (unnormalised,
// e^{+} for the adjoint as ifftn(.)*prod(nos), e^{-} for the forward as fftn).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "nld_internal.cuh"

namespace nld {
namespace {

int nblocks(int64_t n, int threads = 256, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

// one DFT pass along an axis of a complex array viewed as (A, nin, B)
// dir 0: positions -> frequencies, out[f] = sum_p in[p] e^{+2 pi i k(f) l(p) / n}
// dir 1: frequencies -> positions, out[p] = sum_f in[f] e^{-2 pi i k(f) l(p) / n}
__global__ void k_dft_pass(const double2* __restrict__ in, double2* __restrict__ out, int64_t A,
                           int nin, int nout, int64_t B, int n, int M, int lo, int wrap,
                           int dir) {
  const int64_t total = A * nout * B;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e % B;
    const int o = (int)((e / B) % nout);
    const int64_t a = e / ((int64_t)nout * B);
    double re = 0.0, im = 0.0;
    for (int i = 0; i < nin; ++i) {
      const int k = (dir == 0 ? o : i) - M / 2;
      const int p = dir == 0 ? i : o;
      const long long l = wrap ? p : (long long)lo + p;
      long long ph = ((long long)k * l) % n;
      if (ph < 0) ph += n;
      double sn, cs;
      sincospi(2.0 * (double)ph / (double)n, &sn, &cs);
      if (dir == 1) sn = -sn;
      const double2 x = in[(a * nin + i) * B + b];
      re += x.x * cs - x.y * sn;
      im += x.x * sn + x.y * cs;
    }
    out[e] = make_double2(re, im);
  }
}

__global__ void k_planes_to_complex(const double* __restrict__ planes, int64_t ld, int64_t n,
                                    double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_double2(planes[i], planes[ld + i]);
}

__global__ void k_complex_to_planes(const double2* __restrict__ in, int64_t n, int64_t ld,
                                    double* __restrict__ planes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    planes[i] = in[i].x;
    planes[ld + i] = in[i].y;
  }
}

// I0 window factors c(k), k = -M/2 .. M/2-1 (transform.py:140-145)
__global__ void k_window_factors(double* __restrict__ c, int M, int n, int m, double b) {
  for (int kk = threadIdx.x; kk < M; kk += blockDim.x) {
    const int k = kk - M / 2;
    const double w = (2.0 * 3.141592653589793 * (double)k) / (double)n;
    c[kk] = cyl_bessel_i0((double)m * sqrt(b * b - w * w));
  }
}

// divide by prod_s c(k_s) in dimension order (transform.py:191-197), optional
// real multiplier afterwards (gauss_transform_fast's kernel_coeffs, :332)
__global__ void k_deconvolve(const double2* __restrict__ in, double2* __restrict__ out,
                             const double* __restrict__ c, int M, int d,
                             const double* __restrict__ mult) {
  int64_t total = 1;
  for (int s = 0; s < d; ++s) total *= M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 x = in[e];
    int64_t rem = e;
    int ks[3] = {0, 0, 0};
    for (int s = d - 1; s >= 0; --s) {
      ks[s] = (int)(rem % M);
      rem /= M;
    }
    for (int s = 0; s < d; ++s) {
      x.x /= c[ks[s]];
      x.y /= c[ks[s]];
    }
    if (mult) {
      x.x *= mult[e];
      x.y *= mult[e];
    }
    out[e] = x;
  }
}

// exact trigonometric sums (transform.py:74-102)
__global__ void k_ndft(const double* __restrict__ x, int64_t n, int d, int M,
                       const double2* __restrict__ c, double2* __restrict__ out) {
  int64_t total = 1;
  for (int s = 0; s < d; ++s) total *= M;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int64_t e = 0; e < total; ++e) {
      int64_t rem = e;
      double ph = 0.0;
      for (int s = d - 1; s >= 0; --s) {
        const int k = (int)(rem % M) - M / 2;
        rem /= M;
        ph += (double)k * x[j * d + s];
      }
      double sn, cs;
      sincospi(-2.0 * ph, &sn, &cs);
      re += c[e].x * cs - c[e].y * sn;
      im += c[e].x * sn + c[e].y * cs;
    }
    out[j] = make_double2(re, im);
  }
}

__global__ void k_ndft_adjoint(const double* __restrict__ x, int64_t n, int d, int M,
                               const double2* __restrict__ v, double2* __restrict__ out) {
  int64_t total = 1;
  for (int s = 0; s < d; ++s) total *= M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int kk[3] = {0, 0, 0};
    int64_t rem = e;
    for (int s = d - 1; s >= 0; --s) {
      kk[s] = (int)(rem % M) - M / 2;
      rem /= M;
    }
    double re = 0.0, im = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      double ph = 0.0;
      for (int s = 0; s < d; ++s) ph += (double)kk[s] * x[j * d + s];
      double sn, cs;
      sincospi(2.0 * ph, &sn, &cs);
      re += v[j].x * cs - v[j].y * sn;
      im += v[j].x * sn + v[j].y * cs;
    }
    out[e] = make_double2(re, im);
  }
}

// exact O(Nx Ny) discrete Gauss transform (transform.py:231-244)
__global__ void k_gauss_direct(const double* __restrict__ tgt, int64_t nt,
                               const double* __restrict__ src, int64_t ns, int d,
                               const double* __restrict__ alpha, double sigbar,
                               double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t j = 0; j < ns; ++j) {
      double r2 = 0.0;
      for (int s = 0; s < d; ++s) {
        const double diff = tgt[i * d + s] - src[j * d + s];
        r2 += diff * diff;
      }
      acc += alpha[j] * exp(-sigbar * r2);
    }
    out[i] = acc;
  }
}

// kernel_coeffs of FastsumPlan.build (transform.py:302-307): the d-variate
// ifft of the sampled Gaussian, separable: prod_s c1[k_s]
__global__ void k_gauss_coeffs(int M, int d, double sig, double* __restrict__ out) {
  extern __shared__ double c1[];
  for (int kk = threadIdx.x; kk < M; kk += blockDim.x) {
    const int k = kk - M / 2;
    double acc = 0.0;
    for (int jj = 0; jj < M; ++jj) {
      const int j = jj - M / 2;
      const double jm = (double)j / (double)M;
      const int ph = ((k * j) % M + M) % M;
      acc += exp(-(sig * (jm * jm))) * cospi(2.0 * (double)ph / (double)M);
    }
    c1[kk] = acc / (double)M;
  }
  __syncthreads();
  int64_t total = 1;
  for (int s = 0; s < d; ++s) total *= M;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    int64_t rem = e;
    double v = 1.0;
    for (int s = d - 1; s >= 0; --s) {
      v *= c1[rem % M];
      rem /= M;
    }
    out[e] = v;
  }
}

struct Passes {
  int64_t dims[3];
  int d;
};

// run the d separable passes; returns the buffer holding the result
double2* dft_passes(const WinDev& wd, int M, double2* a, double2* b, int dir,
                    cudaStream_t st) {
  const int d = wd.d;
  int64_t dims[3] = {1, 1, 1};
  for (int s = 0; s < d; ++s) dims[s] = dir == 0 ? wd.box_w[s] : M;
  double2* in = a;
  double2* out = b;
  for (int axis = d - 1; axis >= 0; --axis) {
    int64_t A = 1, B = 1;
    for (int s = 0; s < axis; ++s) A *= dims[s];
    for (int s = axis + 1; s < d; ++s) B *= dims[s];
    const int nin = (int)dims[axis];
    const int nout = dir == 0 ? M : wd.box_w[axis];
    k_dft_pass<<<nblocks(A * nout * B), 256, 0, st>>>(in, out, A, nin, nout, B, wd.n, M,
                                                      wd.box_lo[axis], wd.wrap, dir);
    NLD_CUDA(cudaGetLastError());
    dims[axis] = nout;
    std::swap(in, out);
  }
  return in;
}

int64_t scratch_len(const WinDev& wd, int M) {
  // largest intermediate of either pass direction
  int64_t best = 1;
  for (int dir = 0; dir < 2; ++dir) {
    int64_t dims[3] = {1, 1, 1};
    for (int s = 0; s < wd.d; ++s) dims[s] = dir == 0 ? wd.box_w[s] : M;
    int64_t cur = dims[0] * dims[1] * dims[2];
    best = std::max(best, cur);
    for (int axis = wd.d - 1; axis >= 0; --axis) {
      dims[axis] = dir == 0 ? M : wd.box_w[axis];
      best = std::max(best, dims[0] * dims[1] * dims[2]);
    }
  }
  return best;
}

}  // namespace
}  // namespace nld

using nld::Error;

namespace {

template <typename F>
int guard(F&& fn) {
  try {
    fn();
    return NLD_OK;
  } catch (const Error& e) {
    return nld::fail(e.code, e.msg);
  } catch (...) {
    return nld::fail(NLD_ERR_CUDA, "unknown failure");
  }
}

void select_device(const void* ptr) {
  int dev = 0;
  cudaPointerAttributes attr;
  if (ptr && cudaPointerGetAttributes(&attr, ptr) == cudaSuccess &&
      attr.type == cudaMemoryTypeDevice)
    dev = attr.device;
  else
    cudaGetLastError();
  NLD_CUDA(cudaSetDevice(dev));
}

int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

void build_raw(nld_operator* op, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(op->build_mu);
  if (op->built[0]) return;
  nld::build_planset(op, 0, st);
  op->built[0] = true;
}

}  // namespace

extern "C" {

int nld_nfft_create(const double* nodes_dev, int64_t n, int32_t d, int32_t bandwidth,
                    double oversampling, int32_t cutoff, const double* center, double scale,
                    int32_t check_torus, void* stream, nld_operator** out) {
  return guard([&] {
    if (!out) throw Error(NLD_ERR_VALUE, "null output handle");
    *out = nullptr;
    if (n <= 0) throw Error(NLD_ERR_DIMENSION, "at least one node is required");
    if (d < 1 || d > 3) throw Error(NLD_ERR_DIMENSION, "nodes must be (N, d) with d <= 3");
    if (bandwidth <= 0 || bandwidth % 2) throw Error(NLD_ERR_VALUE, "bandwidths must be even positive integers");
    if (oversampling < 1.25) throw Error(NLD_ERR_VALUE, "oversampling factor must be >= 1.25");
    if (cutoff < 1 || cutoff > 8) throw Error(NLD_ERR_VALUE, "window cutoff must lie in [1, 8]");
    select_device(nodes_dev);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* op = new nld_operator();
    try {
      NLD_CUDA(cudaGetDevice(&op->device));
      op->N = op->N_global = n;
      op->D = d;
      op->L = 1;
      op->sigma = 1.0;
      op->params.n_expansion = bandwidth;
      op->params.cutoff = cutoff;
      op->params.oversampling = oversampling;
      op->params.rmax = 0.25;
      op->params.truncation_eps = 1e-8;
      op->params.mode = 0;
      op->params.dense_limit = 0;
      op->raw = 1;
      op->raw_check = check_torus ? 1 : 0;
      for (int s = 0; s < d; ++s) op->raw_center[s] = center ? center[s] : 0.0;
      op->raw_scale = scale;
      op->win_offset = {0, d};
      op->win_index.resize(d);
      for (int s = 0; s < d; ++s) op->win_index[s] = s;
      NLD_CUDA(cudaMalloc(&op->feats, sizeof(double) * n * d));
      NLD_CUDA(cudaMemcpyAsync(op->feats, nodes_dev, sizeof(double) * n * d,
                               cudaMemcpyDeviceToDevice, st));
      build_raw(op, st);
    } catch (...) {
      if (op->built[0]) nld::free_planset(op->sets[0]);
      cudaFree(op->feats);
      delete op;
      throw;
    }
    *out = op;
  });
}

int nld_nfft_adjoint(nld_operator* op, const double* values, double* coeffs,
                     const double* mult, void* stream) {
  return guard([&] {
    if (!op || !op->raw) throw Error(NLD_ERR_VALUE, "not an NFFT plan");
    NLD_CUDA(cudaSetDevice(op->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const nld::PlanSet& ps = op->sets[0];
    nld::ensure_workspace(op, ps, 2);
    const nld::WinDev& wd = ps.wdev_h[0];
    const nld::WinPlan& wp = ps.win[0];
    const int M = wp.M;
    // spread the complex values (two interleaved rhs) into the support box
    nld::spread_stage(op, ps, values, 2, st);
    const int64_t len = nld::scratch_len(wd, M);
    double2 *a = nullptr, *b = nullptr;
    double* c = nullptr;
    NLD_CUDA(cudaMallocAsync(&a, sizeof(double2) * len, st));
    NLD_CUDA(cudaMallocAsync(&b, sizeof(double2) * len, st));
    NLD_CUDA(cudaMallocAsync(&c, sizeof(double) * M, st));
    nld::k_planes_to_complex<<<nld::nblocks(wd.box_size), 256, 0, st>>>(
        op->ws.grid_in, ps.grid_total, wd.box_size, a);
    double2* res = nld::dft_passes(wd, M, a, b, 0, st);
    nld::k_window_factors<<<1, 256, 0, st>>>(c, M, wd.n, wp.m, wp.b);
    nld::k_deconvolve<<<nld::nblocks(ipow(M, wd.d)), 256, 0, st>>>(
        res, reinterpret_cast<double2*>(coeffs), c, M, wd.d, mult);
    NLD_CUDA(cudaGetLastError());
    cudaFreeAsync(a, st);
    cudaFreeAsync(b, st);
    cudaFreeAsync(c, st);
  });
}

int nld_nfft_trafo(nld_operator* op, const double* coeffs, double* values, void* stream) {
  return guard([&] {
    if (!op || !op->raw) throw Error(NLD_ERR_VALUE, "not an NFFT plan");
    NLD_CUDA(cudaSetDevice(op->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const nld::PlanSet& ps = op->sets[0];
    nld::ensure_workspace(op, ps, 2);
    const nld::WinDev& wd = ps.wdev_h[0];
    const nld::WinPlan& wp = ps.win[0];
    const int M = wp.M;
    const int64_t len = nld::scratch_len(wd, M);
    double2 *a = nullptr, *b = nullptr;
    double* c = nullptr;
    NLD_CUDA(cudaMallocAsync(&a, sizeof(double2) * len, st));
    NLD_CUDA(cudaMallocAsync(&b, sizeof(double2) * len, st));
    NLD_CUDA(cudaMallocAsync(&c, sizeof(double) * M, st));
    nld::k_window_factors<<<1, 256, 0, st>>>(c, M, wd.n, wp.m, wp.b);
    nld::k_deconvolve<<<nld::nblocks(ipow(M, wd.d)), 256, 0, st>>>(
        reinterpret_cast<const double2*>(coeffs), a, c, M, wd.d, nullptr);
    double2* res = nld::dft_passes(wd, M, a, b, 1, st);
    nld::k_complex_to_planes<<<nld::nblocks(wd.box_size), 256, 0, st>>>(
        res, wd.box_size, ps.grid_total, op->ws.grid_out);
    NLD_CUDA(cudaGetLastError());
    nld::gather_stage(op, ps, 2, st);
    // wout is [1][N][2]: interleaved complex already
    NLD_CUDA(cudaMemcpyAsync(values, op->ws.wout, sizeof(double) * 2 * op->N,
                             cudaMemcpyDeviceToDevice, st));
    cudaFreeAsync(a, st);
    cudaFreeAsync(b, st);
    cudaFreeAsync(c, st);
  });
}

int nld_ndft(const double* nodes, int64_t n, int32_t d, int32_t bandwidth, const double* in,
             double* out, int32_t adjoint, void* stream) {
  return guard([&] {
    if (d < 1 || d > 3) throw Error(NLD_ERR_DIMENSION, "nodes must be (N, d) with d <= 3");
    select_device(nodes);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (adjoint)
      nld::k_ndft_adjoint<<<nld::nblocks(ipow(bandwidth, d), 128), 128, 0, st>>>(
          nodes, n, d, bandwidth, reinterpret_cast<const double2*>(in),
          reinterpret_cast<double2*>(out));
    else
      nld::k_ndft<<<nld::nblocks(n, 128), 128, 0, st>>>(nodes, n, d, bandwidth,
                                                         reinterpret_cast<const double2*>(in),
                                                         reinterpret_cast<double2*>(out));
    NLD_CUDA(cudaGetLastError());
  });
}

int nld_gauss_direct(const double* targets, int64_t nt, const double* sources, int64_t ns,
                     int32_t d, const double* alpha, double sigbar, double* out, void* stream) {
  return guard([&] {
    if (!(sigbar > 0)) throw Error(NLD_ERR_VALUE, "shape parameter must be positive");
    select_device(targets);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    nld::k_gauss_direct<<<nld::nblocks(nt, 128), 128, 0, st>>>(targets, nt, sources, ns, d,
                                                               alpha, sigbar, out);
    NLD_CUDA(cudaGetLastError());
  });
}

int nld_gauss_coeffs(int32_t bandwidth, int32_t d, double sig_scaled, double* out,
                     void* stream) {
  return guard([&] {
    select_device(out);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    nld::k_gauss_coeffs<<<1, 256, sizeof(double) * bandwidth, st>>>(bandwidth, d, sig_scaled,
                                                                    out);
    NLD_CUDA(cudaGetLastError());
  });
}

int nld_fastsum_geometry(const double* points, int64_t n, int32_t d, double rmax,
                         double* center_host, double* scale_host, void* stream) {
  return guard([&] {
    if (n <= 0) throw Error(NLD_ERR_VALUE, "cannot build a plan from an empty point set");
    if (d < 1 || d > 3) throw Error(NLD_ERR_DIMENSION, "points must be (N, d) with d <= 3");
    if (!(rmax > 0 && rmax <= 0.25)) throw Error(NLD_ERR_VALUE, "rmax must lie in (0, 1/4]");
    select_device(points);
    nld::point_geometry(points, n, d, rmax, center_host, scale_host,
                        static_cast<cudaStream_t>(stream));
  });
}

int nld_window_factors(int32_t bandwidth, int32_t grid, int32_t cutoff, double* out_host) {
  return guard([&] {
    double* c = nullptr;
    NLD_CUDA(cudaMalloc(&c, sizeof(double) * bandwidth));
    const double b = 3.141592653589793 * (2.0 - (double)bandwidth / (double)grid);
    nld::k_window_factors<<<1, 256>>>(c, bandwidth, grid, cutoff, b);
    NLD_CUDA(cudaGetLastError());
    NLD_CUDA(cudaMemcpy(out_host, c, sizeof(double) * bandwidth, cudaMemcpyDeviceToHost));
    cudaFree(c);
  });
}

}  // extern "C"
