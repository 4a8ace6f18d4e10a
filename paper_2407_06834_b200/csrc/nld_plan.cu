// Plan build: torus scaling, Kaiser-Bessel node tables, one-time cell sort,
// subproblem lists and the fused separable convolution kernel K.
//
// Restates, on the device, FastsumPlan.build / map_to_torus / tables_for
// (transform.py:272-320) and NfftPlan.node_tables / window_factors
// (transform.py:140-170) as used lazily by AnovaOperator._build_plans
// (kernel.py:70-77).  Every floating-point step that decides a stencil
// base or a weight uses explicitly rounded operations (no FMA contraction)
// in the same order as the numpy code, so bases are bit-identical and
// weights agree to the ulp-level of sinh.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "nld_internal.cuh"

namespace nld {

namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;   // 2 x 148 SMs

template <typename T>
T* dalloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  NLD_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

struct TmpBuf {
  void* p = nullptr;
  cudaStream_t st;
  explicit TmpBuf(size_t bytes, cudaStream_t s) : st(s) {
    NLD_CUDA(cudaMallocAsync(&p, bytes ? bytes : 1, s));
  }
  ~TmpBuf() { cudaFreeAsync(p, st); }
  template <typename T> T* as() { return static_cast<T*>(p); }
};

// ---- bounding box and radius (transform.py:292-295) ----------------------

__global__ void k_minmax(const double* __restrict__ F, int64_t N, int D,
                         int3 cols, int d, double* __restrict__ part) {
  // part[blk][2*d]: min then max per dim; min/max are order independent.
  __shared__ double smin[kRedThreads][3], smax[kRedThreads][3];
  double lo[3] = {INFINITY, INFINITY, INFINITY};
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int c[3] = {cols.x, cols.y, cols.z};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < d; ++s) {
      double p = F[j * D + c[s]];
      lo[s] = fmin(lo[s], p);
      hi[s] = fmax(hi[s], p);
    }
  }
  for (int s = 0; s < 3; ++s) {
    smin[threadIdx.x][s] = lo[s];
    smax[threadIdx.x][s] = hi[s];
  }
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      for (int s = 0; s < 3; ++s) {
        smin[threadIdx.x][s] = fmin(smin[threadIdx.x][s], smin[threadIdx.x + off][s]);
        smax[threadIdx.x][s] = fmax(smax[threadIdx.x][s], smax[threadIdx.x + off][s]);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < d; ++s) {
      part[blockIdx.x * 6 + s] = smin[0][s];
      part[blockIdx.x * 6 + 3 + s] = smax[0][s];
    }
  }
}

// max_j sum_s (p_js - c_s)^2, summed left to right like numpy's row sum
__global__ void k_radius2(const double* __restrict__ F, int64_t N, int D,
                          int3 cols, int d, double3 ctr,
                          double* __restrict__ part) {
  __shared__ double sm[kRedThreads];
  double best = 0.0;
  int c[3] = {cols.x, cols.y, cols.z};
  double cc[3] = {ctr.x, ctr.y, ctr.z};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    double r2 = 0.0;
    for (int s = 0; s < d; ++s) {
      double dx = __dsub_rn(F[j * D + c[s]], cc[s]);
      double sq = __dmul_rn(dx, dx);
      r2 = (s == 0) ? sq : __dadd_rn(r2, sq);
    }
    best = fmax(best, r2);
  }
  sm[threadIdx.x] = best;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
      sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}

// ---- node tables (transform.py:147-170, :310-320) -------------------------

struct TorusMap {
  double c[3];
  double scale;
  double nf;       // grid size as double
  int m;
  double b;        // KB shape
  double b_pi;     // b / pi
  int check;       // raise ScalingOverflowError for |q| >= 1/2
};

__device__ __forceinline__ double torus_x(const TorusMap& t, double p, int s) {
  double q = __dmul_rn(__dsub_rn(p, t.c[s]), t.scale);
  return q;
}

// KB weight at stencil offset `lo + i` (transform.py:163-168)
__device__ __forceinline__ double kb_weight(const TorusMap& t, double xs,
                                            long long pos) {
  double u = __dsub_rn(xs, (double)pos);
  double tt = __dsub_rn((double)(t.m * t.m), __dmul_rn(u, u));
  if (fabs(tt) <= 1e-14) return t.b_pi;
  if (tt > 0.0) {
    double root = sqrt(tt);
    return sinh(__dmul_rn(t.b, root)) / __dmul_rn(3.141592653589793, root);
  }
  return 0.0;
}

__global__ void k_bases(const double* __restrict__ F, int64_t N, int D,
                        int3 cols, int d, TorusMap tm,
                        int32_t* __restrict__ base, int* __restrict__ flags) {
  int c[3] = {cols.x, cols.y, cols.z};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < d; ++s) {
      double q = torus_x(tm, F[j * D + c[s]], s);
      if (tm.check && !(fabs(q) < 0.5)) atomicOr(flags, 1);   // ScalingOverflowError
      double xs = __dmul_rn(q, tm.nf);
      long long lo = (long long)floor(xs) - tm.m;
      base[j * 3 + s] = (int32_t)lo;
    }
  }
}

__global__ void k_minmax_int(const int32_t* __restrict__ base, int64_t N,
                             int d, int* __restrict__ out /* [6] */) {
  __shared__ int smin[kRedThreads][3], smax[kRedThreads][3];
  int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
  int hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    for (int s = 0; s < d; ++s) {
      int b = base[j * 3 + s];
      lo[s] = min(lo[s], b);
      hi[s] = max(hi[s], b);
    }
  }
  for (int s = 0; s < 3; ++s) {
    smin[threadIdx.x][s] = lo[s];
    smax[threadIdx.x][s] = hi[s];
  }
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
      for (int s = 0; s < 3; ++s) {
        smin[threadIdx.x][s] = min(smin[threadIdx.x][s], smin[threadIdx.x + off][s]);
        smax[threadIdx.x][s] = max(smax[threadIdx.x][s], smax[threadIdx.x + off][s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int s = 0; s < d; ++s) {
      atomicMin(out + s, smin[0][s]);
      atomicMax(out + 3 + s, smax[0][s]);
    }
}

struct BoxDev {
  int lo[3];
  int w[3];
  int wrap;
  int n;
  int d;
};

// box coordinate of unwrapped grid position `pos` along one dimension
__device__ __forceinline__ int box_coord(const BoxDev& bx, int s, long long pos) {
  if (bx.wrap) {
    long long r = pos % bx.n;
    return (int)(r < 0 ? r + bx.n : r);
  }
  return (int)(pos - bx.lo[s]);
}

__global__ void k_keys(const int32_t* __restrict__ base, int64_t N, BoxDev bx,
                       int32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    int key = 0;
    for (int s = 0; s < bx.d; ++s)
      key = key * bx.w[s] + box_coord(bx, s, (long long)base[j * 3 + s] + 1);
    keys[j] = key;
    idx[j] = (int32_t)j;
  }
}

// sorted rows of principal weights (offsets i = 1..2m) + edge flags
__global__ void k_rows(const double* __restrict__ F, int64_t N, int D,
                       int3 cols, int d, TorusMap tm,
                       const int32_t* __restrict__ perm,
                       double* __restrict__ rows, int32_t* __restrict__ pix,
                       int* __restrict__ edge_flag) {
  const int S = 2 * tm.m;
  const int W = S + 2;
  int c[3] = {cols.x, cols.y, cols.z};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    int j = perm[e];
    pix[e] = j;
    int edge = 0;
    for (int s = 0; s < d; ++s) {
      double xs = __dmul_rn(torus_x(tm, F[(int64_t)j * D + c[s]], s), tm.nf);
      long long lo = (long long)floor(xs) - tm.m;
      for (int i = 1; i <= S; ++i)
        rows[e * (S * d) + s * S + (i - 1)] = kb_weight(tm, xs, lo + i);
      if (kb_weight(tm, xs, lo) != 0.0 || kb_weight(tm, xs, lo + W - 1) != 0.0)
        edge = 1;
    }
    edge_flag[e] = edge;
  }
}

__global__ void k_edges(const double* __restrict__ F, int64_t N, int D,
                        int3 cols, int d, TorusMap tm, BoxDev bx, int win,
                        const int32_t* __restrict__ sel, const int* __restrict__ nsel,
                        const int32_t* __restrict__ pix, EdgeDev* __restrict__ out) {
  const int W = 2 * tm.m + 2;
  int c[3] = {cols.x, cols.y, cols.z};
  int count = *nsel;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += gridDim.x * blockDim.x) {
    int e = sel[k];
    int j = pix[e];
    EdgeDev ed;
    ed.pix = j;
    ed.win = win;
    ed.pad = 0;
    for (int s = 0; s < 3; ++s) {
      ed.cc[s] = 0;
      for (int i = 0; i < 18; ++i) ed.w[s][i] = (s >= d && i == 1) ? 1.0 : 0.0;
    }
    for (int s = 0; s < d; ++s) {
      double xs = __dmul_rn(torus_x(tm, F[(int64_t)j * D + c[s]], s), tm.nf);
      long long lo = (long long)floor(xs) - tm.m;
      ed.cc[s] = box_coord(bx, s, lo + 1);
      for (int i = 0; i < W; ++i) ed.w[s][i] = kb_weight(tm, xs, lo + i);
    }
    out[k] = ed;
  }
}

#ifndef NLD_SUB_BALANCED
#define NLD_SUB_BALANCED 1
#endif
// cells and their subproblems
__global__ void k_cells(const int32_t* __restrict__ ukeys,
                        const int32_t* __restrict__ counts,
                        const int32_t* __restrict__ starts,
                        const int32_t* __restrict__ sub_first, int ncell,
                        BoxDev bx, int win, int64_t node_off, int cell_off,
                        int64_t block_base, int blk, int sub_max, CellDev* __restrict__ cells,
                        SubDev* __restrict__ subs, int32_t* __restrict__ cellmap) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncell;
       k += gridDim.x * blockDim.x) {
    int key = ukeys[k];
    CellDev cd;
    int rem = key;
    cd.cc[0] = cd.cc[1] = cd.cc[2] = 0;
    for (int s = bx.d - 1; s >= 0; --s) {
      cd.cc[s] = rem % bx.w[s];
      rem /= bx.w[s];
    }
    int first = sub_first[k];
    int cnt = counts[k];
    int nsub = (cnt + sub_max - 1) / sub_max;
    cd.win = win;
    cd.block0 = block_base + (int64_t)first * blk;
    cd.nsub = nsub;
    cd.blk = blk;
    cells[k] = cd;
    cellmap[key] = cell_off + k;
#if NLD_SUB_BALANCED
    const int per = sub_size(cnt, max(nsub, 1));
#else
    const int per = sub_max;
#endif
    for (int q = 0; q < nsub; ++q) {
      SubDev sd;
      sd.start = node_off + starts[k] + (int64_t)q * per;
      sd.block = cd.block0 + (int64_t)q * blk;
      sd.count = min(per, cnt - q * per);
      sd.cell = cell_off + k;
      sd.win = win;
      sd.pad = 0;
      subs[first + q] = sd;
    }
  }
}

__global__ void k_cellinfo(const int32_t* __restrict__ cellmap, const CellDev* __restrict__ cells,
                           int64_t n, int2* __restrict__ info) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int c = cellmap[k];
    info[k] = c < 0 ? make_int2(0, 0) : make_int2((int)cells[c].block0, cells[c].nsub);
  }
}

__global__ void k_nsub(const int32_t* __restrict__ counts, int ncell, int sub_max,
                       int32_t* __restrict__ nsub) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ncell;
       k += gridDim.x * blockDim.x)
    nsub[k] = (counts[k] + sub_max - 1) / sub_max;
}

__global__ void k_iota(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_fill_int(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Separable fused convolution kernel of one window (transform.py:296-307,
// 140-145, 200-223): K(delta) = sum_k e_k exp(+2 pi i k delta / n),
// e_k = c1_k / c(k)^2, c1 = 1-D ifft of the sampled Gaussian, c = I0 factor.
__global__ void k_kernel_table(double2* __restrict__ K, int n, int M, int m,
                               double b, double sig) {
  extern __shared__ double e[];   // M entries
  for (int kk = threadIdx.x; kk < M; kk += blockDim.x) {
    int k = kk - M / 2;
    double acc = 0.0;
    for (int jj = 0; jj < M; ++jj) {
      int j = jj - M / 2;
      double jm = (double)j / (double)M;
      double g = exp(-(sig * (jm * jm)));
      int ph = ((k * j) % M + M) % M;
      acc += g * cospi(2.0 * (double)ph / (double)M);
    }
    double c1 = acc / (double)M;
    double w = (2.0 * 3.141592653589793 * (double)k) / (double)n;
    double arg = b * b - w * w;
    double cf = cyl_bessel_i0((double)m * sqrt(arg));
    e[kk] = (c1 / cf) / cf;
  }
  __syncthreads();
  for (int dl = threadIdx.x; dl < n; dl += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int kk = 0; kk < M; ++kk) {
      int k = kk - M / 2;
      int ph = ((k * dl) % n + n) % n;
      double sn, cs;
      sincospi(2.0 * (double)ph / (double)n, &sn, &cs);
      re += e[kk] * cs;
      im += e[kk] * sn;
    }
    K[dl] = make_double2(re, im);
  }
}

int blocks_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

int64_t expansion_degree(double sig_scaled, double eps) {
  // transform.py:254-258
  double k = std::ceil(std::sqrt(std::max(sig_scaled, 1.0) * std::log(1.0 / eps)) /
                       3.141592653589793);
  int64_t n = 2 * std::max<int64_t>(16 / 2, (int64_t)k + 1);
  return std::min<int64_t>(n, 192);
}

// FastsumPlan.build geometry (transform.py:292-296): centre of the bounding
// box and scale = rmax / max radius, for an (n, d) point set
void point_geometry(const double* F, int64_t N, int d, double rmax, double* center,
                    double* scale, cudaStream_t st) {
  const int nb = kRedBlocks;
  TmpBuf part(sizeof(double) * nb * 6, st);
  std::vector<double> hpart(nb * 6);
  int3 cols = make_int3(0, d > 1 ? 1 : 0, d > 2 ? 2 : 0);
  k_minmax<<<nb, kRedThreads, 0, st>>>(F, N, d, cols, d, part.as<double>());
  NLD_CUDA(cudaMemcpyAsync(hpart.data(), part.p, sizeof(double) * nb * 6,
                           cudaMemcpyDeviceToHost, st));
  NLD_CUDA(cudaStreamSynchronize(st));
  for (int s = 0; s < d; ++s) {
    double lo = INFINITY, hi = -INFINITY;
    for (int k = 0; k < nb; ++k) {
      lo = std::min(lo, hpart[k * 6 + s]);
      hi = std::max(hi, hpart[k * 6 + 3 + s]);
    }
    center[s] = 0.5 * (lo + hi);
  }
  k_radius2<<<nb, kRedThreads, 0, st>>>(F, N, d, cols, d,
                                        make_double3(center[0], d > 1 ? center[1] : 0.0,
                                                     d > 2 ? center[2] : 0.0),
                                        part.as<double>());
  NLD_CUDA(cudaMemcpyAsync(hpart.data(), part.p, sizeof(double) * nb, cudaMemcpyDeviceToHost,
                           st));
  NLD_CUDA(cudaStreamSynchronize(st));
  double r2 = 0.0;
  for (int k = 0; k < nb; ++k) r2 = std::max(r2, hpart[k]);
  *scale = rmax / std::max(std::sqrt(r2), 1e-30);
}

static bool window_fast(int d, int m) {
  return (m >= 3 && m <= 5) && d >= 1 && d <= 3;
}

void build_planset(nld_operator* op, int which, cudaStream_t st) {
  PlanSet& ps = op->sets[which];
  const int64_t N = op->N;
  const int L = op->L;
  const nld_params& P = op->params;
  ps.sigbar = (which ? 2.0 : 1.0) / (op->sigma * op->sigma);
  ps.win.assign(L, WinPlan());
  const int m = P.cutoff;
  const int S = 2 * m;
  const int nb = kRedBlocks;

  // does the other plan set exist with identical tables?
  PlanSet* other = op->built[1 - which] ? &op->sets[1 - which] : nullptr;

  TmpBuf part(sizeof(double) * nb * 6, st);
  std::vector<double> hpart(nb * 6);
  for (int w = 0; w < L; ++w) {
    WinPlan& wp = ps.win[w];
    wp.d = op->win_offset[w + 1] - op->win_offset[w];
    for (int s = 0; s < wp.d; ++s) wp.cols[s] = op->win_index[op->win_offset[w] + s];
    int3 cols = make_int3(wp.cols[0], wp.cols[1], wp.cols[2]);
    if (op->raw) {
      for (int s = 0; s < wp.d; ++s) wp.center[s] = op->raw_center[s];
      wp.scale = op->raw_scale;
      wp.sig_scaled = 0.0;
    } else {
    k_minmax<<<nb, kRedThreads, 0, st>>>(op->feats, N, op->D, cols, wp.d,
                                         part.as<double>());
    NLD_CUDA(cudaMemcpyAsync(hpart.data(), part.p, sizeof(double) * nb * 6,
                             cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int s = 0; s < wp.d; ++s) {
      for (int k = 0; k < nb; ++k) {
        lo[s] = std::min(lo[s], hpart[k * 6 + s]);
        hi[s] = std::max(hi[s], hpart[k * 6 + 3 + s]);
      }
    }
    // global bounding box across pixel shards (transform.py:292-293)
    comm_host(op, lo, wp.d, RED_F64, RED_OP_MIN);
    comm_host(op, hi, wp.d, RED_F64, RED_OP_MAX);
    for (int s = 0; s < wp.d; ++s) wp.center[s] = 0.5 * (lo[s] + hi[s]);
    k_radius2<<<nb, kRedThreads, 0, st>>>(
        op->feats, N, op->D, cols, wp.d,
        make_double3(wp.center[0], wp.center[1], wp.center[2]), part.as<double>());
    NLD_CUDA(cudaMemcpyAsync(hpart.data(), part.p, sizeof(double) * nb,
                             cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    double r2 = 0.0;
    for (int k = 0; k < nb; ++k) r2 = std::max(r2, hpart[k]);
    comm_host(op, &r2, 1, RED_F64, RED_OP_MAX);
    double radius = std::sqrt(r2);
    wp.scale = P.rmax / std::max(radius, 1e-30);
    wp.sig_scaled = ps.sigbar / (wp.scale * wp.scale);
    }
    int64_t M = P.n_expansion > 0 ? P.n_expansion
                                  : expansion_degree(wp.sig_scaled, P.truncation_eps);
    if (M % 2) throw Error(NLD_ERR_VALUE, "expansion degree must be even");
    wp.M = (int)M;
    wp.n = 2 * (int)std::ceil(P.oversampling * (double)M / 2.0);
    wp.m = m;
    wp.b = 3.141592653589793 * (2.0 - (double)wp.M / (double)wp.n);
  }

  // share node tables with the other plan set when every window matches
  bool share = other != nullptr;
  if (share) {
    for (int w = 0; w < L; ++w) {
      const WinPlan& a = ps.win[w];
      const WinPlan& b = other->win[w];
      if (a.n != b.n || a.M != b.M || a.scale != b.scale) share = false;
      for (int s = 0; s < a.d; ++s)
        if (a.center[s] != b.center[s]) share = false;
    }
  }

  ps.wdev_h.assign(L, WinDev());
  int64_t kern_total = 0;
  for (int w = 0; w < L; ++w) kern_total += ps.win[w].n;
  ps.K = dalloc<double2>(kern_total);
  {
    int64_t koff = 0;
    for (int w = 0; w < L; ++w) {
      const WinPlan& wp = ps.win[w];
      k_kernel_table<<<1, 256, sizeof(double) * wp.M, st>>>(
          ps.K + koff, wp.n, wp.M, wp.m, wp.b, wp.sig_scaled);
      NLD_CUDA(cudaGetLastError());
      ps.wdev_h[w].kern_off = koff;
      koff += wp.n;
    }
  }

  if (share) {
    // copy geometry, point at the other set's tables
    ps.owns_tables = false;
    ps.shares_tables_with = 1 - which;
    for (int w = 0; w < L; ++w) {
      WinPlan keep = ps.win[w];
      ps.win[w] = other->win[w];
      ps.win[w].sig_scaled = keep.sig_scaled;
      int64_t ko = ps.wdev_h[w].kern_off;
      ps.wdev_h[w] = other->wdev_h[w];
      ps.wdev_h[w].kern_off = ko;
    }
    ps.rows = other->rows;
    ps.pix = other->pix;
    ps.key = other->key;
    ps.cellmap = other->cellmap;
    ps.cellinfo = other->cellinfo;
    ps.cells = other->cells;
    ps.n_cells = other->n_cells;
    for (int g = 0; g <= kMaxDim; ++g) {
      ps.subs[g] = other->subs[g];
      ps.n_subs[g] = other->n_subs[g];
    }
    ps.blocks_total = other->blocks_total;
    ps.edges = other->edges;
    ps.n_edges = other->n_edges;
    ps.grid_total = other->grid_total;
    ps.generic_nodes = other->generic_nodes;
    NLD_CUDA(cudaMalloc(&ps.wdev, sizeof(WinDev) * L));
    NLD_CUDA(cudaMemcpyAsync(ps.wdev, ps.wdev_h.data(), sizeof(WinDev) * L,
                             cudaMemcpyHostToDevice, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    return;
  }

  // ---- full tables -------------------------------------------------------
  int64_t row_total = 0;
  for (int w = 0; w < L; ++w) row_total += N * (int64_t)S * ps.win[w].d;
  ps.rows = dalloc<double>(row_total);
  ps.pix = dalloc<int32_t>(N * L);
  ps.key = dalloc<int32_t>(N * L);

  TmpBuf base(sizeof(int32_t) * N * 3, st);
  TmpBuf keys_in(sizeof(int32_t) * N, st), idx_in(sizeof(int32_t) * N, st);
  TmpBuf perm(sizeof(int32_t) * N, st);
  TmpBuf flags(sizeof(int) * 8, st);
  TmpBuf edge_flag(sizeof(int) * N, st);
  TmpBuf ukeys(sizeof(int32_t) * N, st), counts(sizeof(int32_t) * N, st);
  TmpBuf starts(sizeof(int32_t) * N, st), nsubs(sizeof(int32_t) * N, st);
  TmpBuf subfirst(sizeof(int32_t) * N, st);
  TmpBuf nrun(sizeof(int) * 2, st);

  // per-window cell/sub/edge host bookkeeping
  struct WinCells {
    int64_t ncell = 0, nsub = 0, nedge = 0;
    CellDev* cells = nullptr;   // temporary per-window arrays
    SubDev* subs = nullptr;
    EdgeDev* edges = nullptr;
  };
  std::vector<WinCells> wc(L);
  int64_t cellmap_total = 0;
  std::vector<int64_t> cellmap_off(L);
  std::vector<int32_t*> cellmaps(L, nullptr);
  int64_t grid_total = 0;
  int64_t row_off = 0;
  int64_t cells_so_far = 0;
  int64_t block_total = 0;
  int64_t subs_in_group[kMaxDim + 1] = {0, 0, 0, 0};
  std::vector<int64_t> sub_group_off(L);

  for (int w = 0; w < L; ++w) {
    WinPlan& wp = ps.win[w];
    int3 cols = make_int3(wp.cols[0], wp.cols[1], wp.cols[2]);
    TorusMap tm;
    for (int s = 0; s < 3; ++s) tm.c[s] = wp.center[s];
    tm.scale = wp.scale;
    tm.nf = (double)wp.n;
    tm.m = m;
    tm.b = wp.b;
    tm.b_pi = wp.b / 3.141592653589793;
    tm.check = op->raw ? op->raw_check : 1;
    NLD_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 8, st));
    int nbk = blocks_for(N);
    k_bases<<<nbk, 256, 0, st>>>(op->feats, N, op->D, cols, wp.d, tm,
                                 base.as<int32_t>(), flags.as<int>());
    // layout in flags: [0] overflow, [1..3] min, [4..6] max
    int init[8] = {0, INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN,
                   INT32_MIN, 0};
    NLD_CUDA(cudaMemcpyAsync(flags.as<int>() + 1, init + 1, sizeof(int) * 6,
                             cudaMemcpyHostToDevice, st));
    k_minmax_int<<<nb, kRedThreads, 0, st>>>(base.as<int32_t>(), N, wp.d,
                                             flags.as<int>() + 1);
    int hf[8];
    NLD_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    // global support box and overflow flag across shards
    comm_host(op, hf, 1, RED_I32, RED_OP_MAX);
    comm_host(op, hf + 1, 3, RED_I32, RED_OP_MIN);
    comm_host(op, hf + 4, 3, RED_I32, RED_OP_MAX);
    if (hf[0]) throw Error(NLD_ERR_SCALING, "scaled nodes leave the torus [-1/2, 1/2)^d");
    BoxDev bx;
    bx.d = wp.d;
    bx.n = wp.n;
    bx.wrap = 0;
    for (int s = 0; s < 3; ++s) {
      bx.lo[s] = 0;
      bx.w[s] = 1;
    }
    for (int s = 0; s < wp.d; ++s) {
      int lo = hf[1 + s];
      int hi = hf[4 + s] + 2 * m + 1;
      if (hi - lo + 1 > wp.n) bx.wrap = 1;
      bx.lo[s] = lo;
      bx.w[s] = hi - lo + 1;
    }
    if (bx.wrap)
      for (int s = 0; s < wp.d; ++s) {
        bx.lo[s] = 0;
        bx.w[s] = wp.n;
      }
    int64_t box_size = 1;
    for (int s = 0; s < wp.d; ++s) box_size *= bx.w[s];
    if (box_size > (int64_t)INT32_MAX)
      throw Error(NLD_ERR_VALUE, "support box too large");
    for (int s = 0; s < 3; ++s) {
      wp.box_lo[s] = bx.lo[s];
      wp.box_w[s] = bx.w[s];
    }
    wp.wrap = bx.wrap;

    // keys + stable radix sort by cell
    k_keys<<<nbk, 256, 0, st>>>(base.as<int32_t>(), N, bx, keys_in.as<int32_t>(),
                                idx_in.as<int32_t>());
    int end_bit = 1;
    while (end_bit < 31 && ((int64_t)1 << end_bit) < box_size) ++end_bit;
    int32_t* keys_sorted = ps.key + (int64_t)w * N;
    size_t tbytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tbytes, keys_in.as<int32_t>(), keys_sorted,
                                    idx_in.as<int32_t>(), perm.as<int32_t>(), (int)N,
                                    0, end_bit, st);
    {
      TmpBuf tmp(tbytes, st);
      NLD_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tbytes, keys_in.as<int32_t>(),
                                               keys_sorted, idx_in.as<int32_t>(),
                                               perm.as<int32_t>(), (int)N, 0, end_bit,
                                               st));
    }
    double* rows_w = ps.rows + row_off;
    k_rows<<<nbk, 256, 0, st>>>(op->feats, N, op->D, cols, wp.d, tm, perm.as<int32_t>(),
                                rows_w, ps.pix + (int64_t)w * N, edge_flag.as<int>());
    NLD_CUDA(cudaGetLastError());

    // run-length encode the sorted keys -> occupied cells
    tbytes = 0;
    cub::DeviceRunLengthEncode::Encode(nullptr, tbytes, keys_sorted, ukeys.as<int32_t>(),
                                       counts.as<int32_t>(), nrun.as<int>(), (int)N, st);
    {
      TmpBuf tmp(tbytes, st);
      NLD_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, tbytes, keys_sorted,
                                                  ukeys.as<int32_t>(), counts.as<int32_t>(),
                                                  nrun.as<int>(), (int)N, st));
    }
    int ncell = 0;
    NLD_CUDA(cudaMemcpyAsync(&ncell, nrun.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    tbytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbytes, counts.as<int32_t>(),
                                  starts.as<int32_t>(), ncell, st);
    {
      TmpBuf tmp(tbytes, st);
      NLD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tbytes, counts.as<int32_t>(),
                                             starts.as<int32_t>(), ncell, st));
    }
    // nodes per subproblem of this window (nld_internal.cuh: sub_cap)
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      NLD_CUDA(cudaGetDevice(&dev));
      NLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    const int sub_max = sub_cap(N, sms);
    k_nsub<<<blocks_for(ncell), 256, 0, st>>>(counts.as<int32_t>(), ncell, sub_max,
                                              nsubs.as<int32_t>());
    tbytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbytes, nsubs.as<int32_t>(),
                                  subfirst.as<int32_t>(), ncell, st);
    {
      TmpBuf tmp(tbytes, st);
      NLD_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tbytes, nsubs.as<int32_t>(),
                                             subfirst.as<int32_t>(), ncell, st));
    }
    int last_first = 0, last_n = 0;
    NLD_CUDA(cudaMemcpyAsync(&last_first, subfirst.as<int32_t>() + (ncell - 1),
                             sizeof(int), cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaMemcpyAsync(&last_n, nsubs.as<int32_t>() + (ncell - 1), sizeof(int),
                             cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    int64_t nsub = (int64_t)last_first + last_n;

    // cell map over the box
    cellmaps[w] = dalloc<int32_t>(box_size);
    k_fill_int<<<blocks_for(box_size), 256, 0, st>>>(cellmaps[w], box_size, -1);
    wc[w].ncell = ncell;
    wc[w].nsub = nsub;
    wc[w].cells = dalloc<CellDev>(ncell);
    wc[w].subs = dalloc<SubDev>(nsub);
    int blk = 1;
    for (int s = 0; s < wp.d; ++s) blk *= S;
    bool fast = window_fast(wp.d, m);
    // blocks of this window are laid out contiguously after previous ones
    k_cells<<<blocks_for(ncell), 256, 0, st>>>(
        ukeys.as<int32_t>(), counts.as<int32_t>(), starts.as<int32_t>(),
        subfirst.as<int32_t>(), ncell, bx, w, (int64_t)w * N, (int)cells_so_far,
        fast ? block_total : 0, blk, sub_max, wc[w].cells, wc[w].subs, cellmaps[w]);
    NLD_CUDA(cudaGetLastError());
    if (fast) {
      block_total += nsub * blk;
      sub_group_off[w] = subs_in_group[wp.d];
      wp.sub_off = subs_in_group[wp.d];
      subs_in_group[wp.d] += nsub;
    } else {
      ps.generic_nodes += N;
      sub_group_off[w] = -1;
    }
    cells_so_far += ncell;

    // edge nodes (weights at i = 0 or 2m+1)
    {
      TmpBuf iota(sizeof(int32_t) * N, st), sel(sizeof(int32_t) * N, st);
      int32_t* io = iota.as<int32_t>();
      k_iota<<<nbk, 256, 0, st>>>(io, N);
      tbytes = 0;
      cub::DeviceSelect::Flagged(nullptr, tbytes, io, edge_flag.as<int>(), sel.as<int32_t>(),
                                 nrun.as<int>(), (int)N, st);
      {
        TmpBuf tmp(tbytes, st);
        NLD_CUDA(cub::DeviceSelect::Flagged(tmp.p, tbytes, io, edge_flag.as<int>(),
                                            sel.as<int32_t>(), nrun.as<int>(), (int)N, st));
      }
      int ne = 0;
      NLD_CUDA(cudaMemcpyAsync(&ne, nrun.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      NLD_CUDA(cudaStreamSynchronize(st));
      wc[w].nedge = ne;
      if (ne > 0) {
        wc[w].edges = dalloc<EdgeDev>(ne);
        k_edges<<<blocks_for(ne), 128, 0, st>>>(op->feats, N, op->D, cols, wp.d, tm, bx,
                                                w, sel.as<int32_t>(), nrun.as<int>(),
                                                ps.pix + (int64_t)w * N, wc[w].edges);
        NLD_CUDA(cudaGetLastError());
      }
      NLD_CUDA(cudaStreamSynchronize(st));
    }

    wp.n_cells = ncell;
    wp.n_subs = nsub;
    wp.n_edge = wc[w].nedge;

    WinDev& wd = ps.wdev_h[w];
    wd.d = wp.d;
    wd.n = wp.n;
    wd.S = S;
    wd.wrap = bx.wrap;
    for (int s = 0; s < 3; ++s) {
      wd.box_w[s] = bx.w[s];
      wd.box_lo[s] = bx.lo[s];
    }
    wd.box_size = box_size;
    wd.grid_off = grid_total;
    wd.cellmap_off = cellmap_total;
    wd.node_off = (int64_t)w * N;
    wd.row_off = row_off;
    wd.fast = fast ? 1 : 0;
    cellmap_off[w] = cellmap_total;
    cellmap_total += box_size;
    grid_total += box_size;
    row_off += N * (int64_t)S * wp.d;
  }

  // ---- concatenate per-window lists ---------------------------------------
  ps.n_cells = cells_so_far;
  ps.cells = dalloc<CellDev>(cells_so_far);
  ps.cellmap = dalloc<int32_t>(cellmap_total);
  int64_t coff = 0, eoff = 0;
  int64_t edge_total = 0;
  for (int w = 0; w < L; ++w) edge_total += wc[w].nedge;
  ps.n_edges = edge_total;
  ps.edges = edge_total ? dalloc<EdgeDev>(edge_total) : nullptr;
  for (int g = 1; g <= kMaxDim; ++g) {
    ps.n_subs[g] = subs_in_group[g];
    ps.subs[g] = subs_in_group[g] ? dalloc<SubDev>(subs_in_group[g]) : nullptr;
  }
  std::vector<int64_t> gfill(kMaxDim + 1, 0);
  for (int w = 0; w < L; ++w) {
    NLD_CUDA(cudaMemcpyAsync(ps.cells + coff, wc[w].cells, sizeof(CellDev) * wc[w].ncell,
                             cudaMemcpyDeviceToDevice, st));
    coff += wc[w].ncell;
    NLD_CUDA(cudaMemcpyAsync(ps.cellmap + cellmap_off[w], cellmaps[w],
                             sizeof(int32_t) * ps.wdev_h[w].box_size,
                             cudaMemcpyDeviceToDevice, st));
    ps.win[w].edge_off = eoff;
    if (wc[w].nedge) {
      NLD_CUDA(cudaMemcpyAsync(ps.edges + eoff, wc[w].edges, sizeof(EdgeDev) * wc[w].nedge,
                               cudaMemcpyDeviceToDevice, st));
      eoff += wc[w].nedge;
    }
    if (ps.wdev_h[w].fast) {
      int g = ps.win[w].d;
      NLD_CUDA(cudaMemcpyAsync(ps.subs[g] + gfill[g], wc[w].subs,
                               sizeof(SubDev) * wc[w].nsub, cudaMemcpyDeviceToDevice, st));
      gfill[g] += wc[w].nsub;
    }
  }
  NLD_CUDA(cudaStreamSynchronize(st));
  for (int w = 0; w < L; ++w) {
    cudaFree(wc[w].cells);
    cudaFree(wc[w].subs);
    if (wc[w].edges) cudaFree(wc[w].edges);
    cudaFree(cellmaps[w]);
  }
  ps.blocks_total = block_total;
  ps.grid_total = grid_total;
  if (block_total >= (int64_t)INT32_MAX)
    throw Error(NLD_ERR_VALUE, "too many subproblem blocks for 32-bit offsets");
  ps.cellinfo = dalloc<int2>(cellmap_total);
  k_cellinfo<<<blocks_for(cellmap_total), 256, 0, st>>>(ps.cellmap, ps.cells, cellmap_total,
                                                        ps.cellinfo);
  NLD_CUDA(cudaGetLastError());
  NLD_CUDA(cudaMalloc(&ps.wdev, sizeof(WinDev) * L));
  NLD_CUDA(cudaMemcpyAsync(ps.wdev, ps.wdev_h.data(), sizeof(WinDev) * L,
                           cudaMemcpyHostToDevice, st));
  NLD_CUDA(cudaStreamSynchronize(st));
}

void free_planset(PlanSet& ps) {
  cudaFree(ps.wdev);
  cudaFree(ps.sub_exp);
  cudaFree(ps.sub_order);
  cudaFree(ps.K);
  if (ps.owns_tables) {
    cudaFree(ps.rows);
    cudaFree(ps.pix);
    cudaFree(ps.key);
    cudaFree(ps.cellmap);
    cudaFree(ps.cellinfo);
    cudaFree(ps.cells);
    for (int g = 0; g <= kMaxDim; ++g) cudaFree(ps.subs[g]);
    cudaFree(ps.edges);
  }
  ps = PlanSet();
}

}  // namespace nld

