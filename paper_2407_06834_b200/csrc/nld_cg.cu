// Device-resident deflated / plain PCG around the fused system matvec,
// plus the small vector kernels behind DeflatingBasis and the generic pcg.
//
// Reference: pcg (linops.py:193-244), _projected_prec (:252-260),
// deflated_solve (:263-300), plain_solve (:303-319), scs_up/scs_down
// (:114-131), DeflatingBasis (:134-176).
//
// deflated_solve runs CG on the tail block of U^T A U, U the orthogonal basis
// whose first column is 1/sqrt(n).  With x = U[0; y] this is CG in pixel space
// on the complement of 1 with the operator Pi A Pi, the preconditioner
// z = Pi(D^-1 r) and the right-hand side Pi(lam f), Pi = I - 11^T/n, and
// u = mean(f) 1 + x.  U is orthogonal, so every inner product, norm,
// step length and stopping decision is the same quantity as in the reference
// (hard part 4).  The projections need one mean per product
// instead of the two O(n) prefix scans per product of the literal form.
//
// Reductions are two-stage with a fixed block count and a fixed summation
// order, so results are run-to-run deterministic.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "nld_internal.cuh"

namespace nld {

namespace {

constexpr int kRB = 148 * 8;   // reduction blocks (8 per SM: enough loads in flight)
constexpr int kRT = 256;
constexpr int kMaxK = 4;

struct RhsScal {
  double alpha, mq, mz, beta, lam, mu, mf;
  int active;
  int sel;     // column selection: 1 = x into the mixed product input, 2 = copy t -> q
};

enum RedMode { RED_SUM = 0, RED_PQ = 1, RED_UPDATE = 2, RED_PREC = 3, RED_RESID = 4,
               RED_NORM2 = 5 };

struct CgPtr {
  double* x;
  double* r;
  double* p;
  double* q;
  double* b;
  double* t;
  const double* f;
  const double* eta;
  const double* eta2;
  int64_t N;
  int64_t ldf;
  int nrhs;
  int L;
  int prec;
  int deflate;
  unsigned long long* pmax;   // per-rhs max |p| bit pattern (direction update), or null
  double* pflag;              // per-rhs non-finite flag of p
};

__device__ __forceinline__ double dinv_at(const CgPtr& c, const RhsScal& s, int64_t i) {
  // correctly rounded reciprocal without the division's slow path
  if (c.prec == NLD_PREC_JACOBI) return __drcp_rn(s.lam + s.mu * c.eta[i]);
  if (c.prec == NLD_PREC_L2) {
    const double pa = s.lam + s.mu * c.eta[i];
    const double row_sq = c.eta2[i] / (double)(c.L * c.L);
    return 1.0 / sqrt(s.mu * s.mu * row_sq + pa * pa);
  }
  return 1.0;
}

template <int K>
__device__ __forceinline__ void block_store(double (&v)[K], double* part) {
  __shared__ double sh[K][kRT];
#pragma unroll
  for (int k = 0; k < K; ++k) sh[k][threadIdx.x] = v[k];
  __syncthreads();
  for (int off = kRT / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
#pragma unroll
      for (int k = 0; k < K; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) part[k] = sh[k][0];
}

// Vectors are pixel-major [N][nrhs] (element (i, r) at i * nrhs + r), the
// kernels' native layout.  A reduction block holds kRT / nrhs pixel groups
// of nrhs threads; thread r of every group accumulates rhs r, and the groups
// are summed in a fixed order (deterministic).
template <int MODE>
__global__ void __launch_bounds__(kRT)
k_cg_reduce(CgPtr c, const RhsScal* __restrict__ sc, const double* __restrict__ vecA,
            double* __restrict__ part) {
  const int nr = c.nrhs;
  const int grp = kRT / nr;
  const int tid = threadIdx.x;
  const bool live = tid < grp * nr;
  const int r = live ? tid % nr : 0;
  const int g = tid / nr;
  const RhsScal s = sc[r];
  double acc[kMaxK] = {0.0, 0.0, 0.0, 0.0};
  // one element (pixel i, rhs r) per step, four steps' loads issued together
  // (memory-level parallelism); the accumulation order is the plain
  // sequential one, so the result does not depend on the unrolling
  auto body = [&](int64_t i, double va, double vr, double vp, double vq, double vb, double vt) {
    const int64_t e = i * nr + r;
    if (MODE == RED_SUM) {
      acc[0] += va;
    } else if (MODE == RED_NORM2) {
      acc[0] += va * va;
    } else if (MODE == RED_PQ) {
      acc[0] += vq;
      acc[1] += vp * vq;
      acc[2] += vp;
    } else if (MODE == RED_UPDATE || MODE == RED_PREC) {
      // (vb, vt) carry x and eta here: every load of the step is issued up front
      double rr = vr;
      if (MODE == RED_UPDATE && s.active) {
        c.x[e] = vb + s.alpha * vp;
        rr -= s.alpha * (vq - s.mq);
        c.r[e] = rr;
      }
      const double di = c.prec == NLD_PREC_JACOBI ? __drcp_rn(s.lam + s.mu * vt)
                                                  : dinv_at(c, s, i);
      const double zt = di * rr;
      acc[0] += rr * rr;
      acc[1] += zt;
      acc[2] += rr * zt;
      acc[3] += rr;
    } else if (MODE == RED_RESID) {
      const double d = vb - (vt - s.mq);
      acc[0] += d * d;
    }
  };
  auto load = [&](int64_t i, double& va, double& vr, double& vp, double& vq, double& vb,
                  double& vt) {
    const int64_t e = i * nr + r;
    if (MODE == RED_SUM || MODE == RED_NORM2) va = vecA[e];
    if (MODE == RED_PQ || MODE == RED_UPDATE) { vp = c.p[e]; vq = c.q[e]; }
    if (MODE == RED_UPDATE || MODE == RED_PREC) {
      vr = c.r[e];
      if (MODE == RED_UPDATE && s.active) vb = c.x[e];
      if (c.prec == NLD_PREC_JACOBI) vt = c.eta[i];
    }
    if (MODE == RED_RESID) { vb = c.b[e]; vt = c.t[e]; }
  };
  if (live) {
    const int64_t stride = (int64_t)gridDim.x * grp;
    int64_t i = blockIdx.x * (int64_t)grp + g;
    for (; i + 3 * stride < c.N; i += 4 * stride) {
      double va[4] = {}, vr[4] = {}, vp[4] = {}, vq[4] = {}, vb[4] = {}, vt[4] = {};
#pragma unroll
      for (int u = 0; u < 4; ++u) load(i + u * stride, va[u], vr[u], vp[u], vq[u], vb[u], vt[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) body(i + u * stride, va[u], vr[u], vp[u], vq[u], vb[u], vt[u]);
    }
    for (; i < c.N; i += stride) {
      double va = 0, vr = 0, vp = 0, vq = 0, vb = 0, vt = 0;
      load(i, va, vr, vp, vq, vb, vt);
      body(i, va, vr, vp, vq, vb, vt);
    }
  }
  __shared__ double sh[kMaxK][kRT];
#pragma unroll
  for (int k = 0; k < kMaxK; ++k) sh[k][tid] = acc[k];
  __syncthreads();
  if (tid < nr) {
#pragma unroll
    for (int k = 0; k < kMaxK; ++k) {
      double t = 0.0;
      for (int j = 0; j < grp; ++j) t += sh[k][j * nr + tid];
      part[((int64_t)tid * gridDim.x + blockIdx.x) * kMaxK + k] = t;
    }
  }
}

__global__ void k_final(const double* __restrict__ part, int nblk, double* __restrict__ out) {
  // one warp per (rhs, k): lane l sums blocks l, l + 32, ... in order, then a
  // fixed shuffle tree -- deterministic, and 32 loads in flight instead of a
  // chain of nblk dependent ones
  const int rhs = blockIdx.x;
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (k >= kMaxK) return;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += part[((int64_t)rhs * nblk + b) * kMaxK + k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) out[rhs * kMaxK + k] = s;
}

// elementwise kernels over the N * nrhs pixel-major elements
__global__ void k_cg_setup(CgPtr c, const RhsScal* __restrict__ sc, int warm) {
  const int64_t total = c.N * c.nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const RhsScal s = sc[e % c.nrhs];
    const double f = c.t[e];                 // f, pixel-major copy
    const double g = c.deflate ? f - s.mf : f;
    c.b[e] = s.lam * g;
    c.x[e] = warm ? g : 0.0;
  }
}

__global__ void k_cg_resid0(CgPtr c, const RhsScal* __restrict__ sc, int warm) {
  // r = b - Pi A x0 (warm) or r = b (x0 = 0; A 0 == 0 exactly)
  const int64_t total = c.N * c.nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    c.r[e] = warm ? c.b[e] - (c.q[e] - sc[e % c.nrhs].mq) : c.b[e];
}

__global__ void __launch_bounds__(256) k_cg_direction(CgPtr c, const RhsScal* __restrict__ sc,
                                                      int first) {
  // z = Pi(D^-1 r) (or r), p = z + beta p.  Thread layout as in k_cg_reduce:
  // a fixed rhs per thread (its scalars in registers), pixels strided, four
  // pixels' loads in flight per step.  With c.pmax the kernel also takes the
  // per-rhs max |p| (bit patterns: NaN > Inf > finite, as k_vmax) of the
  // whole new p -- inactive rhs keep their p and only read it -- so the next
  // product skips its own pass over p.
  const int nr = c.nrhs;
  const int grp = blockDim.x / nr;
  const bool live = (int)threadIdx.x < grp * nr;
  const int r = live ? threadIdx.x % nr : 0, g = threadIdx.x / nr;
  const RhsScal s = sc[r];
  const bool act = live && s.active;
  const bool want_max = c.pmax != nullptr;
  unsigned long long mx = 0ull;
  if (act || (live && want_max)) {
    const int64_t stride = (int64_t)gridDim.x * grp;
    const bool jac = c.prec == NLD_PREC_JACOBI;
    auto one = [&](int64_t i, double rv, double pv, double ev) {
      double pn = pv;
      if (act) {
        const double di = jac ? __drcp_rn(s.lam + s.mu * ev) : dinv_at(c, s, i);
        const double z = (c.prec == NLD_PREC_NONE) ? rv : di * rv - s.mz;
        pn = first ? z : z + s.beta * pv;
        c.p[i * nr + r] = pn;
      }
      mx = max(mx, (unsigned long long)__double_as_longlong(pn) & 0x7fffffffffffffffull);
    };
    const bool rd_p = !act || !first;
    int64_t i = blockIdx.x * (int64_t)grp + g;
    for (; i + 3 * stride < c.N; i += 4 * stride) {
      double rv[4], pv[4], ev[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = (i + u * stride) * nr + r;
        rv[u] = act ? c.r[e] : 0.0;
        pv[u] = rd_p ? c.p[e] : 0.0;
        ev[u] = (act && jac) ? c.eta[i + u * stride] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) one(i + u * stride, rv[u], pv[u], ev[u]);
    }
    for (; i < c.N; i += stride) {
      const int64_t e = i * nr + r;
      one(i, act ? c.r[e] : 0.0, rd_p ? c.p[e] : 0.0, (act && jac) ? c.eta[i] : 0.0);
    }
  }
  if (!want_max) return;
  __shared__ unsigned long long shm[256];
  shm[threadIdx.x] = mx;
  __syncthreads();
  if ((int)threadIdx.x < nr) {
    unsigned long long m = 0ull;
    for (int j = 0; j < grp; ++j) m = max(m, shm[j * nr + threadIdx.x]);
    if (m) atomicMax(&c.pmax[threadIdx.x], m);
    if (m >= 0x7ff0000000000000ull) c.pflag[threadIdx.x] = 1.0;
  }
}

// column selection between the CG vectors (pixel-major): mode 0 builds the
// product input t = x for rhs awaiting their true-residual check (sel == 1)
// and p otherwise; mode 1 copies t -> q for the rhs flagged sel == 2
__global__ void k_cg_colsel(CgPtr c, const RhsScal* __restrict__ sc, int mode) {
  const int nr = c.nrhs;
  const int grp = blockDim.x / nr;
  if ((int)threadIdx.x >= grp * nr) return;
  const int r = threadIdx.x % nr, g = threadIdx.x / nr;
  const int sel = sc[r].sel;
  if (mode == 1 && sel != 2) return;
  for (int64_t i = blockIdx.x * (int64_t)grp + g; i < c.N; i += (int64_t)gridDim.x * grp) {
    const int64_t e = i * nr + r;
    if (mode == 0) c.t[e] = sel == 1 ? c.x[e] : c.p[e];
    else c.q[e] = c.t[e];
  }
}

__global__ void k_cg_finish(CgPtr c, const RhsScal* __restrict__ sc) {
  // x += mean(f) (deflation), in place before the transpose out
  const int64_t total = c.N * c.nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    if (c.deflate) c.x[e] += sc[e % c.nrhs].mf;
}

int eblocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 8));
}

struct Reducer {
  nld_operator* op = nullptr;
  double* part = nullptr;
  double* out = nullptr;
  std::vector<double> host;
  int nrhs;
  int nblk;
  cudaStream_t st;
  Reducer(nld_operator* o, int nr, int64_t N, cudaStream_t s) : op(o), nrhs(nr), st(s) {
    const int64_t grp = std::max(1, kRT / nr);
    nblk = (int)std::max<int64_t>(1, std::min<int64_t>(kRB, (N + grp - 1) / grp));
    NLD_CUDA(cudaMallocAsync(&part, sizeof(double) * nr * nblk * kMaxK, st));
    NLD_CUDA(cudaMallocAsync(&out, sizeof(double) * nr * kMaxK, st));
    host.resize((size_t)nr * kMaxK);
  }
  ~Reducer() {
    cudaFreeAsync(part, st);
    cudaFreeAsync(out, st);
  }
  template <int MODE>
  const std::vector<double>& run(const CgPtr& c, const RhsScal* sc,
                                 const double* vecA = nullptr) {
    k_cg_reduce<MODE><<<nblk, kRT, 0, st>>>(c, sc, vecA, part);
    NLD_CUDA(cudaGetLastError());
    k_final<<<nrhs, 32 * kMaxK, 0, st>>>(part, nblk, out);
    // sharded: the per-rank partial scalars are summed on the device, on the
    // stream (NCCL), before the one host read the solver's decisions need
    comm_device(op, out, (int64_t)nrhs * kMaxK, st);
    NLD_CUDA(cudaMemcpyAsync(host.data(), out, sizeof(double) * nrhs * kMaxK,
                             cudaMemcpyDeviceToHost, st));
    NLD_CUDA(cudaStreamSynchronize(st));
    return host;
  }
};

// ---- generic vector kernels ---------------------------------------------

__global__ void k_axpby(double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

__global__ void k_dot_part(const double* __restrict__ x, const double* __restrict__ y,
                           int64_t n, double* __restrict__ part) {
  double acc[kMaxK] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)kRT + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kRT)
    acc[0] += x[i] * y[i];
  block_store<kMaxK>(acc, part + blockIdx.x * kMaxK);
}

__global__ void k_reverse(const double* __restrict__ x, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[n - 1 - i];
}

// scs_up: out_i = x_0 + sum_{j>i} x_j; rev = inclusive scan of reversed x
__global__ void k_scs_up(const double* __restrict__ x, const double* __restrict__ rev,
                         double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // suffix sum from i+1 = rev[n-2-i]
    out[i] = (i < n - 1) ? x[0] + rev[n - 2 - i] : x[0];
  }
}

// scs_down: out_0 = total, out_i = cumsum_{i-1}
__global__ void k_scs_down(const double* __restrict__ cs, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (i == 0) ? cs[n - 1] : cs[i - 1];
}

__global__ void k_sq(const double* __restrict__ v, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v[i] * v[i];
}

__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

// U x pieces: pre = sqrt(cumsum v^2); y0 = x0/norm, y_i = b_i v_i x_i
__global__ void k_basis_y(const double* __restrict__ v, const double* __restrict__ pre2,
                          const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  const double norm = sqrt(pre2[n - 1]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == 0) {
      y[0] = x[0] / norm;
    } else {
      const double pm = sqrt(pre2[i - 1]), pi = sqrt(pre2[i]);
      const double b = 1.0 / (pm * pi);
      y[i] = b * v[i] * x[i];
    }
  }
}

__global__ void k_basis_out(const double* __restrict__ v, const double* __restrict__ pre2,
                            const double* __restrict__ x, const double* __restrict__ s,
                            double* __restrict__ out, int64_t n, int adjoint) {
  const double norm = sqrt(pre2[n - 1]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!adjoint) {
      // out = v * scs_up(y); out[1:] -= a * x[1:]
      double o = v[i] * s[i];
      if (i > 0) {
        const double a = sqrt(pre2[i - 1]) / sqrt(pre2[i]);
        o -= a * x[i];
      }
      out[i] = o;
    } else {
      // out0 = s0 / norm; out_i = b v_i s_i - a x_i
      if (i == 0) {
        out[0] = s[0] / norm;
      } else {
        const double pm = sqrt(pre2[i - 1]), pi = sqrt(pre2[i]);
        const double a = pm / pi;
        const double b = 1.0 / (pm * pi);
        out[i] = b * v[i] * s[i] - a * x[i];
      }
    }
  }
}

void inclusive_scan(const double* in, double* out, int64_t n, cudaStream_t st) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, (int)n, st);
  void* tmp = nullptr;
  NLD_CUDA(cudaMallocAsync(&tmp, bytes ? bytes : 1, st));
  NLD_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, (int)n, st));
  cudaFreeAsync(tmp, st);
}

}  // namespace

void dev_axpby(double a, const double* x, double b, const double* y, double* out, int64_t n,
               cudaStream_t st) {
  k_axpby<<<eblocks(n), 256, 0, st>>>(a, x, b, y, out, n);
  NLD_CUDA(cudaGetLastError());
}

double dev_dot(const double* x, const double* y, int64_t n, cudaStream_t st) {
  int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(kRB, (n + kRT - 1) / kRT));
  double *part = nullptr, *out = nullptr;
  NLD_CUDA(cudaMallocAsync(&part, sizeof(double) * nblk * kMaxK, st));
  NLD_CUDA(cudaMallocAsync(&out, sizeof(double) * kMaxK, st));
  k_dot_part<<<nblk, kRT, 0, st>>>(x, y, n, part);
  k_final<<<1, 32 * kMaxK, 0, st>>>(part, nblk, out);
  double h[kMaxK];
  NLD_CUDA(cudaMemcpyAsync(h, out, sizeof(double) * kMaxK, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(part, st);
  cudaFreeAsync(out, st);
  NLD_CUDA(cudaStreamSynchronize(st));
  return h[0];
}

void dev_scs(const double* x, double* out, int64_t n, int down, cudaStream_t st) {
  double* tmp = nullptr;
  double* tmp2 = nullptr;
  NLD_CUDA(cudaMallocAsync(&tmp, sizeof(double) * n, st));
  if (down) {
    inclusive_scan(x, tmp, n, st);
    k_scs_down<<<eblocks(n), 256, 0, st>>>(tmp, out, n);
  } else {
    NLD_CUDA(cudaMallocAsync(&tmp2, sizeof(double) * n, st));
    k_reverse<<<eblocks(n), 256, 0, st>>>(x, tmp2, n);
    inclusive_scan(tmp2, tmp, n, st);
    k_scs_up<<<eblocks(n), 256, 0, st>>>(x, tmp, out, n);
    cudaFreeAsync(tmp2, st);
  }
  NLD_CUDA(cudaGetLastError());
  cudaFreeAsync(tmp, st);
}

void dev_basis(const double* v, const double* x, double* out, int64_t n, int adjoint,
               cudaStream_t st) {
  double *sq = nullptr, *pre2 = nullptr, *y = nullptr, *s = nullptr;
  NLD_CUDA(cudaMallocAsync(&sq, sizeof(double) * n, st));
  NLD_CUDA(cudaMallocAsync(&pre2, sizeof(double) * n, st));
  NLD_CUDA(cudaMallocAsync(&y, sizeof(double) * n, st));
  NLD_CUDA(cudaMallocAsync(&s, sizeof(double) * n, st));
  k_sq<<<eblocks(n), 256, 0, st>>>(v, sq, n);
  inclusive_scan(sq, pre2, n, st);
  if (!adjoint) {
    k_basis_y<<<eblocks(n), 256, 0, st>>>(v, pre2, x, y, n);
    dev_scs(y, s, n, 0, st);
  } else {
    k_mul<<<eblocks(n), 256, 0, st>>>(v, x, y, n);
    dev_scs(y, s, n, 1, st);
  }
  k_basis_out<<<eblocks(n), 256, 0, st>>>(v, pre2, x, s, out, n, adjoint);
  NLD_CUDA(cudaGetLastError());
  cudaFreeAsync(sq, st);
  cudaFreeAsync(pre2, st);
  cudaFreeAsync(y, st);
  cudaFreeAsync(s, st);
}

struct Scratch {
  cudaStream_t st;
  std::vector<void*> p;
  ~Scratch() {
    for (void* q : p) cudaFreeAsync(q, st);
  }
  template <class T>
  T* alloc(size_t count) {
    void* q = nullptr;
    NLD_CUDA(cudaMallocAsync(&q, sizeof(T) * std::max<size_t>(count, 1), st));
    p.push_back(q);
    return static_cast<T*>(q);
  }
};

void cg_solve(nld_operator* op, const double* f, double* u, int nrhs, int64_t ld,
              const double* lam, const double* mu, int prec, int deflate, double tol,
              int maxit, int warm, int* iters, double* relres, int* conv, double* hist,
              int hist_cap, cudaStream_t st) {
  const int64_t N = op->N;
  if (nrhs > kRT) throw Error(NLD_ERR_VALUE, "at most 256 right-hand sides per solve");
  if (deflate && op->N_global < 2)
    throw Error(NLD_ERR_DIMENSION, "basis needs at least two entries");
  for (int r = 0; r < nrhs; ++r)
    if (!(lam[r] > 0) || !(mu[r] > 0))
      throw Error(NLD_ERR_VALUE, "shift lambda and weight mu must be positive");
  // degree vectors (ShiftedSystem.__init__ caches eta, linops.py:37)
  auto degree = [&](int which) -> const double* {
    if (!op->eta[which]) {
      NLD_CUDA(cudaMalloc(&op->eta[which], sizeof(double) * N));
      double* ones = nullptr;
      NLD_CUDA(cudaMallocAsync(&ones, sizeof(double) * N, st));
      std::vector<double> h(N, 1.0);
      NLD_CUDA(cudaMemcpyAsync(ones, h.data(), sizeof(double) * N, cudaMemcpyHostToDevice, st));
      if (op->params.mode == 1) dense_apply(op, which, NLD_APPLY_GAMMA, ones, op->eta[which], 1, N, nullptr, nullptr, st);
      else apply_op(op, which, NLD_APPLY_GAMMA, ones, op->eta[which], 1, N, nullptr, nullptr, st);
      NLD_CUDA(cudaStreamSynchronize(st));
      cudaFreeAsync(ones, st);
    }
    return op->eta[which];
  };
  if (op->params.mode != 1 && !op->built[0]) {
    build_planset(op, 0, st);
    op->built[0] = true;
  }
  const double* eta = degree(0);
  // stream-ordered scratch, released on every exit (including the throws
  // below: breakdown, communicator failure)
  Scratch scratch{st, {}};
  double* eta2 = nullptr;
  if (prec == NLD_PREC_L2) {
    if (op->params.mode != 1 && !op->built[1]) {
      build_planset(op, 1, st);
      op->built[1] = true;
    }
    degree(1);
    // degree_squared = apply_squared(1) * L (kernel.py:148-154)
    eta2 = scratch.alloc<double>(N);
    dev_axpby((double)op->L, op->eta[1], 0.0, op->eta[1], eta2, N, st);
  }

  const int64_t V = N * nrhs;
  // persistent per-operator CG vectors (a solve per image/alpha batch reuses them)
  if (op->ws.cg_cap < V) {
    NLD_CUDA(cudaStreamSynchronize(st));
    cudaFree(op->ws.cg);
    op->ws.cg = nullptr;
    NLD_CUDA(cudaMalloc(&op->ws.cg, sizeof(double) * 6 * V));
    op->ws.cg_cap = V;
  }
  CgPtr c{};
  c.x = op->ws.cg;
  c.r = c.x + op->ws.cg_cap;
  c.p = c.r + op->ws.cg_cap;
  c.q = c.p + op->ws.cg_cap;
  c.b = c.q + op->ws.cg_cap;
  c.t = c.b + op->ws.cg_cap;
  c.f = f;
  c.nrhs = nrhs;
  c.eta = eta;
  c.eta2 = eta2;
  c.N = N;
  c.ldf = ld;
  c.L = op->L;
  c.prec = prec;
  c.deflate = deflate;
  RhsScal* scd = scratch.alloc<RhsScal>(nrhs);
  double* coef = scratch.alloc<double>(2 * nrhs);
  std::vector<RhsScal> sc(nrhs);
  std::vector<double> hcoef(2 * nrhs);
  for (int r = 0; r < nrhs; ++r) {
    sc[r] = RhsScal{0, 0, 0, 0, lam[r], mu[r], 0, 1, 0};
    hcoef[2 * r] = lam[r];
    hcoef[2 * r + 1] = mu[r];
  }
  NLD_CUDA(cudaMemcpyAsync(coef, hcoef.data(), sizeof(double) * 2 * nrhs,
                           cudaMemcpyHostToDevice, st));
  auto push = [&]() {
    NLD_CUDA(cudaMemcpyAsync(scd, sc.data(), sizeof(RhsScal) * nrhs, cudaMemcpyHostToDevice,
                             st));
  };
  // per-rhs max |p| and non-finite flags, taken by the direction update for
  // the next product (which then skips its own pass over p)
  if (nrhs % 16 == 0 && op->params.mode != 1 && op->params.cutoff == 4) {
    c.pmax = scratch.alloc<unsigned long long>(nrhs);
    c.pflag = scratch.alloc<double>(nrhs);
  }
  auto matvec = [&](const double* in, double* out, bool p_max = false) {   // pixel-major in/out
    if (op->params.mode == 1)
      dense_apply(op, 0, NLD_APPLY_SYSTEM, in, out, nrhs, N, coef, eta, st, 1);
    else if (p_max && c.pmax)
      apply_op(op, 0, NLD_APPLY_SYSTEM, in, out, nrhs, N, coef, eta, st, 1, c.pmax, c.pflag);
    else
      apply_op(op, 0, NLD_APPLY_SYSTEM, in, out, nrhs, N, coef, eta, st, 1);
  };
  const double dN = (double)op->N_global;
  Reducer red(op, nrhs, N, st);
  const int eg = eblocks(N * nrhs);
  auto direction = [&](int first) {
    if (c.pmax) {
      NLD_CUDA(cudaMemsetAsync(c.pmax, 0, sizeof(unsigned long long) * nrhs, st));
      NLD_CUDA(cudaMemsetAsync(c.pflag, 0, sizeof(double) * nrhs, st));
    }
    k_cg_direction<<<eg, 256, 0, st>>>(c, scd, first);
    NLD_CUDA(cudaGetLastError());
  };

  std::vector<std::vector<double>> H(nrhs);
  std::vector<double> bnorm(nrhs, 0.0), rz(nrhs, 0.0);
  std::vector<int> it(nrhs, 0), done(nrhs, 0);
  for (int r = 0; r < nrhs; ++r) {
    iters[r] = 0;
    relres[r] = 0.0;
    conv[r] = 0;
  }

  // mean of f (deflation: x_first = g0 carries the mean, linops.py:278-279)
  // f -> pixel-major (in the t vector, free until the first true residual)
  to_pixel_major(f, ld, N, nrhs, c.t, st);
  push();
  {
    const auto& h = red.run<RED_SUM>(c, scd, c.t);
    for (int r = 0; r < nrhs; ++r) sc[r].mf = deflate ? h[r * kMaxK] / dN : 0.0;
  }
  push();
  k_cg_setup<<<eg, 256, 0, st>>>(c, scd, warm);
  if (warm) {
    matvec(c.x, c.q);
    if (deflate) {
      const auto& h = red.run<RED_SUM>(c, scd, c.q);
      for (int r = 0; r < nrhs; ++r) sc[r].mq = h[r * kMaxK] / dN;
    }
    push();
  }
  k_cg_resid0<<<eg, 256, 0, st>>>(c, scd, warm);
  NLD_CUDA(cudaGetLastError());
  std::vector<double> nb(nrhs), nr(nrhs);
  {
    const auto& h = red.run<RED_NORM2>(c, scd, c.b);
    for (int r = 0; r < nrhs; ++r) nb[r] = std::sqrt(h[r * kMaxK]);
  }
  {
    const auto& h = red.run<RED_PREC>(c, scd);
    for (int r = 0; r < nrhs; ++r) {
      nr[r] = std::sqrt(h[r * kMaxK]);
      if (nb[r] == 0.0 && !warm) {
        done[r] = 1;
        conv[r] = 1;
        H[r] = {0.0};
        continue;
      }
      bnorm[r] = std::max(nb[r], nr[r]);
      if (bnorm[r] == 0.0) {
        done[r] = 1;
        conv[r] = 1;
        H[r] = {0.0};
        continue;
      }
      H[r] = {nr[r] / bnorm[r]};
      if (maxit <= 0) {
        done[r] = 1;
        conv[r] = 0;
        relres[r] = H[r][0];
        continue;
      }
      const double mz = (deflate && prec != NLD_PREC_NONE) ? h[r * kMaxK + 1] / dN : 0.0;
      sc[r].mz = mz;
      rz[r] = h[r * kMaxK + 2] - mz * h[r * kMaxK + 3];
      sc[r].beta = 0.0;
    }
  }
  for (int r = 0; r < nrhs; ++r) sc[r].active = done[r] ? 0 : 1;
  push();
  direction(1);

  auto any_active = [&]() {
    for (int r = 0; r < nrhs; ++r)
      if (!done[r]) return true;
    return false;
  };
  // explicit residual || b - Pi A x || for the flagged rhs
  auto true_residual = [&](std::vector<double>& out) {
    matvec(c.x, c.t);
    if (deflate) {
      const auto& h = red.run<RED_SUM>(c, scd, c.t);
      for (int r = 0; r < nrhs; ++r) sc[r].mq = h[r * kMaxK] / dN;
    } else {
      for (int r = 0; r < nrhs; ++r) sc[r].mq = 0.0;
    }
    push();
    const auto& h = red.run<RED_RESID>(c, scd);
    out.resize(nrhs);
    for (int r = 0; r < nrhs; ++r) out[r] = std::sqrt(h[r * kMaxK]) / (bnorm[r] > 0 ? bnorm[r] : 1.0);
  };

  std::vector<double> truer;
  // The reference confirms a converged-looking iterate with an explicit
  // residual b - A x (one extra product, linops.py:218-231).  Here that
  // product rides in the NEXT iteration's batch: the columns of rhs awaiting
  // the check carry x instead of p (columns are independent products), so the
  // check costs no product of its own.  Only when the check fails (the rhs
  // must continue) is its deferred direction formed and an extra product run.
  // Iterates, stopping decisions and histories are the reference's.
  std::vector<int> pending(nrhs, 0);
  std::vector<double> save_rzn(nrhs, 0.0), save_mz(nrhs, 0.0);
  auto any_pending = [&]() {
    for (int r = 0; r < nrhs; ++r)
      if (pending[r]) return true;
    return false;
  };
  while (any_active() ) {
    const bool pend = any_pending();
    if (pend) {
      for (int r = 0; r < nrhs; ++r) sc[r].sel = pending[r] ? 1 : 0;
      push();
      k_cg_colsel<<<kRB, kRT, 0, st>>>(c, scd, 0);
      NLD_CUDA(cudaGetLastError());
      matvec(c.t, c.q);
    } else {
      matvec(c.p, c.q, true);
    }
    auto hpq = red.run<RED_PQ>(c, scd);
    if (pend) {
      // true residuals of the pending rhs: q holds A x in their columns
      for (int r = 0; r < nrhs; ++r)
        if (pending[r]) sc[r].mq = deflate ? hpq[r * kMaxK] / dN : 0.0;
      push();
      CgPtr c2 = c;
      c2.t = c.q;
      const auto& hres = red.run<RED_RESID>(c2, scd);
      std::vector<int> failed;
      for (int r = 0; r < nrhs; ++r) {
        if (!pending[r]) continue;
        const double tr = std::sqrt(hres[r * kMaxK]) / (bnorm[r] > 0 ? bnorm[r] : 1.0);
        H[r].back() = tr;
        pending[r] = 0;
        if (tr <= tol) {
          done[r] = 1;
          conv[r] = 1;
          relres[r] = tr;
          sc[r].active = 0;
        } else if (it[r] >= maxit) {
          done[r] = 1;
          conv[r] = 0;
          relres[r] = tr;
          sc[r].active = 0;
        } else {
          failed.push_back(r);
        }
      }
      if (!failed.empty()) {
        // deferred direction of the rhs that must continue, then their A p
        std::vector<int> keep(nrhs);
        for (int r = 0; r < nrhs; ++r) {
          keep[r] = sc[r].active;
          sc[r].active = 0;
          sc[r].sel = 0;
        }
        for (int r : failed) {
          sc[r].mz = save_mz[r];
          sc[r].beta = save_rzn[r] / rz[r];
          rz[r] = save_rzn[r];
          sc[r].active = 1;
          sc[r].sel = 2;
        }
        push();
        direction(0);
        matvec(c.p, c.t, true);
        k_cg_colsel<<<kRB, kRT, 0, st>>>(c, scd, 1);
        NLD_CUDA(cudaGetLastError());
        for (int r = 0; r < nrhs; ++r) sc[r].active = keep[r];
        for (int r : failed) sc[r].active = 1;
        push();
        hpq = red.run<RED_PQ>(c, scd);
      }
      if (!any_active()) break;
    }
    for (int r = 0; r < nrhs; ++r) {
      if (done[r]) continue;
      const double mq = deflate ? hpq[r * kMaxK] / dN : 0.0;
      const double pap = hpq[r * kMaxK + 1] - mq * hpq[r * kMaxK + 2];
      if (!std::isfinite(pap) || pap <= 0.0)
        throw Error(NLD_ERR_BREAKDOWN, "indefinite or non-finite curvature at iteration " +
                                           std::to_string(it[r]));
      sc[r].mq = mq;
      sc[r].alpha = rz[r] / pap;
      sc[r].active = 1;
    }
    push();
    const auto& hu = red.run<RED_UPDATE>(c, scd);
    std::vector<double> hsave(hu.begin(), hu.end());
    std::vector<int> hit_max(nrhs, 0);
    for (int r = 0; r < nrhs; ++r) {
      if (done[r]) {
        sc[r].active = 0;
        continue;
      }
      it[r] += 1;
      const double rel = std::sqrt(hsave[r * kMaxK]) / bnorm[r];
      H[r].push_back(rel);
      const double mz = (deflate && prec != NLD_PREC_NONE) ? hsave[r * kMaxK + 1] / dN : 0.0;
      const double rzn = hsave[r * kMaxK + 2] - mz * hsave[r * kMaxK + 3];
      if (rel <= tol) {
        // check in the next product; the direction waits for its outcome
        pending[r] = 1;
        save_rzn[r] = rzn;
        save_mz[r] = mz;
        sc[r].active = 0;
        continue;
      }
      if (!std::isfinite(rzn))
        throw Error(NLD_ERR_BREAKDOWN, "non-finite residual inner product");
      sc[r].mz = mz;
      sc[r].beta = rzn / rz[r];
      rz[r] = rzn;
      sc[r].active = 1;
      if (it[r] >= maxit) hit_max[r] = 1;
    }
    push();
    direction(0);
    bool any_max = false;
    for (int r = 0; r < nrhs; ++r) any_max |= hit_max[r] != 0;
    if (any_max) {
      // (pending rhs are resolved by the next loop's product; resolve them
      // here too so this explicit residual serves both)
      true_residual(truer);
      for (int r = 0; r < nrhs; ++r) {
        if (pending[r]) {
          H[r].back() = truer[r];
          pending[r] = 0;
          if (truer[r] <= tol || it[r] >= maxit) {
            done[r] = 1;
            conv[r] = truer[r] <= tol;
            relres[r] = truer[r];
            sc[r].active = 0;
          } else {
            // must continue: its deferred direction
            sc[r].mz = save_mz[r];
            sc[r].beta = save_rzn[r] / rz[r];
            rz[r] = save_rzn[r];
            sc[r].active = 1;
            sc[r].sel = 3;   // marker only
          }
        }
        if (!hit_max[r]) continue;
        done[r] = 1;
        relres[r] = truer[r];
        conv[r] = truer[r] <= tol;
        sc[r].active = 0;
      }
      // directions of rhs released from pending above
      bool rel_dir = false;
      std::vector<int> keep(nrhs);
      for (int r = 0; r < nrhs; ++r) {
        keep[r] = sc[r].active;
        if (sc[r].sel == 3) rel_dir = true;
      }
      if (rel_dir) {
        for (int r = 0; r < nrhs; ++r) sc[r].active = (sc[r].sel == 3) ? 1 : 0;
        push();
        direction(0);
        for (int r = 0; r < nrhs; ++r) {
          sc[r].active = keep[r];
          sc[r].sel = 0;
        }
      }
      push();
    }
    // rhs waiting for their check stay "active" for the loop condition
    bool waiting = false;
    for (int r = 0; r < nrhs; ++r) waiting |= pending[r] != 0;
    if (!any_active() && !waiting) break;
  }
  k_cg_finish<<<eg, 256, 0, st>>>(c, scd);
  to_rhs_major(c.x, N, nrhs, u, ld, st);
  NLD_CUDA(cudaGetLastError());
  NLD_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < nrhs; ++r) {
    iters[r] = it[r];
    if (hist && hist_cap > 0) {
      for (int k = 0; k < hist_cap; ++k)
        hist[(int64_t)r * hist_cap + k] =
            k < (int)H[r].size() ? H[r][k] : std::numeric_limits<double>::quiet_NaN();
    }
  }
}

}  // namespace nld
