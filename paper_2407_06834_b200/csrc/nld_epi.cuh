// Fused gather epilogue shared by the DMMA (nld_mma.cuh) and integer-sliced
// (nld_ozaki.cu) gathers.
#pragma once

#include "nld_internal.cuh"

namespace nld {
namespace mma {

// ---- fused gather epilogue ------------------------------------------------
// The window sum and the degree / shift terms fused into the gather (the
// separate epilogue pass re-read L window outputs + v from HBM).  The output
// buffer itself accumulates the windows, pixel-major [N][nrhs]:
//   kGatherStore    : wout[win] = G_w v          (unfused, per-window buffers)
//   kGatherFirst    : out  = G_0 v
//   kGatherAccum    : out += G_w v
//   kGatherFinal    : out  = epi(out + G_{L-1} v)   (kind's formula)
enum GatherMode { kGatherStore = 0, kGatherFirst = 1, kGatherAccum = 2, kGatherFinal = 3 };

struct GatherEpi {
  int mode;
  int kind;
  int L;
  const double* v;      // pixel-major [N][nrhs]
  const double* eta;    // [N] (SYSTEM / LAPLACIAN)
  const double* coef;   // [nrhs][2] (lam, mu) for SYSTEM
};

// y from the window sum s (unit diagonals included) and x = v, kernel.py:118-127
// (Gamma = (sum_l G_l - L I) / L) and linops.py:43-50
__device__ __forceinline__ double epi_value(int kind, int L, double s, double x, double eta_i,
                                            double lam, double mu) {
  if (kind == NLD_APPLY_WINDOW_SUM) return s;
  const double gam = (s - (double)L * x) / (double)L;
  if (kind == NLD_APPLY_SYSTEM) return lam * x + mu * (eta_i * x - gam);
  if (kind == NLD_APPLY_LAPLACIAN) return eta_i * x - gam;
  return gam;
}

// the same with the reciprocal of L precomputed (one multiply instead of an
// fp64 division per output; differs from epi_value by at most an ulp of gam)
__device__ __forceinline__ double epi_value_r(int kind, double L, double inv_L, double s, double x,
                                              double eta_i, double lam, double mu) {
  if (kind == NLD_APPLY_WINDOW_SUM) return s;
  const double gam = (s - L * x) * inv_L;
  if (kind == NLD_APPLY_SYSTEM) return lam * x + mu * (eta_i * x - gam);
  if (kind == NLD_APPLY_LAPLACIAN) return eta_i * x - gam;
  return gam;
}

__device__ __forceinline__ void gather_put(const GatherEpi& ep, double* o, int64_t e, int64_t i,
                                           int r, double val) {
  if (ep.mode == kGatherStore || ep.mode == kGatherFirst) {
    o[e] = val;
  } else if (ep.mode == kGatherAccum) {
    o[e] += val;
  } else {
    const double s = o[e] + val;
    const double lam = ep.coef ? ep.coef[2 * r] : 0.0, mu = ep.coef ? ep.coef[2 * r + 1] : 0.0;
    const double et = (ep.kind == NLD_APPLY_SYSTEM || ep.kind == NLD_APPLY_LAPLACIAN) ? ep.eta[i] : 0.0;
    o[e] = epi_value(ep.kind, ep.L, s, ep.v[e], et, lam, mu);
  }
}

}  // namespace mma
}  // namespace nld
