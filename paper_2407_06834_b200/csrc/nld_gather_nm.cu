// Integer-sliced fp64 gather with the NODES as the MMA's M dimension
// (reference op: _kernels.gather / _gather_nb, _kernels.py:91-136, for 3-D
// windows with m = 4, 16k right-hand sides).
//
// Per node j and rhs r the gather is
//     y_{j,r} = sum_a A_j[a] T_{j,(r,a)},   T_{j,(r,a)} = sum_{(b,c)} Y_j[(b,c)] G_r[a][(b,c)]
// with Y_j = B_j (x) C_j (64 values, node specific) and G_r the 8 x 8 x 8 grid
// patch at the node's stencil cell (shared by the cell's subproblem).  The
// (b, c) contraction runs on the tensor cores as exact integer products of
// fp64 digit slices (the Ozaki scheme, nld_ozaki.cuh):
//   D[j][(r,a)] (diagonal t) += Ydig_p[j][(b,c)] * Gdig_q[(r,a)][(b,c)],  p + q = t,
// UMMA M = 128 nodes (A operand: the node's Y digits, copied to TMEM once per
// tile), N = 32 columns (r, a) per digit slice for 4 right-hand sides (B
// operand: the cell's G digits in shared memory; the slices q = 0..5-p stacked
// along N so that one UMMA per digit row p accumulates all its diagonals),
// K = 64 = (b, c).  A 128-node tile is four passes of 4 rhs; each pass
// accumulates 6 diagonals x 32 columns = 192 TMEM columns, double-buffered.
//
// Because a TMEM lane is one node, the epilogue contracts a, the remaining
// index, inside the thread: per (node, rhs) eight exact diagonal combines
// and eight FMAs with the node's A_j[a] -- no cross-lane reduction, no
// per-value shared-memory read -- and writes the node's 4 rhs of a pass as
// 32 contiguous bytes of its pixel-major line.  (The previous layout, rhs x a
// as M and nodes as N, needed a 3-stage shuffle butterfly over a per output.)
//
// Roles (one persistent CTA per SM, items = (subproblem, 16-rhs group) dealt
// in snake order of descending size):
//   warps 0-15  epilogue (lane quarter = warp & 3, rhs slot = warp >> 2)
//   warp 16     UMMA issuer (one lane)
//   warp 17     tile loader: per 128-node tile one TMA bulk copy of the Y
//               digits (48 KB) and one of the A parts + pixel indices (8.5 KB)
//               from the plan-time tile table (k_gtile)
//   warp 18     G loader: per item one TMA bulk copy of the cell's G digits
//               (48 KB + exponents, k_gdig_nm, once per product)
#include <algorithm>
#include <cstdint>
#include <vector>

#include "nld_epi.cuh"
#include "nld_internal.cuh"
#include "nld_ozaki.cuh"
#include "nld_umma.cuh"

namespace nld {
namespace oz {
namespace nm {

constexpr int kT = 128;                        // nodes per tile (UMMA M)
constexpr int kYSlice = kT * 64;               // one digit slice: 128 nodes x K = 64 bytes
constexpr int kYBytes = kSl * kYSlice;         // 48 KB
constexpr int kABytes = kT * 8 * 8;            // A_j[a], 8 doubles per node
constexpr int kPBytes = kT * 4;                // pixel index per node (-1: padding)
constexpr int kAPBytes = kABytes + kPBytes;    // 8.5 KB
constexpr int kTileBytes = kYBytes + kAPBytes; // plan-time tile record
constexpr int kPassRows = 32;                  // B rows per slice and pass: 4 rhs x 8 a
constexpr int kGBlk = kPassRows * 64;          // 2 KB
constexpr int kGBytes = 4 * kSl * kGBlk;       // 48 KB: [pass][q][32 x 64]
constexpr int kGItem = kGBytes + 16 * 4;       // + one exponent per rhs
constexpr int kAccCols = kSl * kPassRows;      // 192 accumulator columns per pass
constexpr int kYT0 = 2 * kAccCols;             // Y digits in TMEM: columns 384..479
constexpr int kEpi = 16;
constexpr int kIssuer = kEpi, kTLoader = kEpi + 1, kGLoader = kEpi + 2;
constexpr int kThreads = 32 * (kEpi + 3);
constexpr int kYStages = 2, kAPStages = 3;
static_assert(kSl == 6, "six digit slices");

__host__ __device__ constexpr int smem_bytes() {
  return 2 * kGItem + kYStages * kYBytes + kAPStages * kAPBytes;
}

// ---- plan-time tile table --------------------------------------------------
// Per 3-D subproblem, ceil(count / 128) tile records: the six Y digit slices
// (Y = B (x) C scaled by 2^(46 - max eB - max eC) of the subproblem, K-major
// canonical, 8 KB each), then A_j[0..7] (fp64) and the pixel index; rows past
// the count are zero (pixel -1).
__global__ void __launch_bounds__(kT)
k_gtile(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
        const double* __restrict__ rows, const int32_t* __restrict__ pix,
        const int16_t* __restrict__ sub_exp, const int64_t* __restrict__ tile_off,
        uint8_t* __restrict__ gtile) {
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int32_t* __restrict__ pw = pix + sd.start;
  const int16_t* ex = sub_exp + (int64_t)blockIdx.x * kExpPerSub;
  int eBm = -2000, eCm = -2000;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    eBm = max(eBm, (int)ex[8 + q]);
    eCm = max(eCm, (int)ex[16 + q]);
  }
  const double syB = pow2(46 - eBm), syC = pow2(-eCm);
  const int n = threadIdx.x;
  const int ntile = (sd.count + kT - 1) / kT;
  for (int tl = 0; tl < ntile; ++tl) {
    const int j = tl * kT + n;
    const bool ok = j < sd.count;
    uint8_t* base = gtile + (tile_off[blockIdx.x] + tl) * (int64_t)kTileBytes;
    double b[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      b[i] = ok ? rw[(int64_t)j * 24 + 8 + i] * syB : 0.0;
      c[i] = ok ? rw[(int64_t)j * 24 + 16 + i] * syC : 0.0;
    }
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) {
      uint32_t lo[16], hi[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int bc = kq * 16 + i;
        slice1(b[bc >> 3], c[bc & 7], lo[i], hi[i]);
      }
      store16(lo, hi, base + canon64(n, kq * 16), kYSlice);
    }
    double* A = reinterpret_cast<double*>(base + kYBytes) + n * 8;
#pragma unroll
    for (int a = 0; a < 8; ++a) A[a] = ok ? rw[(int64_t)j * 24 + a] : 0.0;
    reinterpret_cast<int32_t*>(base + kYBytes + kABytes)[n] = ok ? pw[j] : -1;
  }
}

// ---- G digits of every cell, once per product ------------------------------
// Per (cell, 16-rhs group): thread m = (r, a) forms the 64 grid values
// G_r[a][(b, c)] of the support box at the cell, one scale per rhs (max over
// its 8 a-rows), and writes its six digit rows into pass block r & 3 at row
// (r >> 2) * 8 + a: pass p holds rhs {p, 4 + p, 8 + p, 12 + p}, so epilogue
// rhs slot w collects rhs 4w .. 4w + 3 over the four passes.
__global__ void __launch_bounds__(kRows)
k_gdig_nm(const CellDev* __restrict__ cells, const WinDev* __restrict__ wins,
          const double* __restrict__ grid, int64_t grid_ld, int64_t cell_lo, int ngroups,
          uint8_t* __restrict__ gdig) {
  const int64_t cell = cell_lo + blockIdx.x;
  const int grp = blockIdx.y, rg = grp * 16;
  const CellDev cd = cells[cell];
  const WinDev wd = wins[cd.win];
  const int m = threadIdx.x, ga = m & 7, gr = m >> 3;
  const double* __restrict__ gsrc = grid + (int64_t)(rg + gr) * grid_ld + wd.grid_off;
  int p0 = cd.cc[0] + ga;
  if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
  double g[64];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    int p1 = cd.cc[1] + (i >> 3), p2 = cd.cc[2] + (i & 7);
    if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
    if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
    g[i] = gsrc[((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
    mx = fmax(mx, fabs(g[i]));
  }
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  const int eG = max(-900, exp_bound(mx));
  const double sg = pow2(46 - eG);
  uint8_t* base = gdig + (cell * ngroups + grp) * (int64_t)kGItem;
  uint8_t* blk = base + (gr & 3) * (kSl * kGBlk);
  const int n = (gr >> 2) * 8 + ga;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) slice1(g[kb * 16 + i], sg, lo[i], hi[i]);
    store16(lo, hi, blk + canon64(n, kb * 16), kGBlk);
  }
  if (ga == 0) reinterpret_cast<int32_t*>(base + kGBytes)[gr] = eG;
}

// ---- the persistent gather --------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
k_gather_nm(const SubDev* __restrict__ subs, const int32_t* __restrict__ order, int nsub,
            const int16_t* __restrict__ sub_exp, const int64_t* __restrict__ tile_off,
            const uint8_t* __restrict__ gtile, const uint8_t* __restrict__ gdig,
            double* __restrict__ out, int nrhs, mma::GatherEpi ep) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t g_full[2], g_empty[2], y_full[kYStages], y_empty[kYStages];
  __shared__ uint64_t ap_full[kAPStages], ap_empty[kAPStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t taddr_s;
  uint8_t* const sG = smem;                              // [2][kGItem]
  uint8_t* const sY = sG + 2 * kGItem;                   // [2][kYBytes]
  uint8_t* const sAP = sY + kYStages * kYBytes;          // [3][kAPBytes]

  // warp index through a shuffle: warp-uniform to the compiler, so the TMEM
  // addresses derived from it live in uniform registers
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int ngroups = nrhs / 16;
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int rounds = nsub / G, rem = nsub % G;
  const int my_rounds = rounds + ((rem > 0 && ((rounds & 1) ? (G - 1 - b) : b) < rem) ? 1 : 0);
  const int nitems = my_rounds * ngroups;
  auto item_sub = [&](int k) {
    const int i = k / ngroups;
    return order[i * G + ((i & 1) ? (G - 1 - b) : b)];
  };

  if (warp == 0) umma::tmem_alloc<512>(&taddr_s);
  if (tid == 32) {
    for (int k = 0; k < 2; ++k) {
      umma::mbar_init(&g_full[k], 1);
      umma::mbar_init(&g_empty[k], 1 + kEpi);     // last UMMA commit + epilogue warps
      umma::mbar_init(&acc_full[k], 1);
      umma::mbar_init(&acc_empty[k], kEpi);
    }
    for (int k = 0; k < kYStages; ++k) {
      umma::mbar_init(&y_full[k], 1);
      umma::mbar_init(&y_empty[k], 1);            // commit of the TMEM copy
    }
    for (int k = 0; k < kAPStages; ++k) {
      umma::mbar_init(&ap_full[k], 1);
      umma::mbar_init(&ap_empty[k], kEpi);
    }
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = taddr_s;

  if (warp == kGLoader) {
    // ------------------------------------------------------------- G loader
    if (lane == 0) {
      for (int k = 0; k < nitems; ++k) {
        const int gs = k & 1;
        if (k >= 2) umma::mbar_wait(&g_empty[gs], ((k >> 1) - 1) & 1);
        const uint8_t* src = gdig + ((int64_t)subs[item_sub(k)].cell * ngroups + k % ngroups) *
                                        (int64_t)kGItem;
        umma::mbar_arrive_expect_tx(&g_full[gs], kGItem);
        umma::bulk_g2s(sG + gs * kGItem, src, kGItem, &g_full[gs]);
      }
    }
  } else if (warp == kTLoader) {
    // ---------------------------------------------------------- tile loader
    if (lane == 0) {
      int gt = 0;
      for (int k = 0; k < nitems; ++k) {
        const int si = item_sub(k);
        const int ntile = (subs[si].count + kT - 1) / kT;
        const uint8_t* src = gtile + tile_off[si] * (int64_t)kTileBytes;
        for (int tl = 0; tl < ntile; ++tl, ++gt) {
          const int ys = gt % kYStages, as = gt % kAPStages;
          if (gt >= kYStages) umma::mbar_wait(&y_empty[ys], ((gt / kYStages) - 1) & 1);
          umma::mbar_arrive_expect_tx(&y_full[ys], kYBytes);
          umma::bulk_g2s(sY + ys * kYBytes, src + (int64_t)tl * kTileBytes, kYBytes, &y_full[ys]);
          if (gt >= kAPStages) umma::mbar_wait(&ap_empty[as], ((gt / kAPStages) - 1) & 1);
          umma::mbar_arrive_expect_tx(&ap_full[as], kAPBytes);
          umma::bulk_g2s(sAP + as * kAPBytes, src + (int64_t)tl * kTileBytes + kYBytes, kAPBytes,
                         &ap_full[as]);
        }
      }
    }
  } else if (warp == kIssuer) {
    // ---------------------------------------------------------------- issuer
    if (lane == 0) {
      int gt = 0, gp = 0;
      for (int k = 0; k < nitems; ++k) {
        const int gs = k & 1;
        const int ntile = (subs[item_sub(k)].count + kT - 1) / kT;
        umma::mbar_wait(&g_full[gs], (k >> 1) & 1);
        const uint32_t gB = umma::smem_u32(sG + gs * kGItem);
        for (int tl = 0; tl < ntile; ++tl, ++gt) {
          const int ys = gt % kYStages;
          umma::mbar_wait(&y_full[ys], (gt / kYStages) & 1);
          umma::fence_after();
          // the tile's Y digits -> TMEM (the UMMA A operand of all four passes);
          // ordered behind the previous tile's UMMAs, which read the old copy
          const uint32_t yB = umma::smem_u32(sY + ys * kYBytes);
#pragma unroll
          for (int p = 0; p < kSl; ++p)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks)
              umma::tmem_cp_128x256b(tmem + (uint32_t)(kYT0 + p * 16 + ks * 8),
                                     umma::make_sdesc(yB + p * kYSlice + ks * 256, 128, 512));
          umma::commit(&y_empty[ys]);
          for (int ps = 0; ps < 4; ++ps, ++gp) {
            const int ab = gp & 1;
            if (gp >= 2) umma::mbar_wait(&acc_empty[ab], ((gp >> 1) - 1) & 1);
            umma::fence_after();
            const uint32_t dcol = tmem + (uint32_t)(ab * kAccCols);
            const uint32_t bB = gB + ps * (kSl * kGBlk);
            // Y digit p against the stacked G slices q = 0..5-p (N = (6-p) x 32):
            // column (p + q) x 32 + n accumulates diagonal p + q
#pragma unroll
            for (int p = 0; p < kSl; ++p)
#pragma unroll
              for (int ks = 0; ks < 2; ++ks)
                umma::mma_i8_ta(dcol + (uint32_t)(p * kPassRows),
                                tmem + (uint32_t)(kYT0 + p * 16 + ks * 8),
                                umma::make_sdesc(bB + ks * 256, 128, 512),
                                umma::idesc_i8(kT, (kSl - p) * kPassRows),
                                (p > 0 || ks > 0) ? 1u : 0u);
            umma::commit(&acc_full[ab]);
          }
        }
        umma::commit(&g_empty[gs]);   // item k's G digits no longer read
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int lq = warp & 3, w = warp >> 2;
    const int m = lq * 32 + lane;                 // node row of the tile
    const uint32_t tl_lane = tmem + ((uint32_t)(lq * 32) << 16);
    const bool need_eta = ep.kind == NLD_APPLY_SYSTEM || ep.kind == NLD_APPLY_LAPLACIAN;
    const double inv_L = 1.0 / (double)ep.L;
    int gt = 0, gp = 0;
    for (int k = 0; k < nitems; ++k) {
      const int gs = k & 1;
      const int si = item_sub(k);
      const int cnt = subs[si].count;
      const int r0 = (k % ngroups) * 16 + 4 * w;  // this warp's first rhs
      const int16_t* exk = sub_exp + (int64_t)si * kExpPerSub;
      int eBm = -2000, eCm = -2000;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        eBm = max(eBm, (int)exk[8 + q]);
        eCm = max(eCm, (int)exk[16 + q]);
      }
      umma::mbar_wait(&g_full[gs], (k >> 1) & 1);
      const int4 ge = reinterpret_cast<const int4*>(sG + gs * kGItem + kGBytes)[w];
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_empty[gs]);
      // T scale per rhs: G exponent + the subproblem's Y exponents (combine6
      // carries 2^24)
      const int eb = eBm + eCm - 52;
      const int ntile = (cnt + kT - 1) / kT;
      for (int tl = 0; tl < ntile; ++tl, ++gt) {
        const int as = gt % kAPStages;
        umma::mbar_wait(&ap_full[as], (gt / kAPStages) & 1);
        const double2* Ap = reinterpret_cast<const double2*>(sAP + as * kAPBytes) + m * 4;
        const double2 a01 = Ap[0], a23 = Ap[1], a45 = Ap[2], a67 = Ap[3];
        const int px = reinterpret_cast<const int32_t*>(sAP + as * kAPBytes + kABytes)[m];
        __syncwarp();
        if (lane == 0) mbar_arrive(&ap_empty[as]);
        const bool ok = px >= 0;
        const int64_t e = (int64_t)px * nrhs + r0;
        // the running window sum / v / eta of the node, in flight during the passes
        double2 s01 = make_double2(0.0, 0.0), s23 = s01, v01 = s01, v23 = s01;
        double et = 0.0;
        if (ok) {
          if (MODE >= mma::kGatherAccum) {
            s01 = *reinterpret_cast<const double2*>(out + e);
            s23 = *reinterpret_cast<const double2*>(out + e + 2);
          }
          if (MODE == mma::kGatherFinal) {
            v01 = *reinterpret_cast<const double2*>(ep.v + e);
            v23 = *reinterpret_cast<const double2*>(ep.v + e + 2);
            if (need_eta) et = ep.eta[px];
          }
        }
        double y[4];
#pragma unroll
        for (int ps = 0; ps < 4; ++ps, ++gp) {
          const int ab = gp & 1;
          umma::mbar_wait(&acc_full[ab], (gp >> 1) & 1);
          umma::fence_after();
          // the six diagonals of a = 0..3, then of a = 4..7 (24 registers each);
          // hi and lo parts accumulate in separate chains (combine6_parts)
          const uint32_t tc = tl_lane + (uint32_t)(ab * kAccCols + w * 8);
          uint32_t dv[kSl][4];
          double h, l, sh, sl;
#pragma unroll
          for (int t = 0; t < kSl; ++t) umma::tmem_ld4(tc + (uint32_t)(t * kPassRows), dv[t]);
          umma::tmem_wait_ld();
          combine6_parts(dv, 0, h, l);
          sh = h * a01.x;
          sl = l * a01.x;
          combine6_parts(dv, 1, h, l);
          sh = fma(h, a01.y, sh);
          sl = fma(l, a01.y, sl);
          combine6_parts(dv, 2, h, l);
          sh = fma(h, a23.x, sh);
          sl = fma(l, a23.x, sl);
          combine6_parts(dv, 3, h, l);
          sh = fma(h, a23.y, sh);
          sl = fma(l, a23.y, sl);
#pragma unroll
          for (int t = 0; t < kSl; ++t) umma::tmem_ld4(tc + (uint32_t)(t * kPassRows + 4), dv[t]);
          umma::tmem_wait_ld();
          umma::fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[ab]);
          combine6_parts(dv, 0, h, l);
          sh = fma(h, a45.x, sh);
          sl = fma(l, a45.x, sl);
          combine6_parts(dv, 1, h, l);
          sh = fma(h, a45.y, sh);
          sl = fma(l, a45.y, sl);
          combine6_parts(dv, 2, h, l);
          sh = fma(h, a67.x, sh);
          sl = fma(l, a67.x, sl);
          combine6_parts(dv, 3, h, l);
          sh = fma(h, a67.y, sh);
          sl = fma(l, a67.y, sl);
          const double s = fma(sh, 4294967296.0, sl);
          y[ps] = s;
        }
        if (!ok) continue;
        y[0] *= pow2(ge.x + eb);
        y[1] *= pow2(ge.y + eb);
        y[2] *= pow2(ge.z + eb);
        y[3] *= pow2(ge.w + eb);
        double res[4];
        if (MODE == mma::kGatherStore || MODE == mma::kGatherFirst) {
#pragma unroll
          for (int i = 0; i < 4; ++i) res[i] = y[i];
        } else if (MODE == mma::kGatherAccum) {
          res[0] = s01.x + y[0];
          res[1] = s01.y + y[1];
          res[2] = s23.x + y[2];
          res[3] = s23.y + y[3];
        } else {
          const double sv[4] = {s01.x + y[0], s01.y + y[1], s23.x + y[2], s23.y + y[3]};
          const double vv[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double lam = ep.coef ? ep.coef[2 * (r0 + i)] : 0.0;
            const double mu = ep.coef ? ep.coef[2 * (r0 + i) + 1] : 0.0;
            res[i] = mma::epi_value_r(ep.kind, (double)ep.L, inv_L, sv[i], vv[i], et, lam, mu);
          }
        }
        *reinterpret_cast<double2*>(out + e) = make_double2(res[0], res[1]);
        *reinterpret_cast<double2*>(out + e + 2) = make_double2(res[2], res[3]);
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tmem);
}

}  // namespace nm
}  // namespace oz

// ---- host side ------------------------------------------------------------

int64_t gather_gdig_bytes() { return oz::nm::kGItem; }

// plan-time tile table of the sliced gather: when it fits in half of the
// free memory (else the gather of 3-D windows runs on the fp64 DMMA kernels)
void gather_nm_tables(PlanSet& ps, const std::vector<SubDev>& h, cudaStream_t st) {
  if (ps.gtile || h.empty()) return;
  std::vector<int64_t> off(h.size());
  int64_t tiles = 0;
  for (size_t i = 0; i < h.size(); ++i) {
    off[i] = tiles;
    tiles += (h[i].count + oz::nm::kT - 1) / oz::nm::kT;
  }
  const size_t need = (size_t)tiles * oz::nm::kTileBytes;
  size_t free_b = 0, total_b = 0;
  NLD_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (need == 0 || need > free_b / 2) return;
  NLD_CUDA(cudaMalloc(&ps.gtile_off, sizeof(int64_t) * off.size()));
  NLD_CUDA(cudaMalloc(&ps.gtile, need));
  NLD_CUDA(cudaMemcpyAsync(ps.gtile_off, off.data(), sizeof(int64_t) * off.size(),
                           cudaMemcpyHostToDevice, st));
  oz::nm::k_gtile<<<(unsigned)h.size(), oz::nm::kT, 0, st>>>(ps.subs[3], ps.wdev, ps.rows, ps.pix,
                                                             ps.sub_exp, ps.gtile_off, ps.gtile);
  NLD_CUDA(cudaGetLastError());
  // the host offsets must outlive the async copy
  NLD_CUDA(cudaStreamSynchronize(st));
}

template <int MODE>
static void launch_nm(unsigned grid_n, const SubDev* subs, const int32_t* order, unsigned nsub,
                      const int16_t* ex, const int64_t* toff, const uint8_t* gtile,
                      const uint8_t* gdig, double* out, int nrhs, const mma::GatherEpi& ep,
                      cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(oz::nm::k_gather_nm<MODE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  oz::nm::smem_bytes()));
    attr = true;
  }
  oz::nm::k_gather_nm<MODE><<<grid_n, oz::nm::kThreads, oz::nm::smem_bytes(), st>>>(
      subs, order, (int)nsub, ex, toff, gtile, gdig, out, nrhs, ep);
}

void launch_gather_nm(const PlanSet& ps, const SubDev* subs, const int16_t* ex,
                      const int32_t* order, const int64_t* toff, unsigned nsub,
                      const double* grid, int64_t grid_ld, double* out, int nrhs,
                      const mma::GatherEpi& ep, cudaStream_t st, uint8_t* gdig, int64_t cell_lo,
                      int64_t ncell) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    NLD_CUDA(cudaGetDevice(&dev));
    NLD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  oz::nm::k_gdig_nm<<<dim3((unsigned)ncell, (unsigned)(nrhs / 16)), oz::kRows, 0, st>>>(
      ps.cells, ps.wdev, grid, grid_ld, cell_lo, nrhs / 16, gdig);
  NLD_CUDA(cudaGetLastError());
  const unsigned grid_n = std::min<unsigned>(nsub, (unsigned)sms);
  switch (ep.mode) {
    case mma::kGatherStore:
      launch_nm<mma::kGatherStore>(grid_n, subs, order, nsub, ex, toff, ps.gtile, gdig, out, nrhs,
                                   ep, st);
      break;
    case mma::kGatherFirst:
      launch_nm<mma::kGatherFirst>(grid_n, subs, order, nsub, ex, toff, ps.gtile, gdig, out, nrhs,
                                   ep, st);
      break;
    case mma::kGatherAccum:
      launch_nm<mma::kGatherAccum>(grid_n, subs, order, nsub, ex, toff, ps.gtile, gdig, out, nrhs,
                                   ep, st);
      break;
    default:
      launch_nm<mma::kGatherFinal>(grid_n, subs, order, nsub, ex, toff, ps.gtile, gdig, out, nrhs,
                                   ep, st);
      break;
  }
  NLD_CUDA(cudaGetLastError());
}

}  // namespace nld
