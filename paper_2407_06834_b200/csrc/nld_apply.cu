// One application of the ANOVA kernel: per window spread -> fused separable
// convolution (FFT, x kernel coefficients, FFT) -> gather, summed over
// windows with the degree/diagonal epilogue fused into one pass.
//
// Reference path (one window): gauss_transform_fast (transform.py:323-333)
//   = nfft_adjoint (spread _kernels.py:48-88, ifftn, crop, deconvolve)
//   x kernel_coeffs
//   nfft (deconvolve, embed, fftn, gather _kernels.py:91-136);
// summed over windows in AnovaOperator._fast_apply (kernel.py:79-93) and
// shifted in ShiftedSystem.apply (linops.py:43-50).
//
// B200 design:
//  * spread: one CTA per subproblem (<= 512 nodes of ONE stencil cell, sorted
//    once at plan build).  Threads own (a,b) pairs of the (2m)^3 block and
//    accumulate the c-axis in registers; node weights are staged in shared
//    memory and read by broadcast.  No atomics: each subproblem writes its
//    partial block, and `assemble` sums blocks per grid point in a fixed
//    order (deterministic).
//  * conv: the grid operation FFT -> x E_k -> FFT is exactly a separable
//    circulant convolution with a complex 1-D kernel K (the unpaired -M/2
//    frequency makes it complex); it runs pruned to the support box.
//  * gather: one CTA per subproblem; the (2m)^3 grid block of its cell sits in
//    shared memory, each thread owns a node and contracts a -> b -> c.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <cstdlib>

#include "nld_internal.cuh"
#include "nld_switch.cuh"
#include "nld_mma.cuh"

namespace nld {

namespace {

constexpr int kThreads = 128;      // gather / generic CTAs
constexpr int kSpreadWarps = 8;    // spread CTA = 8 warps
constexpr int kSpreadThreads = 32 * kSpreadWarps;
constexpr int kChunk = 128;

template <int D, int MC>
struct Geo {
  static constexpr int S = 2 * MC;
  static constexpr int SA = (D == 3) ? S : 1;
  static constexpr int SB = (D >= 2) ? S : 1;
  static constexpr int SC = S;
  static constexpr int PAIRS = SA * SB;
  static constexpr int R = (PAIRS + 31) / 32;
  static constexpr int TEAM_RAW = (PAIRS + R - 1) / R;
  static constexpr int TEAM = TEAM_RAW <= 1 ? 1 : TEAM_RAW <= 2 ? 2 : TEAM_RAW <= 4 ? 4
                              : TEAM_RAW <= 8 ? 8 : TEAM_RAW <= 16 ? 16 : 32;
  static constexpr int TPW = 32 / TEAM;                // teams per warp
  static constexpr int ROW = S * D;                    // global row (doubles)
  static constexpr int SROW_RAW = D * S;                // [C][B][A]
  static constexpr int SROW = (SROW_RAW % 4 == 0) ? SROW_RAW + 2 : SROW_RAW;  // 16B aligned, bank skew
  static constexpr int BLK = SA * SB * SC;
  static constexpr int SMEM_STAGE = kChunk * SROW + kChunk * kSpreadWarps;
  static constexpr int SMEM_RED = kSpreadWarps * BLK;
  static constexpr int SMEM = SMEM_STAGE > SMEM_RED ? SMEM_STAGE : SMEM_RED;
  static constexpr int GRB = (BLK <= 512) ? 16 : 8;      // gather rhs per smem pass
};

__device__ __forceinline__ int wrap_pos(int p, int w) {
  // box coordinate after a stencil offset; only exceeds [0,w) in wrap mode
  if (p >= w) p -= w;
  if (p < 0) p += w;
  return p;
}

template <int D>
__device__ __forceinline__ int64_t box_flat(const WinDev& wd, const int* p) {
  int64_t f = 0;
  for (int s = 0; s < D; ++s) f = f * wd.box_w[s] + p[s];
  return f;
}

// ---- spread ---------------------------------------------------------------
//
// CTA = one subproblem, all right-hand sides.  The node rows of a chunk are
// staged once in shared memory and reused by every rhs.  Warps map onto
// (rhs slot, point slice): with nrhs >= 8 each warp owns one rhs and the
// whole block (no cross-warp reduction); with fewer rhs several warps share
// an rhs and reduce through shared memory at the end.  Inside a warp, TEAM
// lanes own the (a,b) pairs of the (2m)^D block and accumulate its c-axis
// in registers; C weights are read by 16-byte broadcast.

template <int D, int MC>
__global__ void __launch_bounds__(kSpreadThreads)
k_spread(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
         const double* __restrict__ rows, const int32_t* __restrict__ pix,
         const double* __restrict__ vt, int nrhs, double* __restrict__ blocks) {
  using G = Geo<D, MC>;
  extern __shared__ double sm[];
  double* sv = sm + kChunk * G::SROW;          // [kChunk][kSpreadWarps]
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int tl = lane & (G::TEAM - 1);
  const int rgs = nrhs < kSpreadWarps ? nrhs : kSpreadWarps;   // rhs per group
  const int wpr = kSpreadWarps / rgs;                           // warps per rhs
  const int slot = warp / wpr;
  const int slice = warp - slot * wpr;
  const int team = slice * G::TPW + lane / G::TEAM;
  const int nteam = wpr * G::TPW;
  const bool busy = slot < rgs;

  int pa[G::R], pb[G::R];
  bool pok[G::R];
#pragma unroll
  for (int r = 0; r < G::R; ++r) {
    int p = tl + G::TEAM * r;
    pok[r] = p < G::PAIRS;
    pa[r] = pok[r] ? p / G::SB : 0;
    pb[r] = pok[r] ? p % G::SB : 0;
  }
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * G::ROW;
  const int32_t* __restrict__ pw = pix + sd.start;

  for (int rg = 0; rg < nrhs; rg += rgs) {
    const int rhs = rg + slot;
    const bool act = busy && rhs < nrhs;
    double acc[G::R][G::SC];
#pragma unroll
    for (int r = 0; r < G::R; ++r)
#pragma unroll
      for (int c = 0; c < G::SC; ++c) acc[r][c] = 0.0;
    for (int c0 = 0; c0 < sd.count; c0 += kChunk) {
      const int cn = min(kChunk, sd.count - c0);
      __syncthreads();
      // v of this rhs group, pixel-major input [N][nrhs]
      for (int e = tid; e < cn * rgs; e += kSpreadThreads) {
        const int pt = e / rgs, q = e - pt * rgs;
        sv[pt * kSpreadWarps + q] =
            (rg + q < nrhs) ? vt[(int64_t)pw[c0 + pt] * nrhs + rg + q] : 0.0;
      }
      // rows: dim s -> smem segment (D-1-s)*S (C first, then B, then A)
      if (rg == 0 || sd.count > kChunk) {
        for (int e = tid; e < cn * G::ROW; e += kSpreadThreads) {
          const int pt = e / G::ROW;
          const int k = e - pt * G::ROW;
          const int sdim = k / G::S;
          const int i = k - sdim * G::S;
          sm[pt * G::SROW + (D - 1 - sdim) * G::S + i] = rw[(int64_t)(c0 + pt) * G::ROW + k];
        }
      }
      __syncthreads();
      if (act) {
        for (int pt = team; pt < cn; pt += nteam) {
          const double* row = sm + pt * G::SROW;
          const double v = sv[pt * kSpreadWarps + slot];
          double cw[G::SC];
#pragma unroll
          for (int c = 0; c < G::SC; c += 2) {
            double2 t = *reinterpret_cast<const double2*>(row + c);
            cw[c] = t.x;
            cw[c + 1] = t.y;
          }
#pragma unroll
          for (int r = 0; r < G::R; ++r) {
            double ab;
            if (D == 3) ab = (v * row[2 * G::S + pa[r]]) * row[G::S + pb[r]];
            else if (D == 2) ab = v * row[G::S + pb[r]];
            else ab = v;
#pragma unroll
            for (int c = 0; c < G::SC; ++c) acc[r][c] = fma(ab, cw[c], acc[r][c]);
          }
        }
      }
    }
    // teams of a warp -> lanes [0, TEAM)
#pragma unroll
    for (int off = G::TEAM; off < 32; off <<= 1)
#pragma unroll
      for (int r = 0; r < G::R; ++r)
#pragma unroll
        for (int c = 0; c < G::SC; ++c)
          acc[r][c] += __shfl_xor_sync(0xffffffffu, acc[r][c], off);
    if (wpr == 1) {
      if (act && lane < G::TEAM) {
#pragma unroll
        for (int r = 0; r < G::R; ++r)
          if (pok[r]) {
            const int p = tl + G::TEAM * r;
#pragma unroll
            for (int c = 0; c < G::SC; ++c)
              blocks[(sd.block + p * G::SC + c) * nrhs + rhs] = acc[r][c];
          }
      }
    } else {
      __syncthreads();
      if (busy && lane < G::TEAM) {
#pragma unroll
        for (int r = 0; r < G::R; ++r)
          if (pok[r]) {
            const int p = tl + G::TEAM * r;
#pragma unroll
            for (int c = 0; c < G::SC; ++c) sm[warp * G::BLK + p * G::SC + c] = acc[r][c];
          }
      }
      __syncthreads();
      for (int e = tid; e < rgs * G::BLK; e += kSpreadThreads) {
        const int q = e / G::BLK, k = e - q * G::BLK;
        if (rg + q >= nrhs) continue;
        double sum = 0.0;
        for (int w = 0; w < wpr; ++w) sum += sm[(q * wpr + w) * G::BLK + k];
        blocks[(sd.block + k) * nrhs + rg + q] = sum;
      }
    }
  }
}

// ---- assemble: grid point <- sum of the blocks of the cells covering it -----

// Assemble: grid point <- sum of the partial blocks of the cells covering it.
// 8 lanes share one (grid point, rhs) and split the outermost offset axis;
// their partial sums are combined by a fixed xor tree (deterministic, no
// atomics).  Lane layout: lane = 8 * item + slice.
__global__ void __launch_bounds__(256, 4)
k_assemble(const WinDev* __restrict__ wins, int w0, const int2* __restrict__ cellinfo,
           const double* __restrict__ blocks, int nrhs, double* __restrict__ grid,
           int64_t grid_ld) {
  const int w = w0 + blockIdx.y;
  const WinDev wd = wins[w];
  const int S = wd.S;
  const int d = wd.d;
  const int2* __restrict__ ci = cellinfo + wd.cellmap_off;
  const int on0 = d == 3 ? S : 1, on1 = d >= 2 ? S : 1;
  const int blk = on0 * on1 * S;
  const int slice = threadIdx.x & 7;
  const int64_t total = wd.box_size * nrhs;
  const int64_t items_per_block = blockDim.x >> 3;
  for (int64_t base = blockIdx.x * items_per_block; base < total;
       base += (int64_t)gridDim.x * items_per_block) {
    const int64_t id = base + (threadIdx.x >> 3);
    const bool live = id < total;
    const int r = live ? (int)(id % nrhs) : 0;
    const int64_t e = live ? id / nrhs : 0;
    double sum = 0.0;
    if (live && wd.fast) {
      // point coordinates on (t0, t1, t2), unused leading dims 0
      int t0 = 0, t1 = 0, t2, bw1 = 1, bw2;
      if (d == 3) {
        bw2 = wd.box_w[2];
        bw1 = wd.box_w[1];
        t2 = (int)(e % bw2);
        t1 = (int)((e / bw2) % bw1);
        t0 = (int)(e / ((int64_t)bw2 * bw1));
      } else if (d == 2) {
        bw2 = wd.box_w[1];
        bw1 = wd.box_w[0];
        t2 = (int)(e % bw2);
        t1 = (int)(e / bw2);
      } else {
        bw2 = wd.box_w[0];
        t2 = (int)e;
      }
      const int bw0 = d == 3 ? wd.box_w[0] : 1;
      // the split axis: o0 for d = 3, o1 for d = 2, o2 for d = 1
      for (int sp = slice; sp < S; sp += 8) {
        const int o0s = d == 3 ? sp : 0, o0e = d == 3 ? sp + 1 : 1;
        for (int o0 = o0s; o0 < o0e; ++o0) {
          int c0 = t0 - o0;
          if (c0 < 0) {
            if (!wd.wrap) continue;
            c0 += bw0;
          }
          const int o1s = d == 2 ? sp : 0, o1e = d == 3 ? on1 : (d == 2 ? sp + 1 : 1);
          for (int o1 = o1s; o1 < o1e; ++o1) {
            int c1 = t1 - o1;
            if (c1 < 0) {
              if (!wd.wrap) continue;
              c1 += bw1;
            }
            const int64_t rowkey = ((int64_t)c0 * bw1 + c1) * bw2;
            const int inner01 = (o0 * on1 + o1) * S;
            const int o2s = d == 1 ? sp : 0, o2e = d == 1 ? sp + 1 : S;
            for (int o2 = o2s; o2 < o2e; ++o2) {
              int c2 = t2 - o2;
              if (c2 < 0) {
                if (!wd.wrap) break;
                c2 += bw2;
              }
              const int2 c = ci[rowkey + c2];
              for (int q = 0; q < c.y; ++q)
                sum += blocks[((int64_t)c.x + (int64_t)q * blk + inner01 + o2) * nrhs + r];
            }
          }
        }
      }
    }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    if (live && slice == 0) grid[r * grid_ld + wd.grid_off + e] = sum;
  }
}

// ---- separable assemble (d = 3, S = 8, no wrap) ----------------------------
// G[p] = sum_{o in [0,8)^3} X[p - o][o], X[c][o] = sum of the cell's sub
// blocks.  Three passes, one per offset axis, each summing 8 terms in a fixed
// order (deterministic):
//   Y1[c0][c1][p2][o0][o1] = sum_o2 X[c0][c1][p2-o2][o0][o1][o2]
//   Y2[c0][p1][p2][o0]     = sum_o1 Y1[c0][p1-o1][p2][o0][o1]
//   G[p0][p1][p2]          = sum_o0 Y2[p0-o0][p1][p2][o0]
// (all with the rhs index innermost: [..][nrhs]).
__global__ void __launch_bounds__(128)
k_asm_p12(const WinDev* __restrict__ wins, int w, const int2* __restrict__ cellinfo,
          const double* __restrict__ blocks, int nrhs, double* __restrict__ y2) {
  // Passes 1 and 2 in one kernel (Y1 never reaches memory): one CTA per
  // (c0, p1, p2) line of 8 nrhs values (o0, r).  The line's 64 source cells
  // (o1, o2) are looked up once per CTA, and lines whose cells are all empty
  // -- most of the box -- are only zero-filled (per CTA pass: small batches
  // take several lines at once).  Each value keeps the two
  // passes' summation order: Y1 terms over o2 (first blocks, then the extra
  // blocks of cells split into several subproblems), then those over o1.
  const WinDev wd = wins[w];
  const int B1 = wd.box_w[1], B2 = wd.box_w[2];
  const int nline = wd.box_w[0] * B1 * B2;
  const int2* __restrict__ ci = cellinfo + wd.cellmap_off;
  const int per = 8 * nrhs;
  // small batches: several consecutive lines per CTA pass, so that a single
  // right-hand side still fills the CTA (per >= 8: at most 16 lines)
  const int L = per >= 128 ? 1 : 128 / per;
  __shared__ int2 cs[16 * 64];   // [line][o1][o2]: (first block, number of blocks)
  __shared__ uchar2 rowm[16 * 8];  // [line][o1]: o2 masks (occupied, several blocks)
  for (int l0 = blockIdx.x * L; l0 < nline; l0 += gridDim.x * L) {
    __syncthreads();
    int mine = 0;
    for (int k = threadIdx.x; k < L * 64; k += 128) {
      const int ln = l0 + (k >> 6), o1 = (k >> 3) & 7, o2 = k & 7;
      int2 c = make_int2(0, 0);
      if (ln < nline) {
        const int p2 = ln % B2, p1 = (ln / B2) % B1;
        if (p1 - o1 >= 0 && p2 - o2 >= 0) c = __ldg(ci + ln - o1 * B2 - o2);
      }
      cs[k] = c;
      mine |= c.y > 0;
      // per (line, o1) row of eight cells: which are occupied / split (a warp
      // holds four whole rows; L * 64 is a multiple of 32, so it votes whole)
      const unsigned occ = __ballot_sync(0xffffffffu, c.y > 0);
      const unsigned ext = __ballot_sync(0xffffffffu, c.y > 1);
      if ((k & 7) == 0) {
        const int sh = k & 31;
        rowm[k >> 3] = make_uchar2((occ >> sh) & 0xffu, (ext >> sh) & 0xffu);
      }
    }
    const int any = __syncthreads_or(mine);
    const int nval = min(L, nline - l0) * per;
    double* __restrict__ dst = y2 + (int64_t)l0 * per;
    if (!any) {
      for (int k = threadIdx.x; k < nval; k += 128) dst[k] = 0.0;
      continue;
    }
    for (int k = threadIdx.x; k < nval; k += 128) {
      const int li = k / per, e = k - li * per;
      const int2* __restrict__ cl = cs + li * 64;
      const int o0 = e / nrhs, r = e - o0 * nrhs;
      const double* __restrict__ src = blocks + (int64_t)o0 * 64 * nrhs + r;
      double sum = 0.0;
#pragma unroll 2
      for (int o1 = 0; o1 < 8; ++o1) {
        const uchar2 rm = rowm[li * 8 + o1];
        if (rm.x == 0) continue;   // an empty row adds +0.0
        double inner = 0.0;
#pragma unroll
        for (int o2 = 0; o2 < 8; ++o2) {
          const int2 c = cl[o1 * 8 + o2];
          if (c.y > 0) inner += __ldg(src + ((int64_t)c.x + o1 * 8 + o2) * nrhs);
        }
        if (rm.y != 0) {
#pragma unroll
          for (int o2 = 0; o2 < 8; ++o2) {
            const int2 c = cl[o1 * 8 + o2];
            for (int q = 1; q < c.y; ++q)
              inner += __ldg(src + ((int64_t)c.x + (int64_t)q * 512 + o1 * 8 + o2) * nrhs);
          }
        }
        sum += inner;
      }
      dst[k] = sum;
    }
  }
}

__global__ void __launch_bounds__(256)
k_asm_p3(const WinDev* __restrict__ wins, int w, const double* __restrict__ y2, int nrhs,
         double* __restrict__ grid, int64_t grid_ld) {
  const WinDev wd = wins[w];
  const int B1 = wd.box_w[1], B2 = wd.box_w[2];
  const int64_t total = wd.box_size * nrhs;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(id % nrhs);
    const int64_t e = id / nrhs;
    const int p2 = (int)(e % B2);
    const int p1 = (int)((e / B2) % B1);
    const int p0 = (int)(e / ((int64_t)B2 * B1));
    double sum = 0.0;
#pragma unroll
    for (int o0 = 0; o0 < 8; ++o0) {
      const int c0 = p0 - o0;
      if (c0 < 0) break;
      sum += y2[((((int64_t)c0 * B1 + p1) * B2 + p2) * 8 + o0) * nrhs + r];
    }
    grid[r * grid_ld + wd.grid_off + e] = sum;
  }
}

// ---- edge nodes: the i = 0 / i = 2m+1 stencil slices (rare) ---------------

__device__ __forceinline__ bool edge_combo(const EdgeDev& ed, int d, int W, int S,
                                           int lin, int* ii, double* wprod) {
  // decode lin into per-dim offsets 0..W-1; reject the principal part
  bool principal = true;
  double w = 1.0;
  for (int s = d - 1; s >= 0; --s) {
    ii[s] = lin % W;
    lin /= W;
    if (ii[s] < 1 || ii[s] > S) principal = false;
    w *= ed.w[s][ii[s]];
  }
  *wprod = w;
  return !principal && w != 0.0;
}

__global__ void k_spread_edges(const EdgeDev* __restrict__ edges, int64_t ne,
                               const WinDev* __restrict__ wins,
                               const double* __restrict__ vt, int nrhs,
                               double* __restrict__ grid, int64_t grid_ld) {
  const int rhs = blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ne;
       k += (int64_t)gridDim.x * blockDim.x) {
    const EdgeDev& ed = edges[k];
    const WinDev wd = wins[ed.win];
    const double val = vt[(int64_t)ed.pix * nrhs + rhs];
    const int W = wd.S + 2;
    int total = 1;
    for (int s = 0; s < wd.d; ++s) total *= W;
    for (int lin = 0; lin < total; ++lin) {
      int ii[3];
      double wp;
      if (!edge_combo(ed, wd.d, W, wd.S, lin, ii, &wp)) continue;
      int p[3];
      for (int s = 0; s < wd.d; ++s) p[s] = wrap_pos(ed.cc[s] + ii[s] - 1, wd.box_w[s]);
      int64_t f = 0;
      for (int s = 0; s < wd.d; ++s) f = f * wd.box_w[s] + p[s];
      atomicAdd(grid + rhs * grid_ld + wd.grid_off + f, val * wp);
    }
  }
}

__global__ void k_gather_edges(const EdgeDev* __restrict__ edges, int64_t ne,
                               const WinDev* __restrict__ wins,
                               const double* __restrict__ grid, int64_t grid_ld,
                               double* __restrict__ wout, int64_t win_stride, int nrhs) {
  const int rhs = blockIdx.y;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ne;
       k += (int64_t)gridDim.x * blockDim.x) {
    const EdgeDev& ed = edges[k];
    const WinDev wd = wins[ed.win];
    const int W = wd.S + 2;
    int total = 1;
    for (int s = 0; s < wd.d; ++s) total *= W;
    double y = 0.0;
    for (int lin = 0; lin < total; ++lin) {
      int ii[3];
      double wp;
      if (!edge_combo(ed, wd.d, W, wd.S, lin, ii, &wp)) continue;
      int p[3];
      for (int s = 0; s < wd.d; ++s) p[s] = wrap_pos(ed.cc[s] + ii[s] - 1, wd.box_w[s]);
      int64_t f = 0;
      for (int s = 0; s < wd.d; ++s) f = f * wd.box_w[s] + p[s];
      y += grid[rhs * grid_ld + wd.grid_off + f] * wp;
    }
    wout[((int64_t)ed.win * win_stride + ed.pix) * nrhs + rhs] += y;
  }
}

// ---- generic path (cutoffs without a templated kernel) --------------------

__global__ void k_spread_generic(const WinDev* __restrict__ wins, int w,
                                 const double* __restrict__ rows,
                                 const int32_t* __restrict__ pix,
                                 const int32_t* __restrict__ key,
                                 const double* __restrict__ vt, int nrhs,
                                 double* __restrict__ grid, int64_t grid_ld, int64_t N) {
  const int rhs = blockIdx.y;
  const WinDev wd = wins[w];
  const int S = wd.S, d = wd.d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double* row = rows + wd.row_off + e * (int64_t)S * d;
    const double val = vt[(int64_t)pix[wd.node_off + e] * nrhs + rhs];
    int cc[3] = {0, 0, 0};
    int rem = key[wd.node_off + e];
    for (int s = d - 1; s >= 0; --s) {
      cc[s] = rem % wd.box_w[s];
      rem /= wd.box_w[s];
    }
    int total = 1;
    for (int s = 0; s < d; ++s) total *= S;
    for (int lin = 0; lin < total; ++lin) {
      int l = lin;
      double wp = val;
      int64_t f = 0;
      int ii[3];
      for (int s = d - 1; s >= 0; --s) {
        ii[s] = l % S;
        l /= S;
      }
      for (int s = 0; s < d; ++s) {
        wp *= row[s * S + ii[s]];
        f = f * wd.box_w[s] + wrap_pos(cc[s] + ii[s], wd.box_w[s]);
      }
      atomicAdd(grid + rhs * grid_ld + wd.grid_off + f, wp);
    }
  }
}

__global__ void k_gather_generic(const WinDev* __restrict__ wins, int w, int nrhs,
                                 const double* __restrict__ rows,
                                 const int32_t* __restrict__ pix,
                                 const int32_t* __restrict__ key,
                                 const double* __restrict__ grid, int64_t grid_ld,
                                 double* __restrict__ wout, int64_t N) {
  const int rhs = blockIdx.y;
  const WinDev wd = wins[w];
  const int S = wd.S, d = wd.d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double* row = rows + wd.row_off + e * (int64_t)S * d;
    int cc[3] = {0, 0, 0};
    int rem = key[wd.node_off + e];
    for (int s = d - 1; s >= 0; --s) {
      cc[s] = rem % wd.box_w[s];
      rem /= wd.box_w[s];
    }
    int total = 1;
    for (int s = 0; s < d; ++s) total *= S;
    double y = 0.0;
    for (int lin = 0; lin < total; ++lin) {
      int l = lin;
      double wp = 1.0;
      int64_t f = 0;
      int ii[3];
      for (int s = d - 1; s >= 0; --s) {
        ii[s] = l % S;
        l /= S;
      }
      for (int s = 0; s < d; ++s) {
        wp *= row[s * S + ii[s]];
        f = f * wd.box_w[s] + wrap_pos(cc[s] + ii[s], wd.box_w[s]);
      }
      y += grid[rhs * grid_ld + wd.grid_off + f] * wp;
    }
    wout[((int64_t)w * N + pix[wd.node_off + e]) * nrhs + rhs] = y;
  }
}

// ---- separable convolution pass --------------------------------------------

__global__ void k_conv(const WinDev* __restrict__ wins, int w0, int pass,
                       const double2* __restrict__ K,
                       const double* __restrict__ gin, const double2* __restrict__ cin,
                       double2* __restrict__ cout, double* __restrict__ gout,
                       int64_t grid_ld) {
  const int w = w0 + blockIdx.y;
  const int rhs = blockIdx.z;
  const WinDev wd = wins[w];
  if (pass >= wd.d) return;
  const int axis = wd.d - 1 - pass;
  const bool first = pass == 0;
  const bool last = pass == wd.d - 1;
  const double2* __restrict__ kw = K + wd.kern_off;
  const int n = wd.n;
  int64_t stride = 1;
  for (int s = wd.d - 1; s > axis; --s) stride *= wd.box_w[s];
  const int wa = wd.box_w[axis];
  const int64_t base = rhs * grid_ld + wd.grid_off;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < wd.box_size;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)((e / stride) % wa);
    const int64_t line = e - (int64_t)t * stride;
    double re = 0.0, im = 0.0;
    for (int s = 0; s < wa; ++s) {
      int dl = (s - t) % n;
      if (dl < 0) dl += n;
      const double2 k = kw[dl];
      const int64_t src = base + line + (int64_t)s * stride;
      if (first) {
        const double g = gin[src];
        re = fma(k.x, g, re);
        im = fma(k.y, g, im);
      } else {
        const double2 x = cin[src];
        re = fma(k.x, x.x, re);
        re = fma(-k.y, x.y, re);
        im = fma(k.x, x.y, im);
        im = fma(k.y, x.x, im);
      }
    }
    if (last) gout[base + e] = re;
    else cout[base + e] = make_double2(re, im);
  }
}

// Passes 0 and 1 of a 3-D window (axes 2 and 1) in one kernel: one CTA per
// (p0 slab, rhs) keeps the slab and the axis-2 result in shared memory, so the
// per-window convolution is two launches instead of three and the first
// intermediate never reaches L2.  Same terms, order and FMAs per value as two
// k_conv passes (bit-identical).  Writes the complex slab for pass 2.
__host__ __device__ inline size_t conv01_smem(int B1, int B2) {
  return (size_t)B1 * B2 * (sizeof(double) + sizeof(double2)) +
         (size_t)(2 * (B1 > B2 ? B1 : B2)) * sizeof(double2);
}
__global__ void __launch_bounds__(256)
k_conv01(const WinDev* __restrict__ wins, int w, const double2* __restrict__ K,
         const double* __restrict__ gin, double2* __restrict__ cout, int64_t grid_ld) {
  extern __shared__ double2 cv_smem[];
  const WinDev wd = wins[w];
  const int B1 = wd.box_w[1], B2 = wd.box_w[2], n = wd.n;
  const int slab = B1 * B2, wm = B1 > B2 ? B1 : B2;
  double2* const ta = cv_smem;                       // [B1][B2] axis-2 result
  double2* const ks = ta + slab;                     // kernel at offsets -(wm-1) .. wm-1
  double* const g = reinterpret_cast<double*>(ks + 2 * wm);   // [B1][B2] input slab
  const double2* __restrict__ kw = K + wd.kern_off;
  const int64_t base = (int64_t)blockIdx.y * grid_ld + wd.grid_off + (int64_t)blockIdx.x * slab;
  for (int i = threadIdx.x; i < slab; i += blockDim.x) g[i] = gin[base + i];
  for (int j = threadIdx.x; j < 2 * wm - 1; j += blockDim.x) {
    int dl = (j - (wm - 1)) % n;
    if (dl < 0) dl += n;
    ks[j] = kw[dl];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < slab; i += blockDim.x) {
    const int t = i % B2;
    const double* __restrict__ line = g + (i - t);
    const double2* __restrict__ kk = ks + (wm - 1 - t);      // kk[s] = kw[(s - t) mod n]
    double re = 0.0, im = 0.0;
    for (int s = 0; s < B2; ++s) {
      const double2 k = kk[s];
      re = fma(k.x, line[s], re);
      im = fma(k.y, line[s], im);
    }
    ta[i] = make_double2(re, im);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < slab; i += blockDim.x) {
    const int p2 = i % B2, t = i / B2;
    const double2* __restrict__ kk = ks + (wm - 1 - t);
    double re = 0.0, im = 0.0;
    for (int s = 0; s < B1; ++s) {
      const double2 k = kk[s];
      const double2 x = ta[s * B2 + p2];
      re = fma(k.x, x.x, re);
      re = fma(-k.y, x.y, re);
      im = fma(k.x, x.y, im);
      im = fma(k.y, x.x, im);
    }
    cout[base + i] = make_double2(re, im);
  }
}

// ---- gather -------------------------------------------------------------
//
// CTA = one subproblem, all rhs.  The (2m)^D grid blocks of its cell for a
// group of GRB rhs sit in shared memory; each thread owns a node, holds its
// weights in registers and contracts c -> b -> a for every rhs of the group.

template <int D, int MC>
__global__ void __launch_bounds__(kThreads)
k_gather(const SubDev* __restrict__ subs, const CellDev* __restrict__ cells,
         const WinDev* __restrict__ wins, const double* __restrict__ rows,
         const int32_t* __restrict__ pix, const double* __restrict__ grid,
         int64_t grid_ld, double* __restrict__ wout, int64_t N, int nrhs, int accum) {
  using G = Geo<D, MC>;
  extern __shared__ double gb[];   // [GRB][BLK]
  const SubDev sd = subs[blockIdx.x];
  const CellDev cd = cells[sd.cell];
  const WinDev wd = wins[sd.win];
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * G::ROW;
  // accum < 0: this window's slot of wout [L][N][nrhs]; otherwise wout is the
  // fused product's running window sum [N][nrhs] (store if accum == 0, add if
  // 1 -- each node is in exactly one subproblem of the window: no races)
  double* __restrict__ out = accum < 0 ? wout + (int64_t)sd.win * N * nrhs : wout;
  for (int rg = 0; rg < nrhs; rg += G::GRB) {
    const int rn = min(G::GRB, nrhs - rg);
    __syncthreads();
    for (int e = threadIdx.x; e < rn * G::BLK; e += kThreads) {
      const int q = e / G::BLK;
      const int k = e - q * G::BLK;
      int off[3];
      off[0] = k / (G::SB * G::SC);
      off[1] = (k / G::SC) % G::SB;
      off[2] = k % G::SC;
      int p[3];
      if (D == 3) {
        for (int s = 0; s < 3; ++s) p[s] = wrap_pos(cd.cc[s] + off[s], wd.box_w[s]);
      } else if (D == 2) {
        p[0] = wrap_pos(cd.cc[0] + off[1], wd.box_w[0]);
        p[1] = wrap_pos(cd.cc[1] + off[2], wd.box_w[1]);
      } else {
        p[0] = wrap_pos(cd.cc[0] + off[2], wd.box_w[0]);
      }
      gb[e] = grid[(int64_t)(rg + q) * grid_ld + wd.grid_off + box_flat<D>(wd, p)];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < sd.count; j += kThreads) {
      double wrow[G::ROW];
      const double2* src = reinterpret_cast<const double2*>(rw + (int64_t)j * G::ROW);
#pragma unroll
      for (int k = 0; k < G::ROW / 2; ++k) {
        double2 t = __ldg(src + k);
        wrow[2 * k] = t.x;
        wrow[2 * k + 1] = t.y;
      }
      double* __restrict__ o = out + (int64_t)pix[sd.start + j] * nrhs + rg;
      for (int q = 0; q < rn; ++q) {
        const double* gq = gb + q * G::BLK;
        double y = 0.0;
#pragma unroll
        for (int a = 0; a < G::SA; ++a) {
          double ua = 0.0;
#pragma unroll
          for (int b = 0; b < G::SB; ++b) {
            const double* gr = gq + (a * G::SB + b) * G::SC;
            double t = 0.0;
#pragma unroll
            for (int c = 0; c < G::SC; c += 2) {
              double2 gg = *reinterpret_cast<const double2*>(gr + c);
              t = fma(gg.x, wrow[(D - 1) * G::S + c], t);
              t = fma(gg.y, wrow[(D - 1) * G::S + c + 1], t);
            }
            if (D >= 2) ua = fma(t, wrow[(D - 2) * G::S + b], ua);
            else ua = t;
          }
          if (D == 3) y = fma(ua, wrow[a], y);
          else y = ua;
        }
        o[q] = accum > 0 ? o[q] + y : y;
      }
    }
  }
}

// ---- epilogue: window sum + diagonal/degree terms (kernel.py:86-93,
//      linops.py:43-50) ---------------------------------------------------

constexpr int kTileP = 128;    // pixels per transpose tile
constexpr int kEpiElems = 2048;  // (pixel, rhs) elements per epilogue tile
constexpr int kEpiThreads = 256;
constexpr int kEpiPer = kEpiElems / kEpiThreads;

// Epilogue (kernel.py:86-93, linops.py:43-50) for power-of-two nrhs: a tile
// of TP = 2048/nrhs pixels; the per-window gathers [L][N][nrhs] are read
// coalesced (rhs fastest, 8 independent loads per thread per window), summed,
// transposed through shared memory, and v, eta and the output [nrhs][ld] are
// then accessed rhs-major, also coalesced.
__global__ void __launch_bounds__(kEpiThreads, NLD_EPI_MINB)
k_epilogue_tiled(int kind, int L, int64_t N, int lg_nrhs, const double* __restrict__ v,
                 int64_t ldv, const double* __restrict__ wsum, double* __restrict__ out,
                 int64_t ldo, const double* __restrict__ eta, const double* __restrict__ coef) {
  // rows of TP + 1 (odd stride: conflict-free for the 8-byte accesses); the
  // host routes nrhs <= 256 here, so at most 2048 + 256 doubles
  __shared__ double tile[kEpiElems + 256];
  const int nrhs = 1 << lg_nrhs;
  const int lg_tp = 11 - lg_nrhs;           // TP = 2048 / nrhs
  const int TP = 1 << lg_tp;
  const int64_t ntiles = (N + TP - 1) / TP;
  const int tid = threadIdx.x;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t i0 = tl * TP;
    const int cnt = (int)min((int64_t)TP, N - i0) << lg_nrhs;
    double s[kEpiPer];
#pragma unroll
    for (int k = 0; k < kEpiPer; ++k) s[k] = 0.0;
    for (int w = 0; w < L; ++w) {
      const double* __restrict__ src = wsum + ((int64_t)w * N + i0) * nrhs;
#pragma unroll
      for (int k = 0; k < kEpiPer; ++k) {
        const int e = tid + k * kEpiThreads;
        if (e < cnt) s[k] += src[e];
      }
    }
#pragma unroll
    for (int k = 0; k < kEpiPer; ++k) {
      const int e = tid + k * kEpiThreads;     // e = p * nrhs + r
      const int p = e >> lg_nrhs, r = e & (nrhs - 1);
      tile[r * (TP + 1) + p] = s[k];           // rhs-major, padded rows
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kEpiPer; ++k) {
      const int e = tid + k * kEpiThreads;     // e = r * TP + p
      const int r = e >> lg_tp, p = e & (TP - 1);
      const int64_t i = i0 + p;
      if (i >= N) continue;
      const double x = v[r * ldv + i];
      const double sum = tile[r * (TP + 1) + p];
      double y;
      if (kind == NLD_APPLY_WINDOW_SUM) {
        y = sum;
      } else {
        const double gam = (sum - (double)L * x) / (double)L;
        if (kind == NLD_APPLY_SYSTEM) y = coef[2 * r] * x + coef[2 * r + 1] * (eta[i] * x - gam);
        else if (kind == NLD_APPLY_LAPLACIAN) y = eta[i] * x - gam;
        else y = gam;
      }
      out[r * ldo + i] = y;
    }
    __syncthreads();
  }
}

// generic epilogue (any nrhs; also the dense path where wsum is Gamma v)
__global__ void k_epilogue(int kind, int L, int64_t N, int nrhs, const double* __restrict__ v,
                           int64_t ldv, const double* __restrict__ wsum, int direct,
                           double* __restrict__ out, int64_t ldo,
                           const double* __restrict__ eta, const double* __restrict__ coef) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int r = 0; r < nrhs; ++r) {
      const double x = v[r * ldv + i];
      double gam;
      if (direct) {
        gam = wsum[r * N + i];
      } else {
        double s = 0.0;
        for (int w = 0; w < L; ++w) s += wsum[((int64_t)w * N + i) * nrhs + r];
        if (kind == NLD_APPLY_WINDOW_SUM) {
          out[r * ldo + i] = s;
          continue;
        }
        gam = (s - (double)L * x) / (double)L;
      }
      double y;
      if (kind == NLD_APPLY_SYSTEM) y = coef[2 * r] * x + coef[2 * r + 1] * (eta[i] * x - gam);
      else if (kind == NLD_APPLY_LAPLACIAN) y = eta[i] * x - gam;
      else y = gam;
      out[r * ldo + i] = y;
    }
  }
}

#ifndef NLD_EPI_PM_MINB
#define NLD_EPI_PM_MINB 8
#endif
// pixel-major epilogue: v, out, wout all [.][N][nrhs] -- pure streaming.
// A block is grp = 256 / nrhs pixel groups of nrhs threads (no divisions in
// the element loop).
__global__ void __launch_bounds__(256, NLD_EPI_PM_MINB)
k_epilogue_pm(int kind, int L, int64_t N, int nrhs, const double* __restrict__ v,
              const double* __restrict__ wsum, double* __restrict__ out,
              const double* __restrict__ eta, const double* __restrict__ coef) {
  const int grp = 256 / nrhs;
  const int tid = threadIdx.x;
  if (tid >= grp * nrhs) return;
  const int r = tid % nrhs;
  const int g = tid / nrhs;
  const int64_t total = N * nrhs;
  const double lam = coef ? coef[2 * r] : 0.0, mu = coef ? coef[2 * r + 1] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)grp + g; i < N; i += (int64_t)gridDim.x * grp) {
    const int64_t e = i * nrhs + r;
    double s = 0.0;
#pragma unroll 4
    for (int w = 0; w < L; ++w) s += wsum[(int64_t)w * total + e];
    if (kind == NLD_APPLY_WINDOW_SUM) {
      out[e] = s;
      continue;
    }
    const double x = v[e];
    const double gam = (s - (double)L * x) / (double)L;
    double y;
    if (kind == NLD_APPLY_SYSTEM) y = lam * x + mu * (eta[i] * x - gam);
    else if (kind == NLD_APPLY_LAPLACIAN) y = eta[i] * x - gam;
    else y = gam;
    out[e] = y;
  }
}

// vt [N][nrhs] -> out [nrhs][ldo]
__global__ void __launch_bounds__(256)
k_transpose_out(const double* __restrict__ vt, int64_t N, int nrhs, double* __restrict__ out,
                int64_t ldo) {
  extern __shared__ double tile[];   // [kTileP][nrhs + 1]
  const int ld_t = nrhs + 1;
  const int64_t ntiles = (N + kTileP - 1) / kTileP;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t i0 = tl * kTileP;
    const int np = (int)min((int64_t)kTileP, N - i0);
    for (int e = threadIdx.x; e < np * nrhs; e += blockDim.x) {
      const int p = e / nrhs, r = e - p * nrhs;
      tile[p * ld_t + r] = vt[i0 * nrhs + e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < np * nrhs; e += blockDim.x) {
      const int r = e / np, p = e - r * np;
      out[r * ldo + i0 + p] = tile[p * ld_t + r];
    }
    __syncthreads();
  }
}

// v [nrhs][ld] -> vt [N][nrhs] (pixel-major, for the spread's node gathers)
__global__ void __launch_bounds__(256)
k_transpose_in(const double* __restrict__ v, int64_t ldv, int64_t N, int nrhs,
               double* __restrict__ vt) {
  extern __shared__ double tile[];   // [kTileP][nrhs + 1]
  const int ld_t = nrhs + 1;
  const int64_t ntiles = (N + kTileP - 1) / kTileP;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t i0 = tl * kTileP;
    const int np = (int)min((int64_t)kTileP, N - i0);
    for (int e = threadIdx.x; e < np * nrhs; e += blockDim.x) {
      const int r = e / np, p = e - r * np;
      tile[p * ld_t + r] = v[r * ldv + i0 + p];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < np * nrhs; e += blockDim.x) {
      const int p = e / nrhs, r = e - p * nrhs;
      vt[i0 * nrhs + e] = tile[p * ld_t + r];
    }
    __syncthreads();
  }
}

// ---- dense exact mode (kernel.py:97-114, _kernels.py:205-227) -------------

__global__ void k_dense_apply(const double* __restrict__ F, int64_t N, int D,
                              const int* __restrict__ widx, const int* __restrict__ woff,
                              int L, double inv_s2, const double* __restrict__ v,
                              int64_t ldv, double* __restrict__ out) {
  const int rhs = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t j = 0; j < N; ++j) {
      if (j == i) continue;
      double gsum = 0.0;
      for (int w = 0; w < L; ++w) {
        double r2 = 0.0;
        for (int k = woff[w]; k < woff[w + 1]; ++k) {
          double diff = F[i * D + widx[k]] - F[j * D + widx[k]];
          r2 += diff * diff;
        }
        gsum += exp(-inv_s2 * r2);
      }
      acc += (gsum / (double)L) * v[rhs * ldv + j];
    }
    out[rhs * N + i] = acc;
  }
}

__global__ void k_dense_assemble(const double* __restrict__ F, int64_t N, int D,
                                 const int* __restrict__ widx, const int* __restrict__ woff,
                                 int L, double inv_s2, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * N;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / N, j = e % N;
    double gsum = 0.0;
    if (i != j) {
      for (int w = 0; w < L; ++w) {
        double r2 = 0.0;
        for (int k = woff[w]; k < woff[w + 1]; ++k) {
          double diff = F[i * D + widx[k]] - F[j * D + widx[k]];
          r2 += diff * diff;
        }
        gsum += exp(-inv_s2 * r2);
      }
    }
    out[e] = gsum / (double)L;
  }
}

int grid_blocks(int64_t n, int threads, int cap = 148 * 8) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

// NLD_NO_MMA=1 selects the CUDA-core (DFMA) kernels for the 3-D m=4 shape
// (kept for A/B measurements; both paths are hand-written sm_100a CUDA).
bool use_mma() { return !ab_switch("NLD_NO_MMA", 0); }

// ---- per-window launchers -----------------------------------------------

template <int D, int MC>
void launch_spread(const SubDev* subs, unsigned nsub, const PlanSet& ps, const Workspace& ws,
                   const double* vt, int nrhs, cudaStream_t st) {
  using G = Geo<D, MC>;
  size_t smem = sizeof(double) * G::SMEM;
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(k_spread<D, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  k_spread<D, MC><<<nsub, kSpreadThreads, smem, st>>>(subs, ps.wdev, ps.rows, ps.pix, vt, nrhs,
                                                      ws.blocks);
  NLD_CUDA(cudaGetLastError());
}

template <int D, int MC>
void launch_gather(const SubDev* subs, unsigned nsub, const PlanSet& ps, const Workspace& ws,
                   int64_t N, int nrhs, cudaStream_t st, double* fout = nullptr, int accum = -1) {
  using G = Geo<D, MC>;
  size_t smem = sizeof(double) * G::BLK * std::min(nrhs, G::GRB);
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(k_gather<D, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * G::BLK * G::GRB)));
    attr = true;
  }
  k_gather<D, MC><<<nsub, kThreads, smem, st>>>(subs, ps.cells, ps.wdev, ps.rows, ps.pix,
                                                ws.grid_out, ps.grid_total,
                                                fout ? fout : ws.wout, N, nrhs,
                                                fout ? accum : -1);
  NLD_CUDA(cudaGetLastError());
}

template <int RPW, int NW = mma::kSpWarps>
void launch_spread_mma(const SubDev* subs, unsigned nsub, const PlanSet& ps,
                       const Workspace& ws, const double* vt, int nrhs, cudaStream_t st) {
  const int rpp = std::min(nrhs, NW * RPW);
  const size_t smem = sizeof(double) * mma::spread_smem(rpp);
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(mma::k_spread_mma<RPW, NW>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double) * mma::spread_smem(NW * RPW))));
    attr = true;
  }
  mma::k_spread_mma<RPW, NW><<<nsub, 32 * NW, smem, st>>>(subs, ps.wdev, ps.rows, ps.pix, vt,
                                                          nrhs, ws.blocks);
  NLD_CUDA(cudaGetLastError());
}

static void launch_spread_bc(const SubDev* subs, unsigned nsub, const PlanSet& ps,
                             const Workspace& ws, const double* vt, int nrhs, cudaStream_t st) {
  const size_t smem = sizeof(double) * mma::spread_bc_smem();
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(mma::k_spread_bc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr = true;
  }
  mma::k_spread_bc<<<nsub, 256, smem, st>>>(subs, ps.wdev, ps.rows, ps.pix, vt, nrhs, ws.blocks);
  NLD_CUDA(cudaGetLastError());
}

void launch_gather_mma(const SubDev* subs, unsigned nsub, const PlanSet& ps,
                       const Workspace& ws, int64_t N, int nrhs, cudaStream_t st,
                       const mma::GatherEpi& ep, double* out) {
  if (nrhs >= 8) {
    const size_t smem16 = sizeof(double) * 16 * mma::kGRow;
    static bool attr16 = false;
    if (!attr16) {
      NLD_CUDA(cudaFuncSetAttribute(mma::k_gather_mma16,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem16));
      attr16 = true;
    }
    mma::k_gather_mma16<<<nsub, mma::kGaThreads, smem16, st>>>(
        subs, ps.cells, ps.wdev, ps.rows, ps.pix, ws.grid_out, ps.grid_total,
        ep.mode == mma::kGatherStore ? ws.wout : out, N, nrhs, ep);
  } else {
    const size_t smem = sizeof(double) * mma::kBlk * std::min(nrhs, mma::kGaRhs);
    static bool attr = false;
    if (!attr) {
      NLD_CUDA(cudaFuncSetAttribute(mma::k_gather_mma,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(sizeof(double) * mma::kBlk * mma::kGaRhs)));
      attr = true;
    }
    mma::k_gather_mma<<<nsub, mma::kGaThreads, smem, st>>>(
        subs, ps.cells, ps.wdev, ps.rows, ps.pix, ws.grid_out, ps.grid_total, ws.wout, N, nrhs);
  }
  NLD_CUDA(cudaGetLastError());
}

template <int MC>
void spread_window_fast(const PlanSet& ps, const Workspace& ws, int w, const double* vt,
                        int nrhs, cudaStream_t st) {
  const WinPlan& wp = ps.win[w];
  if (!ps.wdev_h[w].fast || wp.n_subs == 0) return;
  const SubDev* subs = ps.subs[wp.d] + wp.sub_off;
  const unsigned nsub = (unsigned)wp.n_subs;
  if (wp.d == 1) {
    launch_spread<1, MC>(subs, nsub, ps, ws, vt, nrhs, st);
  } else if (wp.d == 2) {
    launch_spread<2, MC>(subs, nsub, ps, ws, vt, nrhs, st);
  } else if (MC == 4 && use_mma()) {
    const int rpw4 = ab_switch("NLD_SPREAD_RPW4", 0);
    const int bc = ab_switch("NLD_SPREAD_BC", 1);   // shared (B (x) C) DMMA spread
    if (use_ozaki() && nrhs % 16 == 0 && ps.oz_ok && ps.sub_exp && ps.sub_order &&
        !ab_switch("NLD_OZAKI_NO_SPREAD", 0)) {
      launch_spread_oz(ps, subs, ps.sub_exp + wp.sub_off * 24, nsub,
                       ws.vmax, vt, nrhs, ws.blocks, st, ps.sub_order + wp.sub_off);
    }
    else if (bc && nrhs % 16 == 0 && ((uintptr_t)vt & 15) == 0)
      launch_spread_bc(subs, nsub, ps, ws, vt, nrhs, st);
    else if (nrhs >= 16 && rpw4) launch_spread_mma<4, 4>(subs, nsub, ps, ws, vt, nrhs, st);
    else if (nrhs >= 16) launch_spread_mma<2>(subs, nsub, ps, ws, vt, nrhs, st);
    else launch_spread_mma<1>(subs, nsub, ps, ws, vt, nrhs, st);
  } else {
    launch_spread<3, MC>(subs, nsub, ps, ws, vt, nrhs, st);
  }
}

// window w's gather runs on the integer-sliced tcgen05 kernel (3-D, m = 4,
// 16k rhs; the caller checks the cutoff)
static bool sliced_gather(const PlanSet& ps, const Workspace& ws, int w, int nrhs) {
  const WinPlan& wp = ps.win[w];
  return ps.wdev_h[w].fast && wp.d == 3 && wp.n_subs > 0 && use_ozaki() && nrhs % 16 == 0 &&
         nrhs <= 256 && ps.oz_ok && ws.gdig && !ab_switch("NLD_OZAKI_NO_GATHER", 0) &&
         w < (int)ps.gcell_n.size() && ps.gcell_n[w] > 0;
}

template <int MC>
void gather_window_fast(const PlanSet& ps, const Workspace& ws, int w, int64_t N, int nrhs,
                        cudaStream_t st, const mma::GatherEpi& ep, double* out) {
  const WinPlan& wp = ps.win[w];
  if (!ps.wdev_h[w].fast || wp.n_subs == 0) return;
  const SubDev* subs = ps.subs[wp.d] + wp.sub_off;
  const unsigned nsub = (unsigned)wp.n_subs;
  // fused product (ep.mode != kGatherStore): 1-/2-D windows run before the
  // 3-D ones and store (first) or add into the running window sum `out`
  double* fout = ep.mode == mma::kGatherStore ? nullptr : out;
  const int acc = ep.mode == mma::kGatherFirst ? 0 : 1;
  if (wp.d == 1) launch_gather<1, MC>(subs, nsub, ps, ws, N, nrhs, st, fout, acc);
  else if (wp.d == 2) launch_gather<2, MC>(subs, nsub, ps, ws, N, nrhs, st, fout, acc);
  else if (MC == 4 && sliced_gather(ps, ws, w, nrhs))
    launch_gather_nm(ps, subs, ps.sub_exp + wp.sub_off * 24, ps.sub_order + wp.sub_off,
                     nsub, ws.grid_out, ps.grid_total,
                     ep.mode == mma::kGatherStore ? ws.wout + (int64_t)w * N * nrhs : out, nrhs,
                     ep, st, ws.gdig, ps.gcell_lo[w], ps.gcell_n[w], ws.gdig_on_aux);
  else if (MC == 4 && use_mma()) launch_gather_mma(subs, nsub, ps, ws, N, nrhs, st, ep, out);
  else launch_gather<3, MC>(subs, nsub, ps, ws, N, nrhs, st);
}

struct EvScope {
  nld_operator* op;
  cudaStream_t st;
  int idx = 0;
  EvScope(nld_operator* o, cudaStream_t s) : op(o), st(s) {}
  void mark() {
    if (op->timing && op->events) cudaEventRecord(op->ev[idx++], st);
  }
};

}  // namespace

void ensure_workspace(nld_operator* op, const PlanSet& ps, int nrhs) {
  Workspace& ws = op->ws;
  // the sliced gather's per-cell G digits exist only where that path runs
  // (m = 4; 16k-rhs batches): other cutoffs neither allocate nor re-check them
  const int64_t nc_need = std::max(ps.n_cells, std::max(op->sets[0].n_cells, op->sets[1].n_cells));
  const bool oz_shape = use_ozaki() && op->params.cutoff == 4 && nc_need > 0;
  const bool need_gdig = oz_shape && nrhs % 16 == 0;
  if (ws.nrhs_cap >= nrhs && ws.grid_total >= ps.grid_total &&
      ws.blocks_total >= ps.blocks_total && (!need_gdig || ws.gdig_cells >= ps.n_cells))
    return;
  double* keep_cg = ws.cg;
  int64_t keep_cap = ws.cg_cap;
  ws.cg = nullptr;
  free_workspace(ws);
  ws.cg = keep_cg;
  ws.cg_cap = keep_cap;
  int cap = std::max(nrhs, 1);
  int64_t gt = std::max(ps.grid_total, std::max(op->sets[0].grid_total, op->sets[1].grid_total));
  int64_t bt = std::max(ps.blocks_total, std::max(op->sets[0].blocks_total, op->sets[1].blocks_total));
  NLD_CUDA(cudaMalloc(&ws.blocks, sizeof(double) * std::max<int64_t>(1, bt) * cap));
  // + one flag per rhs after the grids (non-finite rhs, summed with the grids
  // by the shard allreduce; see k_vmax / k_poison)
  NLD_CUDA(cudaMalloc(&ws.grid_in, sizeof(double) * (std::max<int64_t>(1, gt) * cap + cap)));
  NLD_CUDA(cudaMalloc(&ws.grid_out, sizeof(double) * std::max<int64_t>(1, gt) * cap));
  NLD_CUDA(cudaMalloc(&ws.cbuf0, sizeof(double2) * std::max<int64_t>(1, gt) * cap));
  NLD_CUDA(cudaMalloc(&ws.cbuf1, sizeof(double2) * std::max<int64_t>(1, gt) * cap));
  NLD_CUDA(cudaMalloc(&ws.cbuf2, sizeof(double2) * std::max<int64_t>(1, gt) * cap));
  NLD_CUDA(cudaMalloc(&ws.cbuf3, sizeof(double2) * std::max<int64_t>(1, gt) * cap));
  NLD_CUDA(cudaMalloc(&ws.wout, sizeof(double) * std::max<int64_t>(1, op->N * op->L) * cap));
  NLD_CUDA(cudaMalloc(&ws.vt, sizeof(double) * std::max<int64_t>(1, op->N) * cap));
  NLD_CUDA(cudaMalloc(&ws.coef, sizeof(double) * 2 * cap));
  NLD_CUDA(cudaMalloc(&ws.vmax, sizeof(unsigned long long) * cap));
  {
    // separable-assemble scratch: the largest 3-D box x 64 offsets x nrhs
    int64_t mb = 0;
    for (int k = 0; k < 2; ++k)
      for (const auto& w : op->sets[k].wdev_h)
        if (w.d == 3) mb = std::max(mb, w.box_size);
    for (const auto& w : ps.wdev_h)
      if (w.d == 3) mb = std::max(mb, w.box_size);
    ws.asm_cap = mb * 64 * cap;
    if (ws.asm_cap) {
      NLD_CUDA(cudaMalloc(&ws.asm_y2, sizeof(double) * (ws.asm_cap / 8 + 1)));
      NLD_CUDA(cudaMalloc(&ws.asm_y2b, sizeof(double) * (ws.asm_cap / 8 + 1)));
    }
  }
  {
    // sliced gather: G digits of every cell and 16-rhs group, rebuilt per product
    if (oz_shape && cap >= 16) {
      NLD_CUDA(cudaMalloc(&ws.gdig, (size_t)gather_gdig_bytes() * nc_need * (cap / 16)));
      ws.gdig_cells = nc_need;
    }
  }
  ws.nrhs_cap = cap;
  ws.grid_total = gt;
  ws.blocks_total = bt;
}

void free_workspace(Workspace& ws) {
  cudaFree(ws.asm_y2);
  cudaFree(ws.asm_y2b);
  cudaFree(ws.cbuf2);
  cudaFree(ws.cbuf3);
  cudaFree(ws.cg);
  cudaFree(ws.blocks);
  cudaFree(ws.grid_in);
  cudaFree(ws.grid_out);
  cudaFree(ws.cbuf0);
  cudaFree(ws.cbuf1);
  cudaFree(ws.wout);
  cudaFree(ws.vt);
  cudaFree(ws.coef);
  cudaFree(ws.vmax);
  cudaFree(ws.gdig);
  ws = Workspace();
}

// ---- per-window stages ------------------------------------------------------

// spread of window w (block path) -- main stream
static void spread_window(nld_operator* op, const PlanSet& ps, int w, const double* vt,
                          int nrhs, cudaStream_t st) {
  switch (op->params.cutoff) {
    case 3: spread_window_fast<3>(ps, op->ws, w, vt, nrhs, st); break;
    case 4: spread_window_fast<4>(ps, op->ws, w, vt, nrhs, st); break;
    case 5: spread_window_fast<5>(ps, op->ws, w, vt, nrhs, st); break;
    default: break;
  }
}

// assemble of window w + its generic/edge atomics (writes ws.grid_in)
static void assemble_window(nld_operator* op, const PlanSet& ps, int w, const double* vt,
                            int nrhs, cudaStream_t st, int set = 0) {
  Workspace& ws = op->ws;
  double* const y2 = set ? ws.asm_y2b : ws.asm_y2;
  const WinDev& wd = ps.wdev_h[w];
  const WinPlan& wp = ps.win[w];
  const int64_t y1n = wd.box_size * 64 * nrhs;
  if (wd.fast && wd.d == 3 && wd.S == 8 && !wd.wrap && ws.asm_cap >= y1n) {
    const int lines_per_cta = 8 * nrhs >= 128 ? 1 : 128 / (8 * nrhs);
    k_asm_p12<<<(int)std::min<int64_t>((wd.box_size + lines_per_cta - 1) / lines_per_cta, 148 * 64), 128,
                0, st>>>(ps.wdev, w, ps.cellinfo, ws.blocks, nrhs, y2);
    k_asm_p3<<<grid_blocks(y1n / 64, 256, 148 * 32), 256, 0, st>>>(ps.wdev, w, y2, nrhs,
                                                                   ws.grid_in, ps.grid_total);
  } else {
    dim3 grid(grid_blocks(wd.box_size * nrhs, 32, 148 * 16), 1);
    k_assemble<<<grid, 256, 0, st>>>(ps.wdev, w, ps.cellinfo, ws.blocks, nrhs, ws.grid_in,
                                     ps.grid_total);
  }
  NLD_CUDA(cudaGetLastError());
  if (!wd.fast) {
    dim3 g2(grid_blocks(op->N, 256), nrhs);
    k_spread_generic<<<g2, 256, 0, st>>>(ps.wdev, w, ps.rows, ps.pix, ps.key, vt, nrhs,
                                         ws.grid_in, ps.grid_total, op->N);
    NLD_CUDA(cudaGetLastError());
  }
  if (wp.n_edge) {
    dim3 g3(grid_blocks(wp.n_edge, 128), nrhs);
    k_spread_edges<<<g3, 128, 0, st>>>(ps.edges + wp.edge_off, wp.n_edge, ps.wdev, vt, nrhs,
                                       ws.grid_in, ps.grid_total);
    NLD_CUDA(cudaGetLastError());
  }
}

// 3-D windows whose slab fits the default shared-memory limit take the fused
// first two passes (k_conv01)
static bool conv_fused01(const WinDev& wd) {
  return wd.d == 3 && conv01_smem(wd.box_w[1], wd.box_w[2]) <= 48 * 1024 && wd.box_w[0] <= 65535;
}

// separable convolution of window w: grid_in -> grid_out
static void conv_window(nld_operator* op, const PlanSet& ps, int w, int nrhs, cudaStream_t st,
                        int set = 0) {
  Workspace& ws = op->ws;
  double2* const b0 = set ? ws.cbuf2 : ws.cbuf0;
  double2* const b1 = set ? ws.cbuf3 : ws.cbuf1;
  const WinDev& wd = ps.wdev_h[w];
  int pass0 = 0;
  if (conv_fused01(wd)) {
    // axes 2 and 1 in one kernel (writes the buffer pass 2 reads)
    k_conv01<<<dim3(wd.box_w[0], nrhs), 256, conv01_smem(wd.box_w[1], wd.box_w[2]), st>>>(
        ps.wdev, w, ps.K, ws.grid_in, b1, ps.grid_total);
    NLD_CUDA(cudaGetLastError());
    pass0 = 2;
  }
  for (int pass = pass0; pass < wd.d; ++pass) {
    dim3 grid(grid_blocks(wd.box_size, 128, 1024), 1, nrhs);
    const double2* cin = (pass % 2 == 1) ? b0 : b1;
    double2* cout = (pass % 2 == 0) ? b0 : b1;
    k_conv<<<grid, 128, 0, st>>>(ps.wdev, w, pass, ps.K, ws.grid_in, cin, cout, ws.grid_out,
                                 ps.grid_total);
    NLD_CUDA(cudaGetLastError());
  }
}

// gather of window w from ws.grid_out into ws.wout (+ generic/edges), or --
// fused (ep->mode != kGatherStore, only fast d=3 m=4 windows, nrhs >= 8) --
// accumulated into out with the epilogue applied by the last window.  The
// edge corrections (+=) of the last window run before its fast gather so the
// final formula sees the complete window sum.
static void gather_window(nld_operator* op, const PlanSet& ps, int w, int nrhs,
                          cudaStream_t st, const mma::GatherEpi* ep = nullptr,
                          double* out = nullptr) {
  Workspace& ws = op->ws;
  const int64_t N = op->N;
  const WinDev& wd = ps.wdev_h[w];
  const WinPlan& wp = ps.win[w];
  mma::GatherEpi store{mma::kGatherStore, 0, 0, nullptr, nullptr, nullptr};
  const mma::GatherEpi& e = ep ? *ep : store;
  double* edge_out = ep ? out : ws.wout;
  const int64_t edge_stride = ep ? 0 : N;
  auto edges = [&]() {
    if (!wp.n_edge) return;
    dim3 grid(grid_blocks(wp.n_edge, 128), nrhs);
    k_gather_edges<<<grid, 128, 0, st>>>(ps.edges + wp.edge_off, wp.n_edge, ps.wdev,
                                         ws.grid_out, ps.grid_total, edge_out, edge_stride, nrhs);
    NLD_CUDA(cudaGetLastError());
  };
  if (e.mode == mma::kGatherFinal) edges();
  switch (op->params.cutoff) {
    case 3: gather_window_fast<3>(ps, ws, w, N, nrhs, st, e, out); break;
    case 4: gather_window_fast<4>(ps, ws, w, N, nrhs, st, e, out); break;
    case 5: gather_window_fast<5>(ps, ws, w, N, nrhs, st, e, out); break;
    default: break;
  }
  if (!wd.fast) {
    dim3 grid(grid_blocks(N, 256), nrhs);
    k_gather_generic<<<grid, 256, 0, st>>>(ps.wdev, w, nrhs, ps.rows, ps.pix, ps.key,
                                           ws.grid_out, ps.grid_total, ws.wout, N);
    NLD_CUDA(cudaGetLastError());
  }
  if (e.mode != mma::kGatherFinal) edges();
}

// window w's slice of the support-box grids [nrhs][grid_ld] <-> a contiguous
// [nrhs][box] buffer (+ `extra` trailing values), for a per-window allreduce
__global__ void k_pack_win(const double* __restrict__ grid, int64_t grid_ld, int64_t off,
                           int64_t box, int nrhs, const double* __restrict__ extra, int n_extra,
                           double* __restrict__ buf) {
  const int64_t total = box * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total + n_extra;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < total) {
      const int64_t r = e / box, f = e - r * box;
      buf[e] = grid[r * grid_ld + off + f];
    } else {
      buf[e] = extra[e - total];
    }
  }
}
__global__ void k_unpack_win(const double* __restrict__ buf, int64_t grid_ld, int64_t off,
                             int64_t box, int nrhs, double* __restrict__ extra, int n_extra,
                             double* __restrict__ grid) {
  const int64_t total = box * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total + n_extra;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < total) {
      const int64_t r = e / box, f = e - r * box;
      grid[r * grid_ld + off + f] = buf[e];
    } else {
      extra[e - total] = buf[e];
    }
  }
}

// the shard allreduce of window w's grids alone (so it can run on the aux
// stream behind that window's assemble while the main stream spreads the
// next window): packed into the convolution scratch, summed, unpacked; the
// last window also carries the per-rhs non-finite flags
static void comm_window(nld_operator* op, const PlanSet& ps, int w, int nrhs, bool flags,
                        cudaStream_t st, int set = 0) {
  if (!op->comm) return;
  Workspace& ws = op->ws;
  const WinDev& wd = ps.wdev_h[w];
  double* extra = ws.grid_in + ps.grid_total * nrhs;
  const int ne = flags ? nrhs : 0;
  double* buf = reinterpret_cast<double*>(set ? ws.cbuf2 : ws.cbuf0);
  const int64_t cnt = wd.box_size * nrhs + ne;
  k_pack_win<<<grid_blocks(cnt, 256, 148 * 8), 256, 0, st>>>(ws.grid_in, ps.grid_total,
                                                             wd.grid_off, wd.box_size, nrhs,
                                                             extra, ne, buf);
  NLD_CUDA(cudaGetLastError());
  comm_device(op, buf, cnt, st);
  k_unpack_win<<<grid_blocks(cnt, 256, 148 * 8), 256, 0, st>>>(buf, ps.grid_total, wd.grid_off,
                                                               wd.box_size, nrhs, extra, ne,
                                                               ws.grid_in);
  NLD_CUDA(cudaGetLastError());
}

// spread of all windows into the support boxes ws.grid_in [nrhs][grid_total]
// (+ the shard allreduce).  vt: right-hand sides pixel-major [N][nrhs].
int spread_stage(nld_operator* op, const PlanSet& ps, const double* vt, int nrhs,
                 cudaStream_t st, bool flags) {
  const int L = (int)ps.wdev_h.size();
  for (int w = 0; w < L; ++w) spread_window(op, ps, w, vt, nrhs, st);
  for (int w = 0; w < L; ++w) assemble_window(op, ps, w, vt, nrhs, st);
  // the non-finite flags ride behind the grids in the same allreduce
  comm_device(op, op->ws.grid_in, ps.grid_total * nrhs + (flags ? nrhs : 0), st);
  return 2 * L;
}

int gather_stage(nld_operator* op, const PlanSet& ps, int nrhs, cudaStream_t st) {
  const int L = (int)ps.wdev_h.size();
  for (int w = 0; w < L; ++w) gather_window(op, ps, w, nrhs, st);
  return L;
}

static void ensure_aux(nld_operator* op, int L) {
  if (op->aux && op->aux_windows >= L) return;
  if (!op->aux) {
    NLD_CUDA(cudaStreamCreateWithFlags(&op->aux, cudaStreamNonBlocking));
    NLD_CUDA(cudaStreamCreateWithFlags(&op->aux2, cudaStreamNonBlocking));
    NLD_CUDA(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming));
    NLD_CUDA(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming));
  }
  for (int w = op->aux_windows; w < L; ++w) {
    NLD_CUDA(cudaEventCreateWithFlags(&op->ev_spread[w], cudaEventDisableTiming));
    NLD_CUDA(cudaEventCreateWithFlags(&op->ev_conv[w], cudaEventDisableTiming));
  }
  op->aux_windows = L;
}

void to_pixel_major(const double* v, int64_t ldv, int64_t n, int nrhs, double* vt,
                    cudaStream_t st) {
  k_transpose_in<<<grid_blocks(n, kTileP, 148 * 16), 256,
                   sizeof(double) * kTileP * (nrhs + 1), st>>>(v, ldv, n, nrhs, vt);
  NLD_CUDA(cudaGetLastError());
}

void to_rhs_major(const double* vt, int64_t n, int nrhs, double* out, int64_t ldo,
                  cudaStream_t st) {
  k_transpose_out<<<grid_blocks(n, kTileP, 148 * 16), 256,
                    sizeof(double) * kTileP * (nrhs + 1), st>>>(vt, n, nrhs, out, ldo);
  NLD_CUDA(cudaGetLastError());
}

void apply_op(nld_operator* op, int which, int kind, const double* v, double* out,
              int nrhs, int64_t ld, const double* coef_dev, const double* eta,
              cudaStream_t st, int pixel_major, const unsigned long long* vmax_pre,
              const double* flag_pre) {
  const PlanSet& ps = op->sets[which];
  ensure_workspace(op, ps, nrhs);
  if (use_ozaki() && op->params.cutoff == 4)
    ozaki_exponents(op->sets[which], op->params.no_sliced == 0, st);
  Workspace& ws = op->ws;
  const int64_t N = op->N;
  const int L = op->L;
  EvScope ev(op, st);
  ev.mark();
  int launches = 0;
  // 0. pixel-major copy of the rhs for the node gathers
  const double* vt = v;
  if (!pixel_major && (nrhs > 1 || ld != N)) {
    to_pixel_major(v, ld, N, nrhs, ws.vt, st);
    vt = ws.vt;
    ++launches;
  }
  const bool sliced = use_ozaki() && op->params.cutoff == 4 && nrhs % 16 == 0;
  double* const flags = ws.grid_in + ps.grid_total * nrhs;
  if (sliced && vmax_pre && vt == v) {
    // the caller's kernel that wrote v also took its per-rhs max |v| and
    // non-finite flags (CG: the direction update), saving k_vmax's pass
    NLD_CUDA(cudaMemcpyAsync(ws.vmax, vmax_pre, sizeof(unsigned long long) * nrhs,
                             cudaMemcpyDeviceToDevice, st));
    NLD_CUDA(cudaMemcpyAsync(flags, flag_pre, sizeof(double) * nrhs, cudaMemcpyDeviceToDevice,
                             st));
  } else if (sliced) {
    ozaki_vmax(vt, N, nrhs, ws.vmax, flags, st);
    launches += 1;   // k_vmax (its resets are memsets, not kernels)
  }
  const int no_overlap = ab_switch("NLD_NO_OVERLAP", 0);
  const bool overlap = L <= 16 && !no_overlap;
  // fused gather epilogue (see gather_window): every window on the DMMA
  // gather, pixel-major in/out, out not aliasing v
  const int no_fuse = ab_switch("NLD_NO_FUSED_EPILOGUE", 0);
  // (the sliced gather reads and writes the caller's v / out lines with
  // 32-byte accesses: unaligned buffers take the unfused path through the
  // aligned workspace)
  const bool al32 = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(v)) & 31) == 0;
  bool fused = !no_fuse && pixel_major && nrhs >= 8 && L >= 2 && out != v && al32 &&
               op->params.cutoff == 4 && use_mma();
  // gather order: 1-/2-D windows first, then the 3-D ones (the last of which
  // applies the epilogue); every window on a fast path with subproblems
  std::vector<int> gorder;
  int n3 = 0;
  for (int w = 0; w < L && fused; ++w) {
    const WinDev& wd = ps.wdev_h[w];
    fused = wd.fast && ps.win[w].n_subs > 0;
    if (wd.d != 3) gorder.push_back(w);
    else ++n3;
  }
  fused = fused && n3 > 0;
  for (int w = 0; w < L; ++w)
    if (ps.wdev_h[w].d == 3) gorder.push_back(w);
  if (!fused) {
    gorder.resize(L);
    for (int w = 0; w < L; ++w) gorder[w] = w;
  }
  auto gather_k = [&](int k) {   // the k-th window in gather order
    const int w = gorder[k];
    if (!fused) {
      gather_window(op, ps, w, nrhs, st);
      return;
    }
    mma::GatherEpi ep{k == 0 ? mma::kGatherFirst
                             : (k == L - 1 ? mma::kGatherFinal : mma::kGatherAccum),
                      kind, L, v, eta, coef_dev};
    gather_window(op, ps, w, nrhs, st, &ep, out);
  };
#ifndef NLD_GDIG_AUX
#define NLD_GDIG_AUX 1
#endif
  const bool gdig_aux = NLD_GDIG_AUX && overlap && op->params.cutoff == 4;
  ws.gdig_on_aux = gdig_aux;
  if (overlap) {
    // window w's assemble + convolution (latency / L2 bound) run on the aux
    // stream while the main stream spreads window w+1 and, later, gathers
    // the earlier windows (fp64 tensor bound)
    ensure_aux(op, L);
    for (int w = 0; w < L; ++w) {
      spread_window(op, ps, w, vt, nrhs, st);
      NLD_CUDA(cudaEventRecord(op->ev_spread[w], st));
      // windows alternate between two aux streams (own scratch each): with
      // many small windows (c2: eight 3-D) one stream's assemble chain was
      // slower than the spreads it overlaps
      const int set = w & 1;
      cudaStream_t ax = set ? op->aux2 : op->aux;
      NLD_CUDA(cudaStreamWaitEvent(ax, op->ev_spread[w], 0));
      assemble_window(op, ps, w, vt, nrhs, ax, set);
      comm_window(op, ps, w, nrhs, sliced && w == L - 1, ax, set);
      conv_window(op, ps, w, nrhs, ax, set);
      // the window's G digits too (they depend only on its convolved grid):
      // off the main stream, which spreads and gathers meanwhile
      if (gdig_aux && sliced_gather(ps, ws, w, nrhs))
        launch_gdig_nm(ps, ws.grid_out, ps.grid_total, nrhs, ws.gdig, ps.gcell_lo[w],
                       ps.gcell_n[w], ax);
      NLD_CUDA(cudaEventRecord(op->ev_conv[w], ax));
    }
    ev.mark();
    NLD_CUDA(cudaStreamWaitEvent(st, op->ev_conv[gorder[0]], 0));
    ev.mark();
    ev.mark();
    for (int k = 0; k < L; ++k) {
      if (k > 0) NLD_CUDA(cudaStreamWaitEvent(st, op->ev_conv[gorder[k]], 0));
      gather_k(k);
    }
  } else {
    spread_stage(op, ps, vt, nrhs, st, sliced);
    ev.mark();
    ev.mark();
    for (int w = 0; w < L; ++w) conv_window(op, ps, w, nrhs, st);
    ev.mark();
    for (int k = 0; k < L; ++k) gather_k(k);
  }
  for (int w = 0; w < L; ++w) {
    // spread + gather (+ the sliced gather's per-cell G digits), assemble
    // (two kernels for 3-D m = 4 boxes: k_asm_p12, k_asm_p3), d convolution passes
    // (two kernels for 3-D windows: k_conv01 + the axis-0 pass),
    // generic-path and edge-node kernels
    const WinDev& wd = ps.wdev_h[w];
    const bool fastw = wd.fast && ps.win[w].n_subs;
    const bool asm3 = wd.fast && wd.d == 3 && wd.S == 8 && !wd.wrap;
    launches += (fastw ? 2 : 0) + (fastw && sliced && wd.d == 3 && ws.gdig ? 1 : 0) +
                (asm3 ? 2 : 1) + (conv_fused01(wd) ? 2 : wd.d) + (wd.fast ? 0 : 2) + (ps.win[w].n_edge ? 2 : 0);
  }
  ev.mark();
  // 5. epilogue
  {
    int lg = -1;
    for (int k = 0; k <= 8; ++k)
      if ((1 << k) == nrhs) lg = k;
    if (fused) {
      // done inside the last window's gather
    } else if ((pixel_major || nrhs == 1) && nrhs <= 256) {
      k_epilogue_pm<<<grid_blocks(N, 256 / nrhs, 148 * 16), 256, 0, st>>>(
          kind, L, N, nrhs, v, ws.wout, out, eta, coef_dev);
    } else if (lg >= 0) {
      const int tp = 2048 >> lg;
      k_epilogue_tiled<<<grid_blocks(N, tp, 148 * 8), kEpiThreads, 0, st>>>(
          kind, L, N, lg, v, ld, ws.wout, out, ld, eta, coef_dev);
    } else {
      k_epilogue<<<grid_blocks(N, 256, 148 * 16), 256, 0, st>>>(kind, L, N, nrhs, v, ld, ws.wout,
                                                                 0, out, ld, eta, coef_dev);
    }
    NLD_CUDA(cudaGetLastError());
    if (!fused) ++launches;
  }
  if (sliced) {
    // NaN into the columns of non-finite right-hand sides (a no-op otherwise)
    ozaki_poison(flags, nrhs, out, N, ld, pixel_major || nrhs == 1, st);
    ++launches;
  }
  ev.mark();
  ws.gdig_on_aux = false;
  op->stats.launches = launches;
}

static void dense_tables(nld_operator* op, int** widx, int** woff, cudaStream_t st) {
  NLD_CUDA(cudaMallocAsync(widx, sizeof(int) * op->win_index.size(), st));
  NLD_CUDA(cudaMallocAsync(woff, sizeof(int) * op->win_offset.size(), st));
  NLD_CUDA(cudaMemcpyAsync(*widx, op->win_index.data(), sizeof(int) * op->win_index.size(),
                           cudaMemcpyHostToDevice, st));
  NLD_CUDA(cudaMemcpyAsync(*woff, op->win_offset.data(), sizeof(int) * op->win_offset.size(),
                           cudaMemcpyHostToDevice, st));
}

void dense_apply(nld_operator* op, int which, int kind, const double* v, double* out,
                 int nrhs, int64_t ld, const double* coef_dev, const double* eta,
                 cudaStream_t st, int pixel_major) {
  if (pixel_major && nrhs > 1) {
    // exact mode is desk-scale: go through an rhs-major copy
    double *vr = nullptr, *orr = nullptr;
    NLD_CUDA(cudaMallocAsync(&vr, sizeof(double) * op->N * nrhs, st));
    NLD_CUDA(cudaMallocAsync(&orr, sizeof(double) * op->N * nrhs, st));
    to_rhs_major(v, op->N, nrhs, vr, op->N, st);
    dense_apply(op, which, kind, vr, orr, nrhs, op->N, coef_dev, eta, st, 0);
    to_pixel_major(orr, op->N, op->N, nrhs, out, st);
    cudaFreeAsync(vr, st);
    cudaFreeAsync(orr, st);
    return;
  }
  if (op->N > op->params.dense_limit)
    throw Error(NLD_ERR_DENSE_LIMIT, "dense assembly of " + std::to_string(op->N) +
                                         " nodes exceeds the limit " +
                                         std::to_string(op->params.dense_limit));
  int *widx = nullptr, *woff = nullptr;
  dense_tables(op, &widx, &woff, st);
  double* gam = nullptr;
  NLD_CUDA(cudaMallocAsync(&gam, sizeof(double) * op->N * nrhs, st));
  double inv = (which ? 2.0 : 1.0) / (op->sigma * op->sigma);
  dim3 grid(grid_blocks(op->N, 128), nrhs);
  k_dense_apply<<<grid, 128, 0, st>>>(op->feats, op->N, op->D, widx, woff, op->L, inv, v, ld,
                                      gam);
  NLD_CUDA(cudaGetLastError());
  k_epilogue<<<grid_blocks(op->N, 256), 256, 0, st>>>(kind, op->L, op->N, nrhs, v, ld, gam, 1,
                                                       out, ld, eta, coef_dev);
  NLD_CUDA(cudaGetLastError());
  cudaFreeAsync(gam, st);
  cudaFreeAsync(widx, st);
  cudaFreeAsync(woff, st);
}

void dense_assemble(nld_operator* op, int which, double* out, cudaStream_t st) {
  if (op->N > op->params.dense_limit)
    throw Error(NLD_ERR_DENSE_LIMIT, "dense assembly of " + std::to_string(op->N) +
                                         " nodes exceeds the limit " +
                                         std::to_string(op->params.dense_limit));
  int *widx = nullptr, *woff = nullptr;
  dense_tables(op, &widx, &woff, st);
  double inv = (which ? 2.0 : 1.0) / (op->sigma * op->sigma);
  k_dense_assemble<<<grid_blocks(op->N * op->N, 256, 148 * 32), 256, 0, st>>>(
      op->feats, op->N, op->D, widx, woff, op->L, inv, out);
  NLD_CUDA(cudaGetLastError());
  cudaFreeAsync(widx, st);
  cudaFreeAsync(woff, st);
}

}  // namespace nld
