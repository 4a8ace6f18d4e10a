// fp64 tensor-core (DMMA, mma.sync.m8n8k4.f64) spread and gather for 3-D
// windows with cutoff m = 4 (an 8x8x8 stencil block) -- the BASELINE shape.
//
// Measured on B200: DMMA m8n8k4 sustains 37.06 TFLOP/s (the full fp64 rate)
// against 34 TFLOP/s for a DFMA loop, and it takes its operands from
// registers, which removes the shared-memory broadcast traffic that capped
// the CUDA-core kernels at ~50% of the fp64 pipe.
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64), g = lane >> 2, t = lane & 3:
//   A (8x4 row)  : A[g][t]          B (4x8 col) : B[t][g]
//   C/D (8x8)    : C[g][2t + i], i = 0, 1
//
// spread: block[a][(b,c)] += sum_j (v_j A_j[a]) (B_j[b] C_j[c])
//         M = 8 (a), N = 64 (b,c) as 8 n-tiles (one per b), K = nodes.
// gather: T[(a,b)][j] = sum_c G[a][b][c] C_j[c]   (M = 64 as 8 m-tiles, one
//         per a; K = 8; N = 8 nodes), then y_j = sum_a A_j[a] B_j[b] T[a,b][j]
//         reduced over b across the 8 lanes of a column.
#pragma once

#include "nld_internal.cuh"
#include "nld_epi.cuh"

#ifndef NLD_SPREAD_UNROLL
#define NLD_SPREAD_UNROLL 2
#endif
#ifndef NLD_SPREAD_MINB
#define NLD_SPREAD_MINB 2
#endif
#ifndef NLD_EPI_MINB
#define NLD_EPI_MINB 4
#endif

namespace nld {
namespace mma {

#ifdef NLD_DMMA_NV
#define NLD_DMMA_ASM asm
#else
#define NLD_DMMA_ASM asm volatile
#endif
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  NLD_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr(dst)), "l"(src));
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_addr(dst)), "l"(src));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kSpUnroll = NLD_SPREAD_UNROLL;
constexpr int kS = 8;             // stencil width 2m
constexpr int kRow = 24;          // global row: [A(8)][B(8)][C(8)]
constexpr int kSRow = 28;         // smem row stride: 16B aligned, conflict-free row[g]
constexpr int kBlk = 512;
constexpr int kSpWarps = 8;
constexpr int kSpThreads = 256;
constexpr int kSpChunk = 128;     // nodes per pipeline stage
constexpr int kGaWarps = 8;
constexpr int kGaThreads = 256;
constexpr int kGaRhs = 16;        // rhs whose G blocks sit in smem at once

// shared-memory doubles of the spread for a given rhs-per-pass count
// v rows in shared memory are padded by 2 doubles (even rpp) so the 4 nodes of
// a k-step read from distinct banks (16 rhs = 128 B would map them all to one)
__host__ __device__ constexpr int spread_vst(int rpp) { return (rpp % 2 == 0) ? rpp + 2 : rpp; }

__host__ __device__ constexpr int spread_smem(int rpp) {
  return 2 * (kSpChunk * kSRow + kSpChunk * spread_vst(rpp));
}

// ---- spread ---------------------------------------------------------------
// RPW rhs per warp; rpp = rhs per pass = 8 * RPW (or nrhs if smaller, then
// several warps share an rhs and split the k-steps).
template <int RPW, int NW = kSpWarps>
__global__ void __launch_bounds__(32 * NW, (NW == kSpWarps ? NLD_SPREAD_MINB : 1))
k_spread_mma(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
             const double* __restrict__ rows, const int32_t* __restrict__ pix,
             const double* __restrict__ vt, int nrhs, double* __restrict__ blocks) {
  constexpr int kSpWarps = NW;
  constexpr int kSpThreads = 32 * NW;
  extern __shared__ __align__(16) double sm[];
  const int rpp_max = kSpWarps * RPW;
  const int rpp = nrhs < rpp_max ? nrhs : rpp_max;
  const int rowbuf = kSpChunk * kSRow;                // doubles per row buffer
  const int vst = spread_vst(rpp);                     // v row stride
  const int vbuf = kSpChunk * vst;                     // doubles per v buffer
  double* const sv0 = sm + 2 * rowbuf;
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int slots = (rpp + RPW - 1) / RPW;       // warps-groups with distinct rhs
  const int wpr = kSpWarps / slots;              // warps sharing an rhs slot
  const int slot = warp / wpr;
  const int slice = warp - slot * wpr;
  const bool busy = slot < slots;
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * kRow;
  const int32_t* __restrict__ pw = pix + sd.start;
  const int nchunk = (sd.count + kSpChunk - 1) / kSpChunk;

  for (int rg = 0; rg < nrhs; rg += rpp) {
    const int rn = min(rpp, nrhs - rg);
    double acc[RPW][8][2];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int n = 0; n < 8; ++n) acc[q][n][0] = acc[q][n][1] = 0.0;

    auto stage = [&](int ck, int buf) {
      const int c0 = ck * kSpChunk;
      const int cn = min(kSpChunk, sd.count - c0);
      // rows: 6 granules of 16 B per dimension pair... 12 granules per row
      for (int e = tid; e < cn * 12; e += kSpThreads) {
        const int pt = e / 12, gi = e - pt * 12;
        const int dim = gi >> 2, w4 = gi & 3;
        // smem order [C][B][A]: dim 2 -> 0, dim 1 -> 8, dim 0 -> 16
        cp_async16(sm + buf * rowbuf + pt * kSRow + (2 - dim) * kS + 2 * w4,
                   rw + (int64_t)(c0 + pt) * kRow + dim * kS + 2 * w4);
      }
      if (rn == 16 && rpp == 16 && nrhs % 2 == 0 && ((uintptr_t)vt & 15) == 0) {
        // 16 rhs = one 128-B pixel-major line per node: 8 x 16-B copies
        for (int e = tid; e < cn * 8; e += kSpThreads) {
          const int pt = e >> 3, q = (e & 7) * 2;
          cp_async16(sv0 + buf * vbuf + pt * vst + q, vt + (int64_t)pw[c0 + pt] * nrhs + rg + q);
        }
      } else {
        for (int e = tid; e < cn * rn; e += kSpThreads) {
          const int pt = e / rn, q = e - pt * rn;
          cp_async8(sv0 + buf * vbuf + pt * vst + q, vt + (int64_t)pw[c0 + pt] * nrhs + rg + q);
        }
      }
      // zero-pad to a multiple of 4 nodes so the k-step loop needs no bounds test
      const int cpad = (cn + 3) & ~3;
      for (int e = tid; e < (cpad - cn) * kSRow; e += kSpThreads)
        sm[buf * rowbuf + cn * kSRow + e] = 0.0;
      for (int e = tid; e < (cpad - cn) * vst; e += kSpThreads)
        sv0[buf * vbuf + cn * vst + e] = 0.0;
      cp_commit();
    };

    stage(0, 0);
    for (int ck = 0; ck < nchunk; ++ck) {
      const int buf = ck & 1;
      if (ck + 1 < nchunk) {
        stage(ck + 1, buf ^ 1);
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      const int cn = min(kSpChunk, sd.count - ck * kSpChunk);
      if (busy) {
        const double* R = sm + buf * rowbuf;
        const double* V = sv0 + buf * vbuf;
        const int nks = (cn + 3) >> 2;
        const int q0 = slot * RPW;
#pragma unroll kSpUnroll
        for (int ks = slice; ks < nks; ks += wpr) {
          const int j = ks * 4 + t;
          const double* row = R + j * kSRow;
          double bw[8];
#pragma unroll
          for (int b = 0; b < 8; b += 2) {
            const double2 x = *reinterpret_cast<const double2*>(row + kS + b);
            bw[b] = x.x;
            bw[b + 1] = x.y;
          }
          const double cw = row[g];
          const double aw = row[2 * kS + g];
          double af[RPW];
#pragma unroll
          for (int q = 0; q < RPW; ++q) af[q] = V[j * vst + q0 + q] * aw;
#pragma unroll
          for (int n = 0; n < 8; ++n) {
            const double bf = bw[n] * cw;
#pragma unroll
            for (int q = 0; q < RPW; ++q) dmma(acc[q][n], af[q], bf);
          }
        }
      }
      __syncthreads();
    }
    // block element (a = g, b = n, c = 2t + i)
    if (wpr == 1) {
      if (busy) {
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          const int qq = slot * RPW + q;
          if (qq >= rn) continue;
#pragma unroll
          for (int n = 0; n < 8; ++n)
#pragma unroll
            for (int i = 0; i < 2; ++i)
              blocks[(sd.block + (g * 8 + n) * 8 + 2 * t + i) * nrhs + rg + qq] = acc[q][n][i];
        }
      }
    } else {
      // RPW == 1 here (rpp < 8): reduce the wpr warps of each slot in smem
      double* red = sm;   // kSpWarps * 512 doubles fit in the staging area
      if (busy) {
#pragma unroll
        for (int n = 0; n < 8; ++n)
#pragma unroll
          for (int i = 0; i < 2; ++i) red[warp * kBlk + (g * 8 + n) * 8 + 2 * t + i] = acc[0][n][i];
      }
      __syncthreads();
      for (int e = tid; e < slots * kBlk; e += kSpThreads) {
        const int s = e / kBlk, k = e - s * kBlk;
        if (s >= rn) continue;
        double sum = 0.0;
        for (int w = 0; w < wpr; ++w) sum += red[(s * wpr + w) * kBlk + k];
        blocks[(sd.block + k) * nrhs + rg + s] = sum;
      }
      __syncthreads();
    }
  }
}

// ---- spread with shared (B (x) C) operands (16 rhs per pass) --------------
// Same product as k_spread_mma<2, 8>, but the B-fragments B_j[b] C_j[c] --
// identical for all 8 warps (they differ only in their rhs) -- are formed
// once per CTA into shared memory instead of once per warp, so the DMULs
// that share the fp64 pipe with DMMA drop from 10 to 3 per 16 DMMA.
// Software pipeline over chunks of 48 nodes, one barrier per chunk:
//   iteration ck: cp.async raw rows of chunk ck+2 and v lines of chunk ck+1;
//                 DMMA over chunk ck from BCA[ck&1] (B (x) C | A rows);
//                 in the middle, each warp forms BCA of 6 nodes of chunk
//                 ck+1 from the raw rows (no separate phase: the other warps
//                 keep the tensor pipe busy meanwhile);
//                 wait for the copies, barrier.
// BCA rows are 76 doubles (24 banks apart: the 4 nodes of a k-step are
// conflict-free for the B-fragment and A reads).
constexpr int kBcChunk = 48;
constexpr int kBcRow = 76;
constexpr int kBcV = 18;          // v row stride: 16 rhs + 2 (bank spread)

__host__ __device__ constexpr int spread_bc_smem() {
  return 2 * kBcChunk * kRow + 2 * kBcChunk * kBcV + 2 * kBcChunk * kBcRow;
}

__global__ void __launch_bounds__(256, 2)
k_spread_bc(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
            const double* __restrict__ rows, const int32_t* __restrict__ pix,
            const double* __restrict__ vt, int nrhs, double* __restrict__ blocks) {
  extern __shared__ __align__(16) double sm[];
  double* const raw = sm;                                  // [2][48][24]
  double* const sv = sm + 2 * kBcChunk * kRow;             // [2][48][18]
  double* const bca = sv + 2 * kBcChunk * kBcV;            // [2][48][76]
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * kRow;
  const int32_t* __restrict__ pw = pix + sd.start;
  const int nchunk = (sd.count + kBcChunk - 1) / kBcChunk;
  auto chunk_n = [&](int ck) { return min(kBcChunk, sd.count - ck * kBcChunk); };

  for (int rg = 0; rg < nrhs; rg += 16) {
    double acc[2][8][2];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int n = 0; n < 8; ++n) acc[q][n][0] = acc[q][n][1] = 0.0;

    auto stage_raw = [&](int ck) {
      if (ck >= nchunk) return;
      const double* src = rw + (int64_t)ck * kBcChunk * kRow;
      double* dst = raw + (ck & 1) * kBcChunk * kRow;
      for (int e = tid; e < chunk_n(ck) * (kRow / 2); e += 256) cp_async16(dst + 2 * e, src + 2 * e);
    };
    auto stage_v = [&](int ck) {
      if (ck >= nchunk) return;
      const int c0 = ck * kBcChunk, cn = chunk_n(ck);
      double* dst = sv + (ck & 1) * kBcChunk * kBcV;
      for (int e = tid; e < cn * 8; e += 256) {
        const int pt = e >> 3, q = (e & 7) * 2;
        cp_async16(dst + pt * kBcV + q, vt + (int64_t)pw[c0 + pt] * nrhs + rg + q);
      }
      // pad to a multiple of 4 nodes with v = 0 (uninitialised smem could be NaN)
      for (int e = tid; e < (((cn + 3) & ~3) - cn) * kBcV; e += 256) dst[cn * kBcV + e] = 0.0;
    };
    // this warp's 6 nodes of chunk ck: BCA[p] = [B(x)C | A | pad]
    auto form_bca = [&](int ck) {
      if (ck >= nchunk) return;
      const int cn = chunk_n(ck);
      const double* R = raw + (ck & 1) * kBcChunk * kRow;
      double* O = bca + (ck & 1) * kBcChunk * kBcRow;
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const int e = lane + 32 * i;             // 192 pairs = 6 nodes x 32
        const int p = warp * 6 + (e >> 5), pr = e & 31;
        const int b = pr >> 2, c = (pr & 3) * 2;
        double2 o;
        if (p < cn) {
          const double bw = R[p * kRow + kS + b];
          const double2 cw = *reinterpret_cast<const double2*>(R + p * kRow + 2 * kS + c);
          o.x = bw * cw.x;
          o.y = bw * cw.y;
        } else {
          o.x = o.y = 0.0;
        }
        *reinterpret_cast<double2*>(O + p * kBcRow + b * 8 + c) = o;
      }
      if (lane < 24) {
        const int p = warp * 6 + (lane >> 2), a = (lane & 3) * 2;
        double2 o;
        if (p < cn) o = *reinterpret_cast<const double2*>(R + p * kRow + a);
        else o.x = o.y = 0.0;
        *reinterpret_cast<double2*>(O + p * kBcRow + 64 + a) = o;
      }
    };

    // prologue: BCA(0) formed, raw(1) and v(0) resident
    stage_raw(0);
    stage_v(0);
    cp_commit();
    stage_raw(1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    form_bca(0);
    cp_wait<0>();
    __syncthreads();

    for (int ck = 0; ck < nchunk; ++ck) {
      stage_raw(ck + 2);     // raw buffer ck&1: chunk ck's rows were consumed by form_bca(ck)
      stage_v(ck + 1);
      cp_commit();
      const int nks = (chunk_n(ck) + 3) >> 2;
      const double* B = bca + (ck & 1) * kBcChunk * kBcRow;
      const double* V = sv + (ck & 1) * kBcChunk * kBcV + 2 * warp;
      auto kstep = [&](int ks) {
        const int j = ks * 4 + t;
        const double* row = B + j * kBcRow;
        const double aw = row[64 + g];
        const double2 vv = *reinterpret_cast<const double2*>(V + j * kBcV);
        const double af0 = vv.x * aw, af1 = vv.y * aw;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const double bf = row[n * 8 + g];
          dmma(acc[0][n], af0, bf);
          dmma(acc[1][n], af1, bf);
        }
      };
      const int half = nks >> 1;
#pragma unroll 2
      for (int ks = 0; ks < half; ++ks) kstep(ks);
      form_bca(ck + 1);
#pragma unroll 2
      for (int ks = half; ks < nks; ++ks) kstep(ks);
      cp_wait<0>();
      __syncthreads();
    }
    // block element (a = g, b = n, c = 2t + i), rhs rg + 2 warp + q
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          blocks[(sd.block + (g * 8 + n) * 8 + 2 * t + i) * nrhs + rg + 2 * warp + q] = acc[q][n][i];
    __syncthreads();   // smem reuse by the next rhs group
  }
}

// ---- gather ---------------------------------------------------------------
// Khatri-Rao form: T[a][j] = sum_{(b,c)} G[a][(b,c)] (B_j (x) C_j)[(b,c)]
// (M = 8 rows a, K = 64, N = 8 nodes), then y_j = sum_a A_j[a] T[a][j]
// reduced over a across the 8 lanes of a column.  The (B (x) C) fragments
// depend only on the nodes, so they are formed once per 8-node tile and
// reused for every right-hand side; the G fragments come from shared memory
// (XOR-swizzled: element (a, kk) at a*64 + (kk ^ 4a), conflict-free).
__global__ void __launch_bounds__(kGaThreads, 2)
k_gather_mma(const SubDev* __restrict__ subs, const CellDev* __restrict__ cells,
             const WinDev* __restrict__ wins, const double* __restrict__ rows,
             const int32_t* __restrict__ pix, const double* __restrict__ grid,
             int64_t grid_ld, double* __restrict__ wout, int64_t N, int nrhs) {
  extern __shared__ __align__(16) double gb[];   // [kGaRhs][512]
  const SubDev sd = subs[blockIdx.x];
  const CellDev cd = cells[sd.cell];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * kRow;
  double* __restrict__ out = wout + (int64_t)sd.win * N * nrhs;
  const int ntile = (sd.count + 7) >> 3;
  for (int rg = 0; rg < nrhs; rg += kGaRhs) {
    const int rn = min(kGaRhs, nrhs - rg);
    __syncthreads();
    for (int e = tid; e < rn * kBlk; e += kGaThreads) {
      const int q = e >> 9, k = e & (kBlk - 1);
      const int a = k >> 6, kk = k & 63;
      int p0 = cd.cc[0] + a, p1 = cd.cc[1] + (kk >> 3), p2 = cd.cc[2] + (kk & 7);
      if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
      if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
      if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
      gb[q * kBlk + a * 64 + (kk ^ (4 * a))] =
          grid[(int64_t)(rg + q) * grid_ld + wd.grid_off +
               ((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
    }
    __syncthreads();
    struct Tile {
      double bw[8], c0, c1, aw[2];
      int pj[2];
    };
    auto load_tile = [&](Tile& T, int nt) {
      const int j0 = nt * 8;
      const int jn = j0 + g;
      const bool okn = jn < sd.count;
      const double* r = rw + (int64_t)(okn ? jn : 0) * kRow;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 x = __ldg(reinterpret_cast<const double2*>(r + kS) + k);
        T.bw[2 * k] = okn ? x.x : 0.0;
        T.bw[2 * k + 1] = okn ? x.y : 0.0;
      }
      T.c0 = __ldg(r + 2 * kS + t);
      T.c1 = __ldg(r + 2 * kS + 4 + t);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int j = j0 + 2 * t + i;
        const bool ok = j < sd.count;
        T.aw[i] = ok ? __ldg(rw + (int64_t)j * kRow + g) : 0.0;
        T.pj[i] = (ok && g == 0) ? __ldg(pix + sd.start + j) : 0;
      }
    };
    Tile cur, nxt;
    if (warp < ntile) load_tile(cur, warp);
    for (int nt = warp; nt < ntile; nt += kGaWarps) {
      if (nt + kGaWarps < ntile) load_tile(nxt, nt + kGaWarps);
      const int j0 = nt * 8;
      double bf[16];
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) bf[ks] = cur.bw[ks >> 1] * ((ks & 1) ? cur.c1 : cur.c0);
      const double aw[2] = {cur.aw[0], cur.aw[1]};
      int jp[2] = {j0 + 2 * t, j0 + 2 * t + 1};
      const int pj[2] = {cur.pj[0], cur.pj[1]};
      const int gsw = 4 * g;
      auto finish = [&](const double (&acc)[4][2], int q) {
        double p[2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
          p[i] = aw[i] * ((acc[0][i] + acc[1][i]) + (acc[2][i] + acc[3][i]));
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
          p[1] += __shfl_xor_sync(0xffffffffu, p[1], off);
        }
        if (g == 0) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if (jp[i] < sd.count) out[(int64_t)pj[i] * nrhs + rg + q] = p[i];
        }
      };
      int q = 0;
      // two right-hand sides per pass: 8 independent DMMA chains in flight
      for (; q + 1 < rn; q += 2) {
        const double* G0 = gb + q * kBlk + g * 64;
        const double* G1 = G0 + kBlk;
        double a0[4][2], a1[4][2];
#pragma unroll
        for (int c = 0; c < 4; ++c) a0[c][0] = a0[c][1] = a1[c][0] = a1[c][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const int o = (4 * ks + t) ^ gsw;
          dmma(a0[ks & 3], G0[o], bf[ks]);
          dmma(a1[ks & 3], G1[o], bf[ks]);
        }
        finish(a0, q);
        finish(a1, q + 1);
      }
      if (q < rn) {
        const double* G0 = gb + q * kBlk + g * 64;
        double a0[4][2];
#pragma unroll
        for (int c = 0; c < 4; ++c) a0[c][0] = a0[c][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) dmma(a0[ks & 3], G0[(4 * ks + t) ^ gsw], bf[ks]);
        finish(a0, q);
      }
      cur = nxt;
    }
  }
}

// ---- gather, right-hand sides as the M dimension (nrhs >= 8) -------------
// D[r][j] = sum_{k=(a,b,c)} G_r[k] W_j[k],  W_j = A_j (x) B_j (x) C_j.
// M = 16 rhs (2 m-tiles), N = 8 nodes, K = 512 (128 k-steps).  The W
// fragment W[k = 64a + 4ks + t][node j0 + g] = A[a] * (B (x) C)[4ks + t] costs
// one DMUL and feeds one DMMA per m-tile; the result is already the output
// (no cross-lane reduction).  G rows are padded to 516 doubles so the 8 rhs
// rows of a fragment hit distinct banks.
constexpr int kGRow = 516;

__global__ void __launch_bounds__(kGaThreads, 2)
k_gather_mma16(const SubDev* __restrict__ subs, const CellDev* __restrict__ cells,
               const WinDev* __restrict__ wins, const double* __restrict__ rows,
               const int32_t* __restrict__ pix, const double* __restrict__ grid,
               int64_t grid_ld, double* __restrict__ wout, int64_t N, int nrhs,
               GatherEpi ep) {
  extern __shared__ __align__(16) double gb[];   // [16][kGRow]
  const SubDev sd = subs[blockIdx.x];
  const CellDev cd = cells[sd.cell];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t local = sd.start - wd.node_off;
  const double* __restrict__ rw = rows + wd.row_off + local * kRow;
  double* __restrict__ out = wout + (ep.mode == kGatherStore ? (int64_t)sd.win * N * nrhs : 0);
  const int ntile = (sd.count + 7) >> 3;
  for (int rg = 0; rg < nrhs; rg += 16) {
    const int rn = min(16, nrhs - rg);
    __syncthreads();
    for (int e = tid; e < 16 * kBlk; e += kGaThreads) {
      const int q = e >> 9, k = e & (kBlk - 1);
      double val = 0.0;
      if (q < rn) {
        int p0 = cd.cc[0] + (k >> 6), p1 = cd.cc[1] + ((k >> 3) & 7), p2 = cd.cc[2] + (k & 7);
        if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
        if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
        if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
        val = grid[(int64_t)(rg + q) * grid_ld + wd.grid_off +
                   ((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
      }
      gb[q * kGRow + k] = val;
    }
    __syncthreads();
    const double* G0 = gb + g * kGRow + t;
    const double* G1 = G0 + 8 * kGRow;
    const bool two = rn > 8;
    for (int nt = warp; nt < ntile; nt += kGaWarps) {
      const int j0 = nt * 8;
      const int jn = j0 + g;
      double bc[16], aw[8];
      if (jn < sd.count) {
        const double* r = rw + (int64_t)jn * kRow;
        double bw[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 x = __ldg(reinterpret_cast<const double2*>(r) + k);
          aw[2 * k] = x.x;
          aw[2 * k + 1] = x.y;
          const double2 y = __ldg(reinterpret_cast<const double2*>(r + kS) + k);
          bw[2 * k] = y.x;
          bw[2 * k + 1] = y.y;
        }
        const double c0 = __ldg(r + 2 * kS + t), c1 = __ldg(r + 2 * kS + 4 + t);
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) bc[ks] = bw[ks >> 1] * ((ks & 1) ? c1 : c0);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) aw[k] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) bc[ks] = 0.0;
      }
      double acc[2][4][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[m][c][0] = acc[m][c][1] = 0.0;
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const double wa = aw[a];
#pragma unroll
        for (int ks = 0; ks < 16; ++ks) {
          const double w = bc[ks] * wa;
          const int k = a * 64 + 4 * ks;
          dmma(acc[0][ks & 3], G0[k], w);
          if (two) dmma(acc[1][ks & 3], G1[k], w);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int j = j0 + 2 * t + i;
        if (j >= sd.count) continue;
        const int64_t px = pix[sd.start + j];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int r = m * 8 + g;
          if (r < rn)
            gather_put(ep, out, px * nrhs + rg + r, px, rg + r,
                       (acc[m][0][i] + acc[m][1][i]) + (acc[m][2][i] + acc[m][3][i]));
        }
      }
    }
  }
}

}  // namespace mma
}  // namespace nld
