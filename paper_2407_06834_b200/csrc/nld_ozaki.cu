// Integer-sliced fp64 spread on the 5th-generation tensor cores (tcgen05,
// UMMA kind::i8, accumulators in TMEM) for 3-D windows with m = 4.
//
// The spread of one subproblem (the nodes j of one stencil cell) is the
// product  block[(a, r)][(b, c)] = sum_j X[(a, r)][j] Y[(b, c)][j]  with
// X = v_{j,r} A_j[a] (16 rhs x 8 rows) and Y = B_j[b] C_j[c] (64 columns),
// the same contraction the DMMA kernel (nld_mma.cuh) runs in fp64.  Here the
// operands are scaled by powers of two (per row of X: the subproblem's max
// |v_r| and |A_a|; per column of Y: max |B_b| and |C_c|, precomputed) into
// 46-bit integers and cut into S = 6 signed 8-bit digits,
//     x = sum_p d_p 256^(5-p),   y = sum_q e_q 256^(5-q),   d, e in [-128, 127],
// so that  x y = sum_t 256^(10-t) sum_{p+q=t} d_p e_q.  The integer products
// are exact (s8 x s8 -> s32, |sum| < 2^28 for <= 2048 nodes); the diagonals
// t = 0..S-1 are kept (the dropped ones are below 2^-46 of the operand
// bounds), accumulated in TMEM by issuing A_p against the stacked slices
// [e_0 | e_1 | ...] with the D window shifted by 64 p columns, and combined in
// fp64 in the epilogue.  Accuracy: a few 1e-14 of max|X| max|Y| per term --
// the same order as an fp64 dot product -- far inside the 1e-10 parity bar.
//
// Slicing is one DFMA per element: U = fma(x', y', 2^52 + 0x808080808080)
// rounds x'y' to an integer and leaves x'y' + 0x80..80 in the low 48
// mantissa bits, whose bytes XOR 0x80 are the balanced digits.
#include <algorithm>
#include <vector>
#include <type_traits>
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "nld_internal.cuh"
#include "nld_epi.cuh"
#include "nld_umma.cuh"

namespace nld {
namespace oz {

#ifndef NLD_OZ_SL
#define NLD_OZ_SL 6
#endif
constexpr int kSl = NLD_OZ_SL;         // digits per operand

// -DNLD_OZ_PROF: per-site clock64 totals of the pipeline waits (lane 0 of
// each warp), printed after each launch -- a tuning aid, not built by default
#ifdef NLD_OZ_PROF
__device__ unsigned long long oz_prof[32];
#define OZW(site, ...)                                                      \
  do {                                                                      \
    const long long _t0 = clock64();                                        \
    __VA_ARGS__;                                                            \
    if ((threadIdx.x & 31) == 0)                                            \
      atomicAdd(&oz_prof[site], (unsigned long long)(clock64() - _t0));     \
  } while (0)
#else
#define OZW(site, ...) __VA_ARGS__
#endif
constexpr int kRows = 128;             // M: (a, r) rows, r fastest
constexpr int kChunk = 32;             // nodes per UMMA K step (32 bytes)
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;         // kSl * 64 = 384 used
constexpr int kABytes = kRows * kChunk;          // 4 KB per slice
constexpr int kBBytes = 64 * kChunk;             // 2 KB per slice
// X digits (the M = 128 operand) live in TMEM: per operand stage 6 slices x 8
// columns after the 384 accumulator columns; shared memory holds only the Y
// digits (and raw rows), halving the operand traffic through shared memory
constexpr int kStageBytes = kSl * kBBytes;
constexpr int kXTmem0 = kSl * 64;                // first X column (after the accumulator)
constexpr int kExpPerSub = 24;         // eA[8] eB[8] eC[8]
constexpr double kMagic = 4503599627370496.0 + 141289400074368.0;  // 2^52 + 0x808080808080

__device__ __forceinline__ double pow2(int e) {
  e = max(-1022, min(1023, e));
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// exponent bound: |x| < 2^e for all x with max |x| = m (0 -> 0).  Callers
// clamp it below at -900 so every 2^(46 - e) scale stays finite; a clamped
// (tiny) operand then keeps fewer significant digits, never a wrong scale.
// Non-finite m (a NaN/Inf right-hand side, flagged by k_vmax and poisoned
// after the product) gets 0, so no scale ever overflows.
__device__ __forceinline__ int exp_bound(double m) {
  return (m > 0.0 && m <= 1.7976931348623157e308) ? ilogb(m) + 1 : 0;
}

// canonical K-major no-swizzle offset in a (rows x 32 bytes) tile
__device__ __forceinline__ int canon32(int row, int k) {
  return (row >> 3) * 256 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

// 4 elements' digit p (p = 0 most significant) packed into one word; element
// i's 48-bit field is (hi_i & 0xffff) << 32 | lo_i
__device__ __forceinline__ uint32_t digit_word(uint32_t l0, uint32_t l1, uint32_t l2, uint32_t l3,
                                               uint32_t h0, uint32_t h1, uint32_t h2, uint32_t h3,
                                               int p) {
  const int byte = 5 - p;
  const bool top = byte >= 4;
  const uint32_t s0 = top ? h0 : l0, s1 = top ? h1 : l1, s2 = top ? h2 : l2, s3 = top ? h3 : l3;
  const uint32_t k = byte & 3;
  const uint32_t sel = k | ((k + 4) << 4);
  const uint32_t w01 = __byte_perm(s0, s1, sel);
  const uint32_t w23 = __byte_perm(s2, s3, sel);
  return __byte_perm(w01, w23, 0x5410) ^ 0x80808080u;
}

#define NLD_DW(L, H, i, p) \
  digit_word(L[i], L[i + 1], L[i + 2], L[i + 3], H[i], H[i + 1], H[i + 2], H[i + 3], p)

// all six digit words of 4 elements (w[p] byte i = digit p of element i):
// a 4x4 byte transpose of the low words and a 4x2 one of the high words,
// 12 PRMT + 6 LOP instead of 6 x (3 PRMT + 1 LOP)
__device__ __forceinline__ void pack4(const uint32_t* l, const uint32_t* h, uint32_t* w) {
  const uint32_t a01 = __byte_perm(l[0], l[1], 0x5140), b01 = __byte_perm(l[0], l[1], 0x7362);
  const uint32_t a23 = __byte_perm(l[2], l[3], 0x5140), b23 = __byte_perm(l[2], l[3], 0x7362);
  const uint32_t h01 = __byte_perm(h[0], h[1], 0x5140), h23 = __byte_perm(h[2], h[3], 0x5140);
  w[5] = __byte_perm(a01, a23, 0x5410) ^ 0x80808080u;
  w[4] = __byte_perm(a01, a23, 0x7632) ^ 0x80808080u;
  w[3] = __byte_perm(b01, b23, 0x5410) ^ 0x80808080u;
  w[2] = __byte_perm(b01, b23, 0x7632) ^ 0x80808080u;
  w[1] = __byte_perm(h01, h23, 0x5410) ^ 0x80808080u;
  w[0] = __byte_perm(h01, h23, 0x7632) ^ 0x80808080u;
}

// store the 6 digit slices of 16 elements (lo/hi[16]) as one 16-byte word per
// slice: dst + p * stride
__device__ __forceinline__ void store16(const uint32_t (&lo)[16], const uint32_t (&hi)[16],
                                        uint8_t* dst, int stride) {
  uint32_t w[4][6];
#pragma unroll
  for (int g = 0; g < 4; ++g) pack4(lo + 4 * g, hi + 4 * g, w[g]);
#pragma unroll
  for (int p = 0; p < 6; ++p)
    *reinterpret_cast<uint4*>(dst + p * stride) = make_uint4(w[0][p], w[1][p], w[2][p], w[3][p]);
}
__device__ __forceinline__ void store8(const uint32_t (&lo)[8], const uint32_t (&hi)[8],
                                       uint8_t* dst, int stride) {
  uint32_t w[2][6];
#pragma unroll
  for (int g = 0; g < 2; ++g) pack4(lo + 4 * g, hi + 4 * g, w[g]);
#pragma unroll
  for (int p = 0; p < 6; ++p)
    *reinterpret_cast<uint2*>(dst + p * stride) = make_uint2(w[0][p], w[1][p]);
}

__device__ __forceinline__ void slice1(double x, double y, uint32_t& lo, uint32_t& hi) {
  const long long u = __double_as_longlong(fma(x, y, kMagic));
  lo = (uint32_t)u;
  hi = (uint32_t)(u >> 32);
}

// ---- plan-time exponent table -------------------------------------------
// per subproblem: eA[a], eB[b], eC[c] = exponent bounds of the columns of its
// weight rows (static: the features never change)
__global__ void k_sub_exponents(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
                                const double* __restrict__ rows, int16_t* __restrict__ ex) {
  __shared__ unsigned long long mx[kExpPerSub];
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  if (threadIdx.x < kExpPerSub) mx[threadIdx.x] = 0ull;
  __syncthreads();
  const double* rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int col = threadIdx.x % kExpPerSub;
  double m = 0.0;
  for (int j = threadIdx.x / kExpPerSub; j < sd.count; j += blockDim.x / kExpPerSub)
    m = fmax(m, fabs(rw[(int64_t)j * 24 + col]));
  if (threadIdx.x < (blockDim.x / kExpPerSub) * kExpPerSub)
    atomicMax(&mx[col], (unsigned long long)__double_as_longlong(m));
  __syncthreads();
  if (threadIdx.x < kExpPerSub)
    ex[(int64_t)blockIdx.x * kExpPerSub + threadIdx.x] =
        (int16_t)max(-900, exp_bound(__longlong_as_double((long long)mx[threadIdx.x])));
}

// ---- per-rhs exponent of max |v| over all pixels ---------------------------
// (the X rows are scaled by the rhs's global max |v| times the subproblem's
// max |A_a|; relative to a per-cell max this costs bits only where |v| is
// far below its global max, i.e. where the products are small anyway).
// The max is taken over the bit patterns of |v| (sign cleared): NaN > Inf >
// every finite value, so a non-finite entry is never dropped (fmax would drop
// NaN).  Such a rhs also sets flag[r] = 1: the digit slices of NaN/Inf are
// meaningless, so the product poisons that column afterwards (k_poison), as
// the reference's numpy arithmetic would propagate it (transform.py:323-333).
__global__ void __launch_bounds__(256)
k_vmax(const double* __restrict__ vt, int64_t n, int nrhs, unsigned long long* __restrict__ out,
       double* __restrict__ flag) {
  const int rows = nrhs <= 256 ? 256 / nrhs : 1;
  const int r0 = nrhs <= 256 ? threadIdx.x % nrhs : threadIdx.x;
  const int rstep = nrhs <= 256 ? nrhs : 256;
  const int64_t row0 = (int64_t)blockIdx.x * rows + (nrhs <= 256 ? threadIdx.x / nrhs : 0);
  if (nrhs <= 256 && threadIdx.x >= rows * nrhs) return;
  for (int r = r0; r < nrhs; r += rstep) {
    unsigned long long m = 0ull;
    for (int64_t i = row0; i < n; i += (int64_t)gridDim.x * rows)
      m = max(m, (unsigned long long)__double_as_longlong(vt[i * nrhs + r]) & 0x7fffffffffffffffull);
    if (m) atomicMax(&out[r], m);
    if (m >= 0x7ff0000000000000ull) flag[r] = 1.0;
  }
}

// NaN into every column r of a product whose flag[r] is set (rhs-major
// [nrhs][ld] or pixel-major [N][nrhs]); a no-op unless some flag is set
__global__ void __launch_bounds__(256)
k_poison(const double* __restrict__ flag, int nrhs, double* __restrict__ out, int64_t n,
         int64_t ld, int pixel_major) {
  __shared__ int any;
  if (threadIdx.x == 0) {
    int a = 0;
    for (int r = 0; r < nrhs; ++r) a |= flag[r] != 0.0;
    any = a;
  }
  __syncthreads();
  if (!any) return;
  const int64_t total = n * nrhs;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = pixel_major ? e / nrhs : e % n;
    const int r = (int)(pixel_major ? e % nrhs : e / n);
    if (flag[r] != 0.0) out[pixel_major ? e : (int64_t)r * ld + i] = __longlong_as_double(0x7ff8000000000000ll);
  }
}

// ---- plan-time Y digits for the sliced spread (PY) ------------------------
// Exactly the slicers' Y = B_b C_c (scaled by 2^(46 - eB_b - eC_c)) of every
// 32-node chunk, as six 64 x 32 K-major digit slices (zero past the count).
__global__ void k_spread_ydig(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
                              const double* __restrict__ rows, const int16_t* __restrict__ sub_exp,
                              const int64_t* __restrict__ ychunk, uint8_t* __restrict__ ydig);

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(umma::smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(umma::smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef NLD_SP_COALESCE
#define NLD_SP_COALESCE 1                        // spread loader: line-coalesced cp.async
#endif
constexpr int kRawRows = kChunk * 24 * 8;       // 6 KB of weight rows per chunk
constexpr int kRawV = kChunk * 16 * 8;          // 4 KB of v lines per chunk
constexpr int kRawBytes = kRawRows + kRawV;
#ifndef NLD_SP_RAWSTAGES
#define NLD_SP_RAWSTAGES 8
#endif
constexpr int kRawStages = NLD_SP_RAWSTAGES;   // raw chunks in flight

#ifndef NLD_SP_OPSTAGES
#define NLD_SP_OPSTAGES 2                    // 384 + 2 x 48 TMEM columns <= 512
#endif
constexpr int kOpStages = NLD_SP_OPSTAGES;   // operand stages (slicers <-> tensor core)

__host__ __device__ constexpr int spread_oz_smem() {
  return kOpStages * kStageBytes + kRawStages * kRawBytes;
}

// Precomputed-Y variant (PY): Y = B (x) C depends only on the (static) node
// tables, so its digit slices are cut once at plan time (k_spread_ydig) in
// the UMMA B-operand layout and streamed per chunk by one TMA bulk copy into
// the raw stage, which the UMMAs then read directly.  The slicers cut only X,
// shared memory carries no operand stage, and a raw stage is released by the
// slicers and by the chunk's UMMA commit.  Raw stage: [A rows 32 x 8 doubles |
// v lines 32 x 16 doubles | Y digits 6 x 2 KB].
constexpr int kPyA = kChunk * 8 * 8;             // 2 KB
constexpr int kPyY = kPyA + kRawV;               // Y digits offset
constexpr int kPyRawBytes = kPyY + kSl * kBBytes;   // 18 KB
#ifndef NLD_PY_STAGES
#define NLD_PY_STAGES 8
#endif
#ifndef NLD_PY_YBULK
#define NLD_PY_YBULK 1                           // Y digits by one TMA bulk copy (else cp.async)
#endif
constexpr int kPyRawStages = NLD_PY_STAGES;
constexpr int kYChunkBytes = kSl * kBBytes;      // 12 KB per chunk in HBM
__host__ __device__ constexpr int spread_oz_py_smem() { return kPyRawStages * kPyRawBytes; }

// ---- spread ---------------------------------------------------------------
// One CTA per subproblem (TMEM: 384 of 512 columns -> one CTA per SM),
// warp-specialised, mbarrier-pipelined:
//   warp 9  (loader): cp.async the weight rows and the 16-rhs v lines of
//           32-node chunks into kRawStages raw stages; each lane's copies
//           arrive on the stage's `full` barrier when they land
//           (cp.async.mbarrier.arrive.noinc), so no thread ever waits on them;
//   warps 0-7 (slicers): wait for a raw chunk, cut X = v A and Y = B C into
//           digit slices in operand stage c&1, fence to the async proxy and
//           arrive on the stage's `ready` barrier; after the last chunk they
//           read TMEM and write the block (epilogue);
//   warp 8  (issuer): per chunk, one lane issues the 8 UMMAs and commits them
//           to the stage's `free` barrier (operand stage reusable) and, after
//           the last chunk, to `acc`.
constexpr int kSpreadThreads = 320;
constexpr int kSlicers = 256;
constexpr int kIssuerWarp = 8;
constexpr int kLoaderWarp = 9;

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* mbar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(umma::smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(umma::smem_u32(mbar)) : "memory");
}

template <bool PY>
__global__ void __launch_bounds__(kSpreadThreads, 1)
k_spread_oz(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
            const double* __restrict__ rows, const int32_t* __restrict__ pix,
            const int16_t* __restrict__ sub_exp, const uint8_t* __restrict__ ydig,
            const int64_t* __restrict__ ychunk, const unsigned long long* __restrict__ vmax,
            const double* __restrict__ vt, int nrhs, double* __restrict__ blocks) {
  constexpr int RS = PY ? kPyRawStages : kRawStages;
  constexpr int RB = PY ? kPyRawBytes : kRawBytes;
  constexpr int RowS = PY ? 8 : 24;                 // doubles per node row in the raw stage
  constexpr int VOff = PY ? kPyA : kRawRows;        // v lines in the raw stage
  // 16-byte alignment is all the no-swizzle descriptors need; do not declare
  // more: under -rdc the dynamic window is not 1024-aligned, and the compiler
  // would fold the declared alignment into the descriptor address bits
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t raw_full[RS], raw_empty[RS];
  __shared__ uint64_t op_ready[kOpStages], op_free[kOpStages], acc_full, acc_empty;
  __shared__ uint32_t taddr_s;
  __shared__ double rsc[kRows];       // row scale 2^(ev + eA - 46)
  __shared__ double csc[64];          // column scale 2^(eB + eC + 34)
  __shared__ double sva[kRows];       // 2^(46 - ev_r)
  __shared__ double sa[8], sb[8], sc[8];

  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int32_t* __restrict__ pw = pix + sd.start;
  const int16_t* ex = sub_exp + (int64_t)blockIdx.x * kExpPerSub;
  uint8_t* const raw = smem + (PY ? 0 : kOpStages * kStageBytes);
  const int nchunk = (sd.count + kChunk - 1) / kChunk;
  const int ngroups = nrhs / 16;
  const uint8_t* yd = PY ? ydig + ychunk[blockIdx.x] * (int64_t)kYChunkBytes : nullptr;

  if (warp == 0) umma::tmem_alloc<kTmemCols>(&taddr_s);
  if (tid == 32) {
    for (int k = 0; k < RS; ++k) {
      // 32 noinc cp.async arrivals + the bulk copy's
      umma::mbar_init(&raw_full[k], (PY && !NLD_PY_YBULK) ? 32 : 33);
      umma::mbar_init(&raw_empty[k], kSlicers / 32 + (PY ? 1 : 0));   // (+ the UMMA commit)
    }
    for (int k = 0; k < kOpStages; ++k) {
      umma::mbar_init(&op_ready[k], kSlicers / 32);
      umma::mbar_init(&op_free[k], 1);
    }
    umma::mbar_init(&acc_full, 1);
    umma::mbar_init(&acc_empty, kSlicers / 32);
    umma::mbar_fence_init();
  }
  if (tid < 8) {
    sa[tid] = pow2(-ex[tid]);
    sb[tid] = pow2(46 - ex[8 + tid]);
    sc[tid] = pow2(-ex[16 + tid]);
  }
  if (tid < 64) csc[tid] = ldexp(1.0, ex[8 + (tid >> 3)] + ex[16 + (tid & 7)] + 34);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = taddr_s;
#ifdef NLD_OZ_PROF
  const long long t_role = clock64();
#endif

  if (warp == kLoaderWarp) {
    // ---------------------------------------------------------------- loader
    int g = 0;
    auto pix_at = [&](int c) -> int32_t {
      const int j = c * kChunk + lane;
      return (c < nchunk && j < sd.count) ? __ldg(pw + j) : 0;
    };
    for (int grp = 0; grp < ngroups; ++grp) {
      const int rg = grp * 16;
      // pixel indices: four registers, each refilled with the index of the
      // chunk four ahead right after its copies are issued (no register moves
      // of in-flight loads, so the load latency hides behind four chunks)
      auto body = [&](int c, int32_t px) {
        if (c >= nchunk) return;
        const int s = g % RS;
        if (g >= RS) OZW(16, umma::mbar_wait(&raw_empty[s], ((g / RS) - 1) & 1));
        uint8_t* dst = raw + s * RB;
        const int j0 = c * kChunk, cn = min(kChunk, sd.count - j0);
        if (lane == 0) {
          if constexpr (PY) {
#if NLD_PY_YBULK
            // the chunk's precomputed Y digits: one TMA bulk copy
            umma::mbar_arrive_expect_tx(&raw_full[s], kYChunkBytes);
            umma::bulk_g2s(dst + kPyY, yd + (int64_t)c * kYChunkBytes, kYChunkBytes, &raw_full[s]);
#endif
          } else {
            // the chunk's weight rows are contiguous: one TMA bulk copy
            const uint32_t bytes = (uint32_t)cn * 24 * 8;
            umma::mbar_arrive_expect_tx(&raw_full[s], bytes);
            umma::bulk_g2s(dst, rw + (int64_t)j0 * 24, bytes, &raw_full[s]);
          }
        }
#if defined(NLD_EXP_SNOLOAD)
        if (lane < cn) cp_async16(dst + VOff + lane * 16, vt + (int64_t)(uint32_t)px * nrhs + rg);
#elif NLD_SP_COALESCE
        // coalesced: each instruction copies whole lines -- 8 lanes per 128-byte
        // v line (4 nodes per instruction), 4 lanes per 64-byte A part (8 nodes);
        // the node's pixel comes from its lane by shuffle
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int nd = q * 4 + (lane >> 3), pc = lane & 7;
          const int32_t pxn = __shfl_sync(0xffffffffu, px, nd);
          if (nd < cn)
            cp_async16(dst + VOff + nd * 128 + pc * 16,
                       vt + (int64_t)(uint32_t)pxn * nrhs + rg + 2 * pc);
        }
#if !NLD_PY_YBULK
        if constexpr (PY) {
#pragma unroll
          for (int q = 0; q < kYChunkBytes / 512; ++q)
            cp_async16(dst + kPyY + (q * 32 + lane) * 16,
                       yd + (int64_t)c * kYChunkBytes + (q * 32 + lane) * 16);
        }
#endif
        if constexpr (PY) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int nd = q * 8 + (lane >> 2), pc = lane & 3;
            if (nd < cn) cp_async16(dst + nd * 64 + pc * 16, rw + (int64_t)(j0 + nd) * 24 + 2 * pc);
          }
        }
#else
        if (lane < cn) {
          if constexpr (PY) {
            // A part (8 doubles) of the node's weight row
            const double* as = rw + (int64_t)(j0 + lane) * 24;
#pragma unroll
            for (int q = 0; q < 4; ++q) cp_async16(dst + lane * 64 + 16 * q, as + 2 * q);
          }
#ifdef NLD_EXP_CONTIG_V
          const double* vs = vt + (int64_t)(j0 + lane) * nrhs + rg;   // timing experiment only
#else
          const double* vs = vt + (int64_t)(uint32_t)px * nrhs + rg;
#endif
          uint8_t* vd = dst + VOff + lane * 128;
#pragma unroll
          for (int q = 0; q < 8; ++q) cp_async16(vd + 16 * q, vs + 2 * q);
        }
#endif
#ifdef NLD_EXP_WAITGROUP
        cp_commit();
        cp_wait<0>();
        mbar_arrive(&raw_full[s]);
#else
        cp_async_mbar_arrive(&raw_full[s]);
#endif
        ++g;
      };
      int32_t p0 = pix_at(0), p1 = pix_at(1), p2 = pix_at(2), p3 = pix_at(3);
      for (int c = 0; c < nchunk; c += 4) {
        body(c, p0);
        p0 = pix_at(c + 4);
        body(c + 1, p1);
        p1 = pix_at(c + 5);
        body(c + 2, p2);
        p2 = pix_at(c + 6);
        body(c + 3, p3);
        p3 = pix_at(c + 7);
      }
    }
  } else if (warp == kIssuerWarp) {
    // ---------------------------------------------------------------- issuer
    int g = 0;
    for (int grp = 0; grp < ngroups; ++grp) {
      if (grp > 0) OZW(18, umma::mbar_wait(&acc_empty, (grp - 1) & 1));   // epilogue drained TMEM
      for (int c = 0; c < nchunk; ++c, ++g) {
        const int st = g % kOpStages, s = g % RS;
        OZW(17, umma::mbar_wait(&op_ready[st], (g / kOpStages) & 1));
        if constexpr (PY) umma::mbar_wait(&raw_full[s], (g / RS) & 1);   // Y digits landed
        umma::fence_after();
        if (lane == 0) {
          const uint32_t bB = PY ? umma::smem_u32(raw + s * RB + kPyY)
                                 : umma::smem_u32(smem + st * kStageBytes);
          const uint32_t xa = tmem + (uint32_t)(kXTmem0 + st * kSl * 8);
#ifndef NLD_EXP_SNOMMA
#pragma unroll
          for (int p = 0; p < kSl; ++p) {
#pragma unroll
            for (int q0 = 0; q0 < kSl - p; q0 += 4) {
              const int nq = min(4, kSl - p - q0);
              const uint64_t db = umma::make_sdesc(bB + q0 * kBBytes, 128, 256);
              umma::mma_i8_ta(tmem + (uint32_t)((p + q0) * 64), xa + (uint32_t)(p * 8), db,
                              umma::idesc_i8(kRows, nq * 64), (c > 0 || p > 0) ? 1u : 0u);
            }
          }
#endif
          umma::commit(&op_free[st]);
          if constexpr (PY) umma::commit(&raw_empty[s]);   // Y digits consumed
          if (c == nchunk - 1) umma::commit(&acc_full);
        }
        __syncwarp();
      }
    }
  } else {
    // --------------------------------------------------------------- slicers
    int g = 0;
    for (int grp = 0; grp < ngroups; ++grp) {
      const int rg = grp * 16;
      if (tid < kRows) {
        const int a = tid >> 4, r = tid & 15;
        // |v| below 2^-900 would push 2^(46 - ev) out of range; clamping ev
        // keeps it finite (tiny v just keeps fewer digits)
        const int ev = max(-900, exp_bound(__longlong_as_double((long long)vmax[rg + r])));
        sva[tid] = pow2(46 - ev);
        rsc[tid] = ldexp(1.0, ev + ex[a] - 46);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kSlicers));      // slicers only
      for (int c = 0; c < nchunk; ++c, ++g) {
        const int st = g % kOpStages, s = g % RS;
#ifndef NLD_EXP_NORAWWAIT
        OZW(19, umma::mbar_wait(&raw_full[s], (g / RS) & 1));
#endif
        if (g >= kOpStages) OZW(20, umma::mbar_wait(&op_free[st], ((g / kOpStages) - 1) & 1));
        uint8_t* sB = smem + st * kStageBytes;
        const double* R = reinterpret_cast<const double*>(raw + s * RB);
        const double* Vr = reinterpret_cast<const double*>(raw + s * RB + VOff);
        const int cn = min(kChunk, sd.count - c * kChunk);
        // full chunks (all but a subproblem's last) skip the per-node guards
        auto slice_chunk = [&](auto full) {
          {
            const int m = tid & 127, h = tid >> 7;
            const int a = m >> 4, r = m & 15;
            const double sx = sva[m] * sa[a];      // exact: a product of powers of two
            uint32_t lo[16], hi[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int j = h * 16 + i;
              double x = 0.0, y = 0.0;
              if (full || j < cn) {
                x = Vr[j * 16 + r];
                y = R[j * RowS + a] * sx;
              }
              slice1(x, y, lo[i], hi[i]);
            }
            // row m = TMEM lane m (warp w holds lanes 32 (w % 4)..): 16 nodes =
            // 4 columns per digit slice
            uint32_t w4[4][6];
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) pack4(lo + 4 * g4, hi + 4 * g4, w4[g4]);
            const uint32_t xt = tmem + ((uint32_t)((m >> 5) * 32) << 16) +
                                (uint32_t)(kXTmem0 + st * kSl * 8 + h * 4);
#pragma unroll
            for (int p = 0; p < kSl; ++p)
              umma::tmem_st4(xt + (uint32_t)(p * 8), w4[0][p], w4[1][p], w4[2][p], w4[3][p]);
          }
          if constexpr (!PY) {
            const int n = tid & 63, gq = tid >> 6;
            const int b = n >> 3, cc = n & 7;
            const double sy = sb[b] * sc[cc];
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int j = gq * 8 + i;
              double x = 0.0, y = 0.0;
              if (full || j < cn) {
                x = R[j * 24 + 8 + b] * sy;
                y = R[j * 24 + 16 + cc];
              }
              slice1(x, y, lo[i], hi[i]);
            }
            store8(lo, hi, sB + canon32(n, gq * 8), kBBytes);
          }
        };
#ifndef NLD_EXP_SNOSLICE
        if (cn == kChunk) OZW(23, slice_chunk(std::true_type{}));
        else OZW(23, slice_chunk(std::false_type{}));
#endif
        OZW(22, umma::tmem_wait_st());
        umma::fence_before();
        if constexpr (!PY) umma::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_ready[st]);
          mbar_arrive(&raw_empty[s]);
        }
      }
      // epilogue: accumulators of this rhs group -> block
      OZW(21, umma::mbar_wait(&acc_full, grp & 1));
      umma::fence_after();
#ifndef NLD_EXP_SNOEPI
      {
        const int lg = warp & 3, half = warp >> 2;
        const int m = lg * 32 + lane;
        const int a = m >> 4, r = m & 15;
        const double rs = rsc[m];
        const uint32_t tl = tmem + ((uint32_t)(lg * 32) << 16);
#pragma unroll 1
        for (int c0 = half * 32; c0 < half * 32 + 32; c0 += 16) {
          uint32_t dv[kSl][16];
#pragma unroll
          for (int t = 0; t < kSl; ++t) umma::tmem_ld16(tl + (uint32_t)(t * 64 + c0), dv[t]);
          umma::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int t = kSl - 1; t >= 0; --t)
              acc = fma(acc, 0.00390625, (double)(int32_t)dv[t][i]);
            const int bc = c0 + i;
            blocks[(sd.block + a * 64 + bc) * nrhs + rg + r] = acc * rs * csc[bc];
          }
        }
      }
#endif
      umma::fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty);
      asm volatile("bar.sync 1, %0;\n" ::"n"(kSlicers));      // rsc reuse by the next group
    }
  }
#ifdef NLD_OZ_PROF
  if (lane == 0)
    atomicAdd(&oz_prof[24 + (warp == kLoaderWarp ? 0 : warp == kIssuerWarp ? 1 : 2)],
              (unsigned long long)(clock64() - t_role));
#endif
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<kTmemCols>(tmem);
}

__global__ void __launch_bounds__(256)
k_spread_ydig(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
              const double* __restrict__ rows, const int16_t* __restrict__ sub_exp,
              const int64_t* __restrict__ ychunk, uint8_t* __restrict__ ydig) {
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int16_t* ex = sub_exp + (int64_t)blockIdx.x * kExpPerSub;
  const int n = threadIdx.x & 63, gq = threadIdx.x >> 6;
  const int b = n >> 3, cc = n & 7;
  const double sy = pow2(46 - ex[8 + b]) * pow2(-ex[16 + cc]);
  const int nchunk = (sd.count + kChunk - 1) / kChunk;
  uint8_t* base = ydig + ychunk[blockIdx.x] * (int64_t)kYChunkBytes;
  for (int c = 0; c < nchunk; ++c) {
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = c * kChunk + gq * 8 + i;
      double x = 0.0, y = 0.0;
      if (j < sd.count) {
        x = rw[(int64_t)j * 24 + 8 + b] * sy;
        y = rw[(int64_t)j * 24 + 16 + cc];
      }
      slice1(x, y, lo[i], hi[i]);
    }
    store8(lo, hi, base + (int64_t)c * kYChunkBytes + canon32(n, gq * 8), kBBytes);
  }
}

// ---- persistent spread (plan-time Y digits) ---------------------------------
// One CTA per SM walks (subproblem, rhs group) items -- the window's
// subproblems in descending size, dealt in snake order as in the persistent
// gather -- so the per-subproblem fixed costs of k_spread_oz (TMEM
// allocation, barrier set-up, pipeline fill behind the first v gathers,
// drain, epilogue) overlap the neighbouring items: the loader and the slicers
// stream across item boundaries, and 4 dedicated epilogue warps drain an
// item's accumulator (releasing TMEM as soon as it is read) while the slicers
// already cut the next item's first chunks.  The only serialisation left per
// item is the TMEM drain (the accumulator is single-buffered: 384 of 512
// columns).  Scales are per-thread registers (no per-item shared state).
//   warps 0-7 slicers (X digits -> TMEM)   warp 8 UMMA issuer
//   warp 9    loader                       warps 10-13 epilogue
constexpr int kSPEpi0 = 10;
constexpr int kSPThreads = 32 * 14;

__global__ void __launch_bounds__(kSPThreads, 1)
k_spread_ozp(const SubDev* __restrict__ subs, const int32_t* __restrict__ order, int nsub,
             const WinDev* __restrict__ wins, const double* __restrict__ rows,
             const int32_t* __restrict__ pix, const int16_t* __restrict__ sub_exp,
             const uint8_t* __restrict__ ydig, const int64_t* __restrict__ ychunk,
             const unsigned long long* __restrict__ vmax, const double* __restrict__ vt,
             int nrhs, double* __restrict__ blocks) {
  constexpr int RS = kPyRawStages, RB = kPyRawBytes;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t raw_full[RS], raw_empty[RS];
  __shared__ uint64_t op_ready[kOpStages], op_free[kOpStages], acc_full, acc_empty;
  __shared__ uint32_t taddr_s;
  uint8_t* const raw = smem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ngroups = nrhs / 16;
  const int G = (int)gridDim.x, b = (int)blockIdx.x;
  const int rounds = nsub / G, rem = nsub % G;
  const int my_rounds = rounds + ((rem > 0 && ((rounds & 1) ? (G - 1 - b) : b) < rem) ? 1 : 0);
  const int nitems = my_rounds * ngroups;
  auto item_sub = [&](int k) {
    const int i = k / ngroups;
    return order[i * G + ((i & 1) ? (G - 1 - b) : b)];
  };

  if (warp == 0) umma::tmem_alloc<kTmemCols>(&taddr_s);
  if (tid == 32) {
    for (int k = 0; k < RS; ++k) {
      umma::mbar_init(&raw_full[k], 33);                  // 32 noinc cp.async + the bulk copy
      umma::mbar_init(&raw_empty[k], kSlicers / 32 + 1);  // slicers + the UMMA commit
    }
    for (int k = 0; k < kOpStages; ++k) {
      umma::mbar_init(&op_ready[k], kSlicers / 32);
      umma::mbar_init(&op_free[k], 1);
    }
    umma::mbar_init(&acc_full, 1);
    umma::mbar_init(&acc_empty, 4);                       // epilogue warps
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = taddr_s;

  if (warp == kLoaderWarp) {
    // ---------------------------------------------------------------- loader
    int g = 0;
    for (int k = 0; k < nitems; ++k) {
      const int si = item_sub(k);
      const SubDev sd = subs[si];
      const WinDev wd = wins[sd.win];
      const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
      const int32_t* __restrict__ pw = pix + sd.start;
      const uint8_t* yd = ydig + ychunk[si] * (int64_t)kYChunkBytes;
      const int rg = (k % ngroups) * 16;
      const int nchunk = (sd.count + kChunk - 1) / kChunk;
      int32_t px = (lane < sd.count) ? __ldg(pw + lane) : 0;
      for (int c = 0; c < nchunk; ++c, ++g) {
        const int s = g % RS;
        // next chunk's pixel index, loaded before this chunk's copies
        const int jn = (c + 1) * kChunk + lane;
        const int32_t px_next = (c + 1 < nchunk && jn < sd.count) ? __ldg(pw + jn) : 0;
        if (g >= RS) umma::mbar_wait(&raw_empty[s], ((g / RS) - 1) & 1);
        uint8_t* dst = raw + s * RB;
        const int j0 = c * kChunk, cn = min(kChunk, sd.count - j0);
        if (lane == 0) {
          umma::mbar_arrive_expect_tx(&raw_full[s], kYChunkBytes);
          umma::bulk_g2s(dst + kPyY, yd + (int64_t)c * kYChunkBytes, kYChunkBytes, &raw_full[s]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int nd = q * 4 + (lane >> 3), pc = lane & 7;
          const int32_t pxn = __shfl_sync(0xffffffffu, px, nd);
          if (nd < cn)
            cp_async16(dst + kPyA + nd * 128 + pc * 16,
                       vt + (int64_t)(uint32_t)pxn * nrhs + rg + 2 * pc);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int nd = q * 8 + (lane >> 2), pc = lane & 3;
          if (nd < cn) cp_async16(dst + nd * 64 + pc * 16, rw + (int64_t)(j0 + nd) * 24 + 2 * pc);
        }
        cp_async_mbar_arrive(&raw_full[s]);
        px = px_next;
      }
    }
  } else if (warp == kIssuerWarp) {
    // ---------------------------------------------------------------- issuer
    int g = 0;
    for (int k = 0; k < nitems; ++k) {
      const SubDev sd = subs[item_sub(k)];
      const int nchunk = (sd.count + kChunk - 1) / kChunk;
      if (k > 0) umma::mbar_wait(&acc_empty, (k - 1) & 1);   // previous item drained
      for (int c = 0; c < nchunk; ++c, ++g) {
        const int st = g % kOpStages, s = g % RS;
        umma::mbar_wait(&op_ready[st], (g / kOpStages) & 1);
        umma::mbar_wait(&raw_full[s], (g / RS) & 1);
        umma::fence_after();
        if (lane == 0) {
          const uint32_t bB = umma::smem_u32(raw + s * RB + kPyY);
          const uint32_t xa = tmem + (uint32_t)(kXTmem0 + st * kSl * 8);
#pragma unroll
          for (int p = 0; p < kSl; ++p) {
#pragma unroll
            for (int q0 = 0; q0 < kSl - p; q0 += 4) {
              const int nq = min(4, kSl - p - q0);
              const uint64_t db = umma::make_sdesc(bB + q0 * kBBytes, 128, 256);
              umma::mma_i8_ta(tmem + (uint32_t)((p + q0) * 64), xa + (uint32_t)(p * 8), db,
                              umma::idesc_i8(kRows, nq * 64), (c > 0 || p > 0) ? 1u : 0u);
            }
          }
          umma::commit(&op_free[st]);
          umma::commit(&raw_empty[s]);
          if (c == nchunk - 1) umma::commit(&acc_full);
        }
        __syncwarp();
      }
    }
  } else if (warp < kIssuerWarp) {
    // --------------------------------------------------------------- slicers
    const int m = tid & 127, h = tid >> 7;
    const int a = m >> 4, r = m & 15;
    int g = 0;
    for (int k = 0; k < nitems; ++k) {
      const int si = item_sub(k);
      const SubDev sd = subs[si];
      const int rg = (k % ngroups) * 16;
      const int nchunk = (sd.count + kChunk - 1) / kChunk;
      // X row scale: the rhs's max |v| times the subproblem's max |A_a|
      const int ev = max(-900, exp_bound(__longlong_as_double((long long)vmax[rg + r])));
      const double sx = pow2(46 - ev) * pow2(-(int)sub_exp[(int64_t)si * kExpPerSub + a]);
      for (int c = 0; c < nchunk; ++c, ++g) {
        const int st = g % kOpStages, s = g % RS;
        umma::mbar_wait(&raw_full[s], (g / RS) & 1);
        if (g >= kOpStages) umma::mbar_wait(&op_free[st], ((g / kOpStages) - 1) & 1);
        const double* R = reinterpret_cast<const double*>(raw + s * RB);
        const double* Vr = reinterpret_cast<const double*>(raw + s * RB + kPyA);
        const int cn = min(kChunk, sd.count - c * kChunk);
        uint32_t lo[16], hi[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = h * 16 + i;
          double x = 0.0, y = 0.0;
          if (j < cn) {
            x = Vr[j * 16 + r];
            y = R[j * 8 + a] * sx;
          }
          slice1(x, y, lo[i], hi[i]);
        }
        uint32_t w4[4][6];
#pragma unroll
        for (int g4 = 0; g4 < 4; ++g4) pack4(lo + 4 * g4, hi + 4 * g4, w4[g4]);
        const uint32_t xt = tmem + ((uint32_t)((m >> 5) * 32) << 16) +
                            (uint32_t)(kXTmem0 + st * kSl * 8 + h * 4);
#pragma unroll
        for (int p = 0; p < kSl; ++p)
          umma::tmem_st4(xt + (uint32_t)(p * 8), w4[0][p], w4[1][p], w4[2][p], w4[3][p]);
        umma::tmem_wait_st();
        umma::fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_ready[st]);
          mbar_arrive(&raw_empty[s]);
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int lg = warp & 3;
    const int m = lg * 32 + lane;
    const int a = m >> 4, r = m & 15;
    const uint32_t tl = tmem + ((uint32_t)(lg * 32) << 16);
    for (int k = 0; k < nitems; ++k) {
      const int si = item_sub(k);
      const SubDev sd = subs[si];
      const int rg = (k % ngroups) * 16;
      const int16_t* ex = sub_exp + (int64_t)si * kExpPerSub;
      const int ev = max(-900, exp_bound(__longlong_as_double((long long)vmax[rg + r])));
      const double rs = ldexp(1.0, ev + ex[a] - 46);
      int eb[8], ec[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        eb[q] = ex[8 + q];
        ec[q] = ex[16 + q];
      }
      umma::mbar_wait(&acc_full, k & 1);
      umma::fence_after();
      double* bo = blocks + (sd.block + a * 64) * nrhs + rg + r;
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t dv[kSl][16];
#pragma unroll
        for (int t = 0; t < kSl; ++t) umma::tmem_ld16(tl + (uint32_t)(t * 64 + c0), dv[t]);
        umma::tmem_wait_ld();
        if (c0 == 48) {
          // every column read: the next item's UMMAs may overwrite the accumulator
          umma::fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int t = kSl - 1; t >= 0; --t) acc = fma(acc, 0.00390625, (double)(int32_t)dv[t][i]);
          const int bc = c0 + i;
          bo[(int64_t)bc * nrhs] = acc * rs * pow2(eb[bc >> 3] + ec[bc & 7] + 34);
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<kTmemCols>(tmem);
}

// ---- gather ---------------------------------------------------------------
// T[(a, r)][j] = sum_{(b,c)} G_r[a][(b,c)] Y_j[(b,c)],  Y_j = B_j (x) C_j,
// then y_r[j] = sum_a A_j[a] T[(a, r)][j]  (the DMMA gather's contraction,
// nld_mma.cuh k_gather_mma16, with the a-sum moved to the epilogue).
// UMMA M = 128 rows (a, r): the G digits of one subproblem (K = 64 = (b,c),
// scaled per row), N = 32-node tiles with the Y digit slices stacked along N
// ([e_0 | .. | e_{S-1-p}] against G digit p, D window shifted by 32 p), so a
// tile's 6 diagonals take 192 TMEM columns and two tiles double-buffer.
//   warp 9  (loader): cp.async each tile's weight rows -> raw stage;
//   warps 4-7 (slicers): Y digits of a tile -> operand stage;
//   warp 8  (issuer): 12 UMMAs per tile (2 K steps x 6 digit rows);
//   warps 0-3 (epilogue): TMEM -> fp64 T -> x A_j[a] -> sum over a (shuffle +
//           shared memory) -> fused window-sum / degree / shift epilogue.
// The G digits are formed by all ten warps at the start of each rhs group.
constexpr int kGTile = 32;                       // nodes per tile
constexpr int kGA = kRows * 64;                  // 8 KB per G digit slice (K = 64)
constexpr int kGB = kGTile * 64;                 // 2 KB per Y digit slice
constexpr int kGBStage = kSl * kGB;              // 12 KB
// One CTA per SM (default): double-buffered 192-column TMEM accumulator, the G
// digits in TMEM as the A operand, 8 epilogue warps.  NLD_GATHER_CTAS=2 builds
// the two-CTA variant (single accumulator and G digits in shared memory per CTA,
// 4 epilogue warps) whose G setup / drain overlap the other CTA's tiles -- within
// 1% of the default on B200.
#ifndef NLD_GATHER_CTAS
#define NLD_GATHER_CTAS 1
#endif
constexpr int kGCtas = NLD_GATHER_CTAS;
constexpr int kGAccBufs = kGCtas == 2 ? 1 : 2;
// one CTA per SM: the subproblem's G digits live in TMEM (96 columns after the
// two 192-column accumulators) and feed the UMMAs as the TMEM A operand
constexpr bool kGTmemA = kGCtas == 1;
constexpr int kGTmemA0 = 2 * kSl * kGTile;      // 384
constexpr int kGTmemCols = kGCtas == 2 ? 256 : 512;
constexpr int kGOpStages = kGCtas == 2 ? 2 : 3;
constexpr int kGRowS = 26;                       // smem row stride (doubles): conflict-free
constexpr int kGRaw = kGTile * kGRowS * 8 + kGTile * 4;   // rows + pixel indices per tile
constexpr int kGRawStages = kGCtas == 2 ? 4 : 6; // slicers run ahead of the MMA, the
                                                 // epilogue trails it
constexpr int kGEpiWarps = kGCtas == 2 ? 4 : 8;
constexpr int kGatherThreads = 32 * (kGEpiWarps + 4);   // epilogue, 2 slicer, issuer, loader
constexpr int kGSlicerWarp0 = kGEpiWarps;
constexpr int kGIssuerWarp = kGEpiWarps + 2;
constexpr int kGLoaderWarp = kGEpiWarps + 3;
constexpr int kGNodeGroups = kGTile / 8 / (kGEpiWarps / 4);   // 8-node groups per epilogue warp

// sum_t D_t 2^(40 - 8t), t = 0..5, from the six int32 diagonals of a K = 64
// product (|D_t| <= (t + 1) 2^20): the pairs D_2k 2^8 + D_2k+1 are exact in
// int32 (|.| < 1.35e9), so three IMADs, three exact int32 -> fp64 conversions
// and (X01 2^16 + X23) 2^16 + X45 with one rounding (the first FMA is exact).
// The caller's scale carries the 2^-24 (vs sum_t D_t 2^(16 - 8t)).
#ifndef NLD_OZ_COMBINE64
#define NLD_OZ_COMBINE64 0
#endif
static_assert(kSl == 6, "combine6 assumes six digits");
__device__ __forceinline__ double i2d(uint32_t x);
template <int NCOL>
__device__ __forceinline__ double combine6(const uint32_t (&dv)[6][NCOL], int i) {
#if NLD_OZ_COMBINE64
  // reference form: two exact 45-bit integers on the 64-bit integer path
  const long long H = ((long long)(int32_t)dv[0][i] << 16) + ((long long)(int32_t)dv[1][i] << 8) +
                      (long long)(int32_t)dv[2][i];
  const long long L = ((long long)(int32_t)dv[3][i] << 16) + ((long long)(int32_t)dv[4][i] << 8) +
                      (long long)(int32_t)dv[5][i];
  const double hd = __longlong_as_double(H + 0x4338000000000000LL) - 6755399441055744.0;
  const double ld = __longlong_as_double(L + 0x4338000000000000LL) - 6755399441055744.0;
  return fma(ld, 5.9604644775390625e-08, hd) * 16777216.0;   // x 2^24 (exact)
#else
  const uint32_t x01 = dv[0][i] * 256u + dv[1][i];
  const uint32_t x23 = dv[2][i] * 256u + dv[3][i];
  const uint32_t x45 = dv[4][i] * 256u + dv[5][i];
  return fma(fma(i2d(x01), 65536.0, i2d(x23)), 65536.0, i2d(x45));
#endif
}

// exact int32 -> fp64 without I2F: 2^52 + 2^31 + x has x + 2^31 in its mantissa
__device__ __forceinline__ double i2d(uint32_t x) {
#ifdef NLD_OZ_I2F
  return (double)(int32_t)x;
#else
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
#endif
}

__host__ __device__ constexpr int gather_oz_smem() {
  return (kGTmemA ? 0 : kSl * kGA) + kGOpStages * kGBStage + kGRawStages * kGRaw;
}

// canonical K-major no-swizzle offset in a (rows x 64 bytes) tile
__device__ __forceinline__ int canon64(int row, int k) {
  return (row >> 3) * 512 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

__global__ void __launch_bounds__(kGatherThreads, kGCtas)
k_gather_oz(const SubDev* __restrict__ subs, const CellDev* __restrict__ cells,
            const WinDev* __restrict__ wins, const double* __restrict__ rows,
            const int32_t* __restrict__ pix, const int16_t* __restrict__ sub_exp,
            const double* __restrict__ grid, int64_t grid_ld, double* __restrict__ out,
            int64_t N, int nrhs, mma::GatherEpi ep) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t raw_full[kGRawStages], raw_empty[kGRawStages];
  __shared__ uint64_t op_ready[kGOpStages], op_free[kGOpStages];
  __shared__ uint64_t acc_full[kGAccBufs], acc_empty[kGAccBufs];
  __shared__ uint32_t taddr_s;
  __shared__ double gmax[2][kRows];
  __shared__ double tsc[kRows];           // T scale per row: 2^(eG + eY - 92 + 80)

  const SubDev sd = subs[blockIdx.x];
  const CellDev cd = cells[sd.cell];
  const WinDev wd = wins[sd.win];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int32_t* __restrict__ pw = pix + sd.start;
  const int16_t* ex = sub_exp + (int64_t)blockIdx.x * kExpPerSub;
  uint8_t* const sGA = smem;
  uint8_t* const sGB = sGA + (kGTmemA ? 0 : kSl * kGA);
  uint8_t* const sRaw = sGB + kGOpStages * kGBStage;
  const int ntile = (sd.count + kGTile - 1) / kGTile;
  const int ngroups = nrhs / 16;
  // Y scale: one per subproblem, |B_j[b] C_j[c]| < 2^(eBm + eCm)
  int eBm = -2000, eCm = -2000;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    eBm = max(eBm, (int)ex[8 + k]);
    eCm = max(eCm, (int)ex[16 + k]);
  }
  const double syB = pow2(46 - eBm), syC = pow2(-eCm);

  if (warp == 0) umma::tmem_alloc<kGTmemCols>(&taddr_s);
  if (tid == 32) {
    for (int k = 0; k < kGRawStages; ++k) {
      umma::mbar_init(&raw_full[k], 32);
      umma::mbar_init(&raw_empty[k], 2 + kGEpiWarps);   // slicer + epilogue warps
    }
    for (int k = 0; k < kGOpStages; ++k) {
      umma::mbar_init(&op_ready[k], 2);       // slicer warps
      umma::mbar_init(&op_free[k], 1);
    }
    for (int k = 0; k < kGAccBufs; ++k) {
      umma::mbar_init(&acc_full[k], 1);
      umma::mbar_init(&acc_empty[k], kGEpiWarps);
    }
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = taddr_s;

  int gt = 0;   // tiles processed so far over all rhs groups (phase bookkeeping)
  for (int grp = 0; grp < ngroups; ++grp) {
    const int rg = grp * 16;
    // ---- G digits of this rhs group (all warps) ---------------------------
    // thread t < 256: row m = t & 127 = (a, r), bc half h = t >> 7; two passes
    // over the (L2-resident) support box: the row max, then the digits
    const int m = tid & 127, h = (tid >> 7) & 1;
    const int ga = m & 7, gr = m >> 3;        // rows ordered (r, a): a fastest
    auto gval = [&](int bc) -> double {
      int p0 = cd.cc[0] + ga, p1 = cd.cc[1] + (bc >> 3), p2 = cd.cc[2] + (bc & 7);
      if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
      if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
      if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
      return grid[(int64_t)(rg + gr) * grid_ld + wd.grid_off +
                  ((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
    };
    if (tid < 256) {
      double mx = 0.0;
#pragma unroll 8
      for (int i = 0; i < 32; ++i) mx = fmax(mx, fabs(gval(h * 32 + i)));
      gmax[h][m] = mx;
    }
    __syncthreads();
    if (tid < 256) {
      // clamped like ev: the digit scale and tsc must use the same exponent
      const int eG = max(-900, exp_bound(fmax(gmax[0][m], gmax[1][m])));
      const double sg = pow2(46 - eG);
      if (h == 0) tsc[m] = ldexp(1.0, eG + eBm + eCm - 52);   // (eG-46)+(eBm+eCm-46)+80-16-24
#pragma unroll 1
      for (int kb = 0; kb < 2; ++kb) {
        uint32_t lo[16], hi[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) slice1(gval(h * 32 + kb * 16 + i), sg, lo[i], hi[i]);
        if constexpr (kGTmemA) {
          uint32_t w4[4][6];
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) pack4(lo + 4 * g4, hi + 4 * g4, w4[g4]);
          // lane m, 16 columns per digit slice (K = 64 bytes); this thread's
          // 16 values are columns h * 8 + kb * 4 .. + 3
          const uint32_t gt_addr = tmem + ((uint32_t)((m >> 5) * 32) << 16) +
                                   (uint32_t)(kGTmemA0 + h * 8 + kb * 4);
#pragma unroll
          for (int p = 0; p < kSl; ++p)
            umma::tmem_st4(gt_addr + (uint32_t)(p * 16), w4[0][p], w4[1][p], w4[2][p], w4[3][p]);
        } else {
          store16(lo, hi, sGA + canon64(m, h * 32 + kb * 16), kGA);
        }
      }
    }
    if constexpr (kGTmemA) umma::tmem_wait_st();
    umma::fence_async_smem();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();

#ifdef NLD_OZ_PROF
    const long long t_role = clock64();
#endif
    if (warp == kGLoaderWarp) {
      // -------------------------------------------------------------- loader
      for (int tl = 0; tl < ntile; ++tl) {
        const int g = gt + tl, s = g % kGRawStages;
        if (g >= kGRawStages) OZW(0, umma::mbar_wait(&raw_empty[s], ((g / kGRawStages) - 1) & 1));
        const int j0 = tl * kGTile, cn = min(kGTile, sd.count - j0);
        const double* src = rw + (int64_t)j0 * 24;
        uint8_t* dst = sRaw + s * kGRaw;
        for (int e = lane; e < cn * 12; e += 32) {
          const int node = e / 12, gi = e - node * 12;
          cp_async16(dst + node * kGRowS * 8 + 16 * gi, src + 2 * e);
        }
        if (lane < cn) cp_async4(dst + kGTile * kGRowS * 8 + 4 * lane, pw + j0 + lane);
        cp_async_mbar_arrive(&raw_full[s]);
      }
    } else if (warp == kGIssuerWarp) {
      // -------------------------------------------------------------- issuer
      for (int tl = 0; tl < ntile; ++tl) {
        const int g = gt + tl, st = g % kGOpStages, ab = g % kGAccBufs;
        if (g >= kGAccBufs) OZW(1, umma::mbar_wait(&acc_empty[ab], ((g / kGAccBufs) - 1) & 1));
        OZW(2, umma::mbar_wait(&op_ready[st], (g / kGOpStages) & 1));
        umma::fence_after();
        if (lane == 0) {
          const uint32_t aB = umma::smem_u32(sGA);
          const uint32_t bB = umma::smem_u32(sGB + st * kGBStage);
          const uint32_t dcol = tmem + (uint32_t)(ab * kSl * kGTile);
#ifndef NLD_EXP_GNOMMA
          // p outer, ks inner: the two K steps of one digit row hit the same D
          // window back to back and chain in the tensor pipe (a D window / N
          // change between every UMMA costs ~60% more: scripts/umma/probe_pattern.cu)
#pragma unroll
          for (int p = 0; p < kSl; ++p)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t db = umma::make_sdesc(bB + ks * 256, 128, 512);
              if constexpr (kGTmemA) {
                umma::mma_i8_ta(dcol + (uint32_t)(p * kGTile),
                                tmem + (uint32_t)(kGTmemA0 + p * 16 + ks * 8), db,
                                umma::idesc_i8(kRows, (kSl - p) * kGTile),
                                (ks > 0 || p > 0) ? 1u : 0u);
              } else {
                const uint64_t da = umma::make_sdesc(aB + p * kGA + ks * 256, 128, 512);
                umma::mma_i8(dcol + (uint32_t)(p * kGTile), da, db,
                             umma::idesc_i8(kRows, (kSl - p) * kGTile),
                             (ks > 0 || p > 0) ? 1u : 0u);
              }
            }
#endif
          umma::commit(&op_free[st]);
          umma::commit(&acc_full[ab]);
        }
        __syncwarp();
      }
    } else if (warp >= kGSlicerWarp0) {
      // ------------------------------------------------------------- slicers
      const int sw = warp - kGSlicerWarp0;     // 0..1
      const int kq = lane >> 3;                // bc quarter (16 values)
      for (int tl = 0; tl < ntile; ++tl) {
        const int g = gt + tl, s = g % kGRawStages, st = g % kGOpStages;
        OZW(3, umma::mbar_wait(&raw_full[s], (g / kGRawStages) & 1));
        if (g >= kGOpStages) OZW(4, umma::mbar_wait(&op_free[st], ((g / kGOpStages) - 1) & 1));
        uint8_t* sB = sGB + st * kGBStage;
#ifndef NLD_EXP_GNOSLICE
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          // 8 nodes per warp and pass; rows 26 doubles apart: conflict-free
          const int n = pass * 16 + sw * 8 + (lane & 7);
          const double* R = reinterpret_cast<const double*>(sRaw + s * kGRaw) + n * kGRowS;
          const bool ok = tl * kGTile + n < sd.count;
          uint32_t lo[16], hi[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int bc = kq * 16 + i;
            double x = 0.0, y = 0.0;
            if (ok) {
              x = R[8 + (bc >> 3)] * syB;
              y = R[16 + (bc & 7)] * syC;
            }
            slice1(x, y, lo[i], hi[i]);
          }
        store16(lo, hi, sB + canon64(n, kq * 16), kGB);
        }
#endif
        umma::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_ready[st]);
          mbar_arrive(&raw_empty[s]);
        }
      }
    } else {
      // ------------------------------------------------------------ epilogue
      // TMEM lane = row (r, a) with a fastest: the 8 a-rows of one rhs sit in
      // 8 adjacent lanes, so the sum over a is an in-warp butterfly that also
      // scatters the 8 nodes of a group over those lanes (lane a ends with
      // node a's sum) -- no shared-memory round trip, no named barriers
      const int lg = warp & 3, nh = warp >> 2;          // TMEM lane group, node half
      const int a = lane & 7, r = 4 * lg + (lane >> 3);
      const int mrow = lg * 32 + lane;
      const double ts = tsc[mrow];
      const uint32_t tl_lane = tmem + ((uint32_t)(lg * 32) << 16);
      const bool need_eta = ep.kind == NLD_APPLY_SYSTEM || ep.kind == NLD_APPLY_LAPLACIAN;
      for (int tl = 0; tl < ntile; ++tl) {
        const int g = gt + tl, ab = g % kGAccBufs, s = g % kGRawStages;
        const int j0 = tl * kGTile;
        umma::mbar_wait(&raw_full[s], (g / kGRawStages) & 1);
        const double* R = reinterpret_cast<const double*>(sRaw + s * kGRaw);
        const int32_t* sp = reinterpret_cast<const int32_t*>(sRaw + s * kGRaw + kGTile * kGRowS * 8);
        // this lane's two outputs: node nb + a of each 8-node group, rhs r
        int64_t oe[kGNodeGroups];
        double prev[kGNodeGroups], vx[kGNodeGroups], et[kGNodeGroups];
#pragma unroll
        for (int q = 0; q < kGNodeGroups; ++q) {
          const int nn = (nh * kGNodeGroups + q) * 8 + a;
          const bool ok = j0 + nn < sd.count;
          const int64_t px = ok ? (int64_t)sp[nn] : -1;
          oe[q] = ok ? px * nrhs + rg + r : -1;
          prev[q] = (ok && ep.mode >= mma::kGatherAccum) ? out[oe[q]] : 0.0;
          vx[q] = (ok && ep.mode == mma::kGatherFinal) ? ep.v[oe[q]] : 0.0;
          et[q] = (ok && ep.mode == mma::kGatherFinal && need_eta) ? ep.eta[px] : 0.0;
        }
        umma::mbar_wait(&acc_full[ab], (g / kGAccBufs) & 1);
        umma::fence_after();
        double ysum[kGNodeGroups];
#pragma unroll
        for (int q = 0; q < kGNodeGroups; ++q) {
          const int nb = (nh * kGNodeGroups + q) * 8;
          uint32_t dv[kSl][8];
#pragma unroll
          for (int tt = 0; tt < kSl; ++tt)
            umma::tmem_ld8(tl_lane + (uint32_t)(ab * kSl * kGTile + tt * kGTile + nb), dv[tt]);
          umma::tmem_wait_ld();
          if (q == kGNodeGroups - 1) {
            umma::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
          }
          double v8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)   // rows past the count are stale: never stored
            v8[i] = combine6(dv, i) * ts * R[(nb + i) * kGRowS + a];
          // butterfly reduce-scatter over the 8 a-lanes (lane bits 0..2)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool up = lane & 4;
            const double send = up ? v8[i] : v8[i + 4];
            const double keep = up ? v8[i + 4] : v8[i];
            v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const bool up = lane & 2;
            const double send = up ? v8[i] : v8[i + 2];
            const double keep = up ? v8[i + 2] : v8[i];
            v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          }
          {
            const bool up = lane & 1;
            const double send = up ? v8[0] : v8[1];
            const double keep = up ? v8[1] : v8[0];
            ysum[q] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&raw_empty[s]);
#pragma unroll
        for (int q = 0; q < kGNodeGroups; ++q) {
          if (oe[q] < 0) continue;
          const double y = ysum[q];
          double res;
          if (ep.mode == mma::kGatherStore || ep.mode == mma::kGatherFirst) {
            res = y;
          } else if (ep.mode == mma::kGatherAccum) {
            res = prev[q] + y;
          } else {
            const double lam = ep.coef ? ep.coef[2 * (rg + r)] : 0.0;
            const double mu = ep.coef ? ep.coef[2 * (rg + r) + 1] : 0.0;
            res = mma::epi_value(ep.kind, ep.L, prev[q] + y, vx[q], et[q], lam, mu);
          }
          out[oe[q]] = res;
        }
      }
    }
    gt += ntile;
    umma::fence_before();
    __syncthreads();      // G digits / tsc reused by the next rhs group
    umma::fence_after();
  }
  if (warp == 0) umma::tmem_free<kGTmemCols>(tmem);
}

// ---- plan-time Y digits for the sliced gather (GY) -------------------------
// Y_j[(b, c)] = B_j[b] C_j[c] scaled per subproblem (2^(46 - max eB - max eC),
// exactly the slicers' scaling), six K-major slices of each 32-node tile
// (32 nodes x 64 bytes, canonical layout), zero past the count.
__global__ void __launch_bounds__(128)
k_gather_ydig(const SubDev* __restrict__ subs, const WinDev* __restrict__ wins,
              const double* __restrict__ rows, const int16_t* __restrict__ sub_exp,
              const int64_t* __restrict__ ychunk, uint8_t* __restrict__ gydig) {
  const SubDev sd = subs[blockIdx.x];
  const WinDev wd = wins[sd.win];
  const double* __restrict__ rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
  const int16_t* ex = sub_exp + (int64_t)blockIdx.x * kExpPerSub;
  int eBm = -2000, eCm = -2000;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    eBm = max(eBm, (int)ex[8 + q]);
    eCm = max(eCm, (int)ex[16 + q]);
  }
  const double syB = pow2(46 - eBm), syC = pow2(-eCm);
  const int t = threadIdx.x, n = t >> 2, kq = t & 3;     // node, bc quarter
  const int ntile = (sd.count + kGTile - 1) / kGTile;
  uint8_t* base = gydig + ychunk[blockIdx.x] * (int64_t)(kSl * kGB);
  for (int tl = 0; tl < ntile; ++tl) {
    const int j = tl * kGTile + n;
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int bc = kq * 16 + i;
      double x = 0.0, y = 0.0;
      if (j < sd.count) {
        x = rw[(int64_t)j * 24 + 8 + (bc >> 3)] * syB;
        y = rw[(int64_t)j * 24 + 16 + (bc & 7)] * syC;
      }
      slice1(x, y, lo[i], hi[i]);
    }
    store16(lo, hi, base + (int64_t)tl * (kSl * kGB) + canon64(n, kq * 16), kGB);
  }
}

// ---- G digits of every cell, once per product (persistent gather) ----------
// Per (cell, 16-rhs group): the 128 rows (r, a) x 64 (b, c) of the support-box
// grid at the cell, scaled per rhs (max over its 8 a-rows and 64 values) and
// cut into six digit slices in the UMMA A-operand layout (canonical K-major,
// 6 x 8 KB), followed by the 128 row exponents (int32).  Massively parallel
// (every cell at once), so the gather's per-subproblem G setup becomes one
// 48 KB TMA load that the pipeline prefetches a subproblem ahead.
constexpr int kGdigBytes = kSl * kGA + kRows * 4;

__global__ void __launch_bounds__(kRows)
k_gdig(const CellDev* __restrict__ cells, const WinDev* __restrict__ wins,
       const double* __restrict__ grid, int64_t grid_ld, int64_t cell_lo, int ngroups,
       uint8_t* __restrict__ gdig) {
  const int64_t cell = cell_lo + blockIdx.x;
  const int grp = blockIdx.y, rg = grp * 16;
  const CellDev cd = cells[cell];
  const WinDev wd = wins[cd.win];
  const int m = threadIdx.x, ga = m & 7, gr = m >> 3;
  auto gval = [&](int bc) -> double {
    int p0 = cd.cc[0] + ga, p1 = cd.cc[1] + (bc >> 3), p2 = cd.cc[2] + (bc & 7);
    if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
    if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
    if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
    return grid[(int64_t)(rg + gr) * grid_ld + wd.grid_off +
                ((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
  };
  double g[64];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    g[i] = gval(i);
    mx = fmax(mx, fabs(g[i]));
  }
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
  mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  const int eG = max(-900, exp_bound(mx));
  const double sg = pow2(46 - eG);
  uint8_t* base = gdig + (cell * ngroups + grp) * (int64_t)kGdigBytes;
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) slice1(g[kb * 16 + i], sg, lo[i], hi[i]);
    store16(lo, hi, base + canon64(m, kb * 16), kGA);
  }
  reinterpret_cast<int32_t*>(base + kSl * kGA)[m] = eG;
}

// ---- persistent gather -----------------------------------------------------
// One CTA per SM walks a list of work items (subproblem, rhs group): the
// subproblems in descending node count, dealt to the CTAs in snake order so
// every CTA gets a near-equal share.  All warp roles stream across item
// boundaries; the G digits are double-buffered in shared memory, so the
// slicer warps cut item k+1's G while the issuer and the epilogue finish item
// k -- no per-subproblem launch, TMEM allocation, pipeline fill or drain (the
// fixed cost that grows when pixel sharding makes subproblems small).
//   warps 0-7  epilogue       warps 8-11 slicers (G digits + Y digits)
//   warp 12    UMMA issuer    warp 13    loader
#ifndef NLD_GP_EPI
#define NLD_GP_EPI 16
#endif
constexpr int kPEpi = NLD_GP_EPI;                // 8 or 16 epilogue warps
constexpr int kPG = 16 / kPEpi;                  // 8-node groups per epilogue warp and tile
constexpr int kPSl0 = kPEpi;
constexpr int kPSlicers = 4;
constexpr int kPIssuer = kPEpi + 4;
constexpr int kPLoader = kPEpi + 5;
constexpr int kPThreads = 32 * (kPEpi + 6);
#ifndef NLD_GP_RS
#define NLD_GP_RS 6
#endif
#ifndef NLD_GP_OS
#define NLD_GP_OS 3
#endif
constexpr int kPRS = NLD_GP_RS, kPOS = NLD_GP_OS;   // raw / operand stages
#ifndef NLD_GP_GTMEM
#define NLD_GP_GTMEM 1      // G digits copied to TMEM per item (UMMA A from TMEM)
#endif

__host__ __device__ constexpr int gather_ozp_smem() {
  return 2 * kSl * kGA + kPOS * kGBStage + kPRS * kGRaw;
}
// plan-time Y digits (GY): no operand stages; each raw stage carries the
// tile's 12 KB of Y digits after its rows and pixel indices
// (GY: only the A parts of the weight rows are staged -- 8 doubles per node --
// then the pixel indices, then the Y digits)
constexpr int kGYRowS = 8;
constexpr int kGYOff = kGTile * kGYRowS * 8 + kGTile * 4;       // 2 KB + 128 B
constexpr int kGRawGY = kGYOff + kSl * kGB;
__host__ __device__ constexpr int gather_ozp_gy_smem() { return 2 * kSl * kGA + kPRS * kGRawGY; }

template <bool GY>
__global__ void __launch_bounds__(kPThreads, 1)
k_gather_ozp(const SubDev* __restrict__ subs, const int32_t* __restrict__ order, int nsub,
             const CellDev* __restrict__ cells, const WinDev* __restrict__ wins,
             const double* __restrict__ rows, const int32_t* __restrict__ pix,
             const int16_t* __restrict__ sub_exp, const double* __restrict__ grid,
             int64_t grid_ld, double* __restrict__ out, int64_t N, int nrhs, mma::GatherEpi ep,
             const uint8_t* __restrict__ gdig, const uint8_t* __restrict__ gydig,
             const int64_t* __restrict__ ychunk) {
  constexpr int RS = kPRS, OS = kPOS;              // raw / operand stages
  constexpr int kRawB = GY ? kGRawGY : kGRaw;      // raw stage bytes
  constexpr int kRowS = GY ? kGYRowS : kGRowS;     // doubles per staged node row
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint64_t raw_full[RS], raw_empty[RS], op_ready[OS], op_free[OS];
  __shared__ uint64_t acc_full[2], acc_empty[2], g_full[2], g_empty[2];
  __shared__ uint32_t taddr_s;
  __shared__ double tsc[2][kRows];
  __shared__ __align__(16) int32_t gexs[2][kRows];   // precomputed-G row exponents

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* const sGA = smem;                                    // [2][6][128 x 64]
  uint8_t* const sGB = sGA + 2 * kSl * kGA;                     // [3][6][32 x 64]
  uint8_t* const sRaw = sGB + (GY ? 0 : OS * kGBStage);         // [6][rows | pix (| Y)]
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
    for (int k = 0; k < RS; ++k) {
      // GY: 32 noinc cp.async arrivals + the Y bulk copy's; released by the
      // epilogue warps and the tile's UMMA commit (no slicer pass over Y)
      umma::mbar_init(&raw_full[k], GY ? 33 : 32);
      umma::mbar_init(&raw_empty[k], GY ? kPEpi + 1 : kPSlicers + kPEpi);
    }
    for (int k = 0; k < OS; ++k) {
      umma::mbar_init(&op_ready[k], kPSlicers);
      umma::mbar_init(&op_free[k], 1);
    }
    for (int k = 0; k < 2; ++k) {
      umma::mbar_init(&acc_full[k], 1);
      umma::mbar_init(&acc_empty[k], kPEpi);
      umma::mbar_init(&g_full[k], gdig ? 1 : kPSlicers);   // TMA arrival / slicer warps
      umma::mbar_init(&g_empty[k], 1 + kPEpi);     // last MMA commit + epilogue warps
    }
    umma::mbar_fence_init();
  }
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = taddr_s;
#ifdef NLD_OZ_PROF
  const long long t_role = clock64();
#endif

  if (warp == kPLoader) {
    // ---------------------------------------------------------------- loader
    int gt = 0;
    for (int k = 0; k < nitems; ++k) {
      const SubDev sd = subs[item_sub(k)];
      const WinDev wd = wins[sd.win];
      const double* rw = rows + wd.row_off + (sd.start - wd.node_off) * 24;
      const int32_t* pw = pix + sd.start;
      const int ntile = (sd.count + kGTile - 1) / kGTile;
      const uint8_t* gyd = GY ? gydig + ychunk[item_sub(k)] * (int64_t)(kSl * kGB) : nullptr;
      for (int tl = 0; tl < ntile; ++tl, ++gt) {
        const int s = gt % RS;
        if (gt >= RS) OZW(0, umma::mbar_wait(&raw_empty[s], ((gt / RS) - 1) & 1));
        const int j0 = tl * kGTile, cn = min(kGTile, sd.count - j0);
        const double* src = rw + (int64_t)j0 * 24;
        uint8_t* dst = sRaw + s * kRawB;
        if constexpr (GY) {
          if (lane == 0) {
            umma::mbar_arrive_expect_tx(&raw_full[s], kSl * kGB);
            umma::bulk_g2s(dst + kGYOff, gyd + (int64_t)tl * (kSl * kGB), kSl * kGB, &raw_full[s]);
          }
        }
#ifndef NLD_EXP_PNOLOAD
        if constexpr (GY) {
          // A parts only: 4 lanes per node's 64 bytes, 8 nodes per instruction
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int nd = q * 8 + (lane >> 2), pc = lane & 3;
            if (nd < cn) cp_async16(dst + nd * 64 + pc * 16, src + (int64_t)nd * 24 + 2 * pc);
          }
        } else {
          for (int e = lane; e < cn * 12; e += 32) {
            const int node = e / 12, gi = e - node * 12;
            cp_async16(dst + node * kGRowS * 8 + 16 * gi, src + 2 * e);
          }
        }
#endif
        if (lane < cn) cp_async4(dst + kGTile * kRowS * 8 + 4 * lane, pw + j0 + lane);
        cp_async_mbar_arrive(&raw_full[s]);
      }
    }
  } else if (warp == kPIssuer) {
    // ---------------------------------------------------------------- issuer
    int gt = 0;
    for (int k = 0; k < nitems; ++k) {
      const int gs = k & 1;
      const SubDev sd = subs[item_sub(k)];
      const int ntile = (sd.count + kGTile - 1) / kGTile;
      OZW(9, umma::mbar_wait(&g_full[gs], (k >> 1) & 1));
#if NLD_GP_GTMEM
      // item k's G digits: shared-memory staging -> TMEM (the UMMA A operand,
      // read from TMEM instead of shared memory by every tile's 12 UMMAs).
      // tcgen05.cp runs in issue order behind item k-1's UMMAs, so the copy
      // never overwrites digits still being read; its commit frees the staging
      umma::fence_after();
      if (lane == 0) {
        const uint32_t aB = umma::smem_u32(sGA + gs * kSl * kGA);
#pragma unroll
        for (int p = 0; p < kSl; ++p)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            umma::tmem_cp_128x256b(tmem + (uint32_t)(kGTmemA0 + p * 16 + ks * 8),
                                   umma::make_sdesc(aB + p * kGA + ks * 256, 128, 512));
        umma::commit(&g_empty[gs]);
      }
      __syncwarp();
#endif
      for (int tl = 0; tl < ntile; ++tl, ++gt) {
        const int st = gt % OS, ab = gt & 1;
        if (gt >= 2) OZW(1, umma::mbar_wait(&acc_empty[ab], ((gt >> 1) - 1) & 1));
        const int s = gt % RS;
        if constexpr (GY) OZW(2, umma::mbar_wait(&raw_full[s], (gt / RS) & 1));   // Y landed
        else OZW(2, umma::mbar_wait(&op_ready[st], (gt / OS) & 1));
        umma::fence_after();
        if (lane == 0) {
          const uint32_t aB = umma::smem_u32(sGA + gs * kSl * kGA);
          const uint32_t bB = GY ? umma::smem_u32(sRaw + s * kRawB + kGYOff)
                                 : umma::smem_u32(sGB + st * kGBStage);
          const uint32_t dcol = tmem + (uint32_t)(ab * kSl * kGTile);
          // p outer, ks inner: the two K steps of one digit row hit the same D
          // window back to back and chain in the tensor pipe (a D window / N
          // change between every UMMA costs ~60% more: scripts/umma/probe_pattern.cu)
#ifndef NLD_EXP_PNOMMA
#pragma unroll
          for (int p = 0; p < kSl; ++p)
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint64_t db = umma::make_sdesc(bB + ks * 256, 128, 512);
#if NLD_GP_GTMEM
              umma::mma_i8_ta(dcol + (uint32_t)(p * kGTile),
                              tmem + (uint32_t)(kGTmemA0 + p * 16 + ks * 8), db,
                              umma::idesc_i8(kRows, (kSl - p) * kGTile),
                              (ks > 0 || p > 0) ? 1u : 0u);
#else
              const uint64_t da = umma::make_sdesc(aB + p * kGA + ks * 256, 128, 512);
              umma::mma_i8(dcol + (uint32_t)(p * kGTile), da, db,
                           umma::idesc_i8(kRows, (kSl - p) * kGTile), (ks > 0 || p > 0) ? 1u : 0u);
#endif
            }
#endif
          if constexpr (GY) umma::commit(&raw_empty[s]);   // Y digits consumed
          else umma::commit(&op_free[st]);
          umma::commit(&acc_full[ab]);
#if !NLD_GP_GTMEM
          if (tl == ntile - 1) umma::commit(&g_empty[gs]);   // item k's G digits released
#endif
        }
        __syncwarp();
      }
    }
  } else if (warp >= kPSl0) {
    // ------------------------------------------- slicers: G digits, Y digits
    const int t = tid - 32 * kPSl0;            // 0..127
    int gt = 0;
    for (int k = 0; k < nitems; ++k) {
      const int gs = k & 1;
      const int si = item_sub(k);
      const SubDev sd = subs[si];
      const CellDev cd = cells[sd.cell];
      const WinDev wd = wins[sd.win];
      const int16_t* ex = sub_exp + (int64_t)si * kExpPerSub;
      const int rg = (k % ngroups) * 16;
      const int ntile = (sd.count + kGTile - 1) / kGTile;
      int eBm = -2000, eCm = -2000;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        eBm = max(eBm, (int)ex[8 + q]);
        eCm = max(eCm, (int)ex[16 + q]);
      }
      const double syB = pow2(46 - eBm), syC = pow2(-eCm);
      if (gdig) {
        // precomputed G digits (k_gdig): one thread loads them with TMA into
        // the staging buffer, a subproblem ahead of the MMAs
        if (t == 0) {
          if (k >= 2) OZW(5, umma::mbar_wait(&g_empty[gs], ((k >> 1) - 1) & 1));
          const uint8_t* src = gdig + ((int64_t)sd.cell * ngroups + (k % ngroups)) * kGdigBytes;
          umma::mbar_arrive_expect_tx(&g_full[gs], (uint32_t)(kSl * kGA + kRows * 4));
#pragma unroll
          for (int p = 0; p < kSl; ++p)
            umma::bulk_g2s(sGA + gs * kSl * kGA + p * kGA, src + p * kGA, kGA, &g_full[gs]);
          umma::bulk_g2s(&gexs[gs][0], src + kSl * kGA, kRows * 4, &g_full[gs]);
        }
      } else {
      if (k >= 2) OZW(5, umma::mbar_wait(&g_empty[gs], ((k >> 1) - 1) & 1));
      {
        // G digits: row m = (r, a) = t, its 64 (b, c) from the support box
        const int m = t, ga = m & 7, gr = m >> 3;
        auto gval = [&](int bc) -> double {
          int p0 = cd.cc[0] + ga, p1 = cd.cc[1] + (bc >> 3), p2 = cd.cc[2] + (bc & 7);
          if (p0 >= wd.box_w[0]) p0 -= wd.box_w[0];
          if (p1 >= wd.box_w[1]) p1 -= wd.box_w[1];
          if (p2 >= wd.box_w[2]) p2 -= wd.box_w[2];
          return grid[(int64_t)(rg + gr) * grid_ld + wd.grid_off +
                      ((int64_t)p0 * wd.box_w[1] + p1) * wd.box_w[2] + p2];
        };
        double mx = 0.0;
#ifndef NLD_EXP_PNOG
#pragma unroll 16
        for (int i = 0; i < 64; ++i) mx = fmax(mx, fabs(gval(i)));
#endif
        // one scale per rhs (max over its 8 a-rows, adjacent lanes): the
        // epilogue scales once per output, after the sum over a
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        const int eG = max(-900, exp_bound(mx));
        const double sg = pow2(46 - eG);
        tsc[gs][m] = ldexp(1.0, eG + eBm + eCm - 52);   // combine6 carries 2^24
        uint8_t* dA = sGA + gs * kSl * kGA;
#pragma unroll 1
        for (int kb = 0; kb < 4; ++kb) {
          uint32_t lo[16], hi[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) slice1(gval(kb * 16 + i), sg, lo[i], hi[i]);
          store16(lo, hi, dA + canon64(m, kb * 16), kGA);
        }
        umma::fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&g_full[gs]);
      }
      }
      if constexpr (GY) continue;   // Y digits come precomputed with the raw stage
      // Y digits of each tile: 8 nodes per warp, node = lane & 7, bc quarter
      // kq = lane >> 3, so each quarter-warp's 16-byte stores cover one
      // contiguous 128-byte line (conflict-free)
      const int n = (t >> 5) * 8 + (lane & 7), kq = lane >> 3;
      for (int tl = 0; tl < ntile; ++tl, ++gt) {
        const int s = gt % RS, st = gt % OS;
        OZW(3, umma::mbar_wait(&raw_full[s], (gt / RS) & 1));
        if (gt >= OS) OZW(4, umma::mbar_wait(&op_free[st], ((gt / OS) - 1) & 1));
#ifndef NLD_EXP_PNOSLICE
        const double* R = reinterpret_cast<const double*>(sRaw + s * kRawB) + n * kGRowS;
        const bool ok = tl * kGTile + n < sd.count;
        uint32_t lo[16], hi[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int bc = kq * 16 + i;
          double x = 0.0, y = 0.0;
          if (ok) {
            x = R[8 + (bc >> 3)] * syB;
            y = R[16 + (bc & 7)] * syC;
          }
          slice1(x, y, lo[i], hi[i]);
        }
        store16(lo, hi, sGB + st * kGBStage + canon64(n, kq * 16), kGB);
#endif
        umma::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&op_ready[st]);
          mbar_arrive(&raw_empty[s]);
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int lg = warp & 3, nh = warp >> 2;
    const int a = lane & 7, r = 4 * lg + (lane >> 3);
    const int mrow = lg * 32 + lane;
    const uint32_t tl_lane = tmem + ((uint32_t)(lg * 32) << 16);
    const bool need_eta = ep.kind == NLD_APPLY_SYSTEM || ep.kind == NLD_APPLY_LAPLACIAN;
    const double inv_L = 1.0 / (double)ep.L;
    // The running window sum, v and eta of a tile's pixels are scattered
    // global loads: they are issued one tile ahead (software pipeline over
    // the flat tile sequence, across item boundaries), so their latency
    // hides behind the current tile's TMEM drain instead of stalling it.
    struct EpiIn {
      int64_t oe[kPG];
      double prev[kPG], vx[kPG], et[kPG];
    };
    // (count, rhs group) of the tile's item are passed in: the item's SubDev
    // is read once per item, one item ahead, not per tile
    auto epi_load = [&](int cnt, int rgn, int tt, int gg) {
      EpiIn e;
      const int sn = gg % RS;
      OZW(7, umma::mbar_wait(&raw_full[sn], (gg / RS) & 1));
      const int32_t* spn = reinterpret_cast<const int32_t*>(sRaw + sn * kRawB + kGTile * kRowS * 8);
#pragma unroll
      for (int q = 0; q < kPG; ++q) {
        const int nn = (nh * kPG + q) * 8 + a;
        const bool ok = tt * kGTile + nn < cnt;
#ifdef NLD_EXP_CONTIG_G
        const int64_t px = ok ? (int64_t)(tt * kGTile + nn) : -1;   // timing experiment only
#else
        const int64_t px = ok ? (int64_t)spn[nn] : -1;
#endif
        e.oe[q] = ok ? px * nrhs + rgn + r : -1;
#ifdef NLD_EXP_PNOGLD
        e.prev[q] = e.vx[q] = e.et[q] = 0.0;   // timing experiment only
#else
        e.prev[q] = (ok && ep.mode >= mma::kGatherAccum) ? out[e.oe[q]] : 0.0;
        e.vx[q] = (ok && ep.mode == mma::kGatherFinal) ? ep.v[e.oe[q]] : 0.0;
        e.et[q] = (ok && ep.mode == mma::kGatherFinal && need_eta) ? ep.eta[px] : 0.0;
#endif
      }
      return e;
    };
    EpiIn nxt;
    int cnt_next = 0;
    if (nitems > 0) {
      cnt_next = subs[item_sub(0)].count;
      nxt = epi_load(cnt_next, 0, 0, 0);
    }
    int gt = 0;
    for (int k = 0; k < nitems; ++k) {
      const int gs = k & 1;
      const int cnt = cnt_next;
      if (k + 1 < nitems) cnt_next = subs[item_sub(k + 1)].count;
      const int rg = (k % ngroups) * 16;
      const int ntile = (cnt + kGTile - 1) / kGTile;
      // this lane's rhs coefficients, once per item
      const double lam_r = (ep.mode == mma::kGatherFinal && ep.coef) ? ep.coef[2 * (rg + r)] : 0.0;
      const double mu_r = (ep.mode == mma::kGatherFinal && ep.coef) ? ep.coef[2 * (rg + r) + 1] : 0.0;
      OZW(6, umma::mbar_wait(&g_full[gs], (k >> 1) & 1));
      double ts;
      if (gdig) {
        // T scale of the row: G exponent (per rhs) + the subproblem's Y exponents
        const int16_t* exk = sub_exp + (int64_t)item_sub(k) * kExpPerSub;
        int eBm = -2000, eCm = -2000;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          eBm = max(eBm, (int)exk[8 + q]);
          eCm = max(eCm, (int)exk[16 + q]);
        }
        ts = ldexp(1.0, gexs[gs][mrow] + eBm + eCm - 52);
      } else {
        ts = tsc[gs][mrow];
      }
      for (int tl = 0; tl < ntile; ++tl, ++gt) {
        const int ab = gt & 1, s = gt % RS;
        const double* R = reinterpret_cast<const double*>(sRaw + s * kRawB);
        const EpiIn cur = nxt;
        if (tl + 1 < ntile) nxt = epi_load(cnt, rg, tl + 1, gt + 1);
        else if (k + 1 < nitems) nxt = epi_load(cnt_next, ((k + 1) % ngroups) * 16, 0, gt + 1);
        const int64_t* oe = cur.oe;
        const double *prev = cur.prev, *vx = cur.vx, *et = cur.et;
        OZW(8, umma::mbar_wait(&acc_full[ab], (gt >> 1) & 1));
        umma::fence_after();
        double ysum[kPG];
#pragma unroll
        for (int q = 0; q < kPG; ++q) {
          const int nb = (nh * kPG + q) * 8;
          uint32_t dv[kSl][8];
#pragma unroll
          for (int tt = 0; tt < kSl; ++tt)
#ifndef NLD_EXP_PNOTLD
            umma::tmem_ld8(tl_lane + (uint32_t)(ab * kSl * kGTile + tt * kGTile + nb), dv[tt]);
#else
            dv[tt][0] = tt;
#endif
          umma::tmem_wait_ld();
          if (q == kPG - 1) {
            umma::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[ab]);
          }
          double v8[8];
#ifdef NLD_EXP_PNOEPI
#pragma unroll
          for (int i = 0; i < 8; ++i) v8[i] = (double)(int)dv[i % 6][i];
#else
#pragma unroll
          for (int i = 0; i < 8; ++i)
            v8[i] = combine6(dv, i) * R[(nb + i) * kRowS + a];
#endif
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const bool up = lane & 4;
            const double send = up ? v8[i] : v8[i + 4];
            const double keep = up ? v8[i + 4] : v8[i];
            v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const bool up = lane & 2;
            const double send = up ? v8[i] : v8[i + 2];
            const double keep = up ? v8[i + 2] : v8[i];
            v8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          }
          {
            const bool up = lane & 1;
            const double send = up ? v8[0] : v8[1];
            const double keep = up ? v8[1] : v8[0];
            ysum[q] = (keep + __shfl_xor_sync(0xffffffffu, send, 1)) * ts;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&raw_empty[s]);
#pragma unroll
        for (int q = 0; q < kPG; ++q) {
          if (oe[q] < 0) continue;
          const double y = ysum[q];
          double res;
          if (ep.mode == mma::kGatherStore || ep.mode == mma::kGatherFirst) {
            res = y;
          } else if (ep.mode == mma::kGatherAccum) {
            res = prev[q] + y;
          } else {
            res = mma::epi_value_r(ep.kind, (double)ep.L, inv_L, prev[q] + y, vx[q], et[q], lam_r,
                                   mu_r);
          }
#ifndef NLD_EXP_PNOGST
          out[oe[q]] = res;
#else
          if (res == 1.2345e-300) out[oe[q]] = res;   // timing experiment only
#endif
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&g_empty[gs]);   // tsc[gs] no longer read
    }
  }
#ifdef NLD_OZ_PROF
  if (lane == 0)
    atomicAdd(&oz_prof[24 + (warp == kPLoader ? 0 : warp == kPIssuer ? 1 : warp >= kPSl0 ? 2 : 3)],
              (unsigned long long)(clock64() - t_role));
#endif
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<512>(tmem);
}

}  // namespace oz

// ---- host side ------------------------------------------------------------

// integer-sliced tensor-core path: on by default for its shapes (3-D windows,
// m = 4, rhs batches of 16k); NLD_OZAKI=0 selects the fp64 DMMA kernels
bool use_ozaki() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("NLD_OZAKI");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int16_t* ozaki_exponents(PlanSet& ps, cudaStream_t st) {
  if (ps.sub_exp || ps.n_subs[3] == 0) return ps.sub_exp;
  NLD_CUDA(cudaMalloc(&ps.sub_exp, sizeof(int16_t) * oz::kExpPerSub * ps.n_subs[3]));
  oz::k_sub_exponents<<<(unsigned)ps.n_subs[3], 240, 0, st>>>(ps.subs[3], ps.wdev, ps.rows,
                                                               ps.sub_exp);
  NLD_CUDA(cudaGetLastError());
  // per window, its 3-D subproblems in descending node count (window-local
  // indices): the persistent gather deals them out in snake order
  std::vector<SubDev> h(ps.n_subs[3]);
  NLD_CUDA(cudaMemcpyAsync(h.data(), ps.subs[3], sizeof(SubDev) * h.size(), cudaMemcpyDeviceToHost,
                           st));
  NLD_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> ord(h.size());
  for (const WinPlan& wp : ps.win) {
    if (wp.d != 3 || wp.n_subs == 0) continue;
    int32_t* o = ord.data() + wp.sub_off;
    for (int64_t i = 0; i < wp.n_subs; ++i) o[i] = (int32_t)i;
    const SubDev* hs = h.data() + wp.sub_off;
    std::stable_sort(o, o + wp.n_subs,
                     [&](int32_t x, int32_t y) { return hs[x].count > hs[y].count; });
  }
  NLD_CUDA(cudaMalloc(&ps.sub_order, sizeof(int32_t) * ord.size()));
  NLD_CUDA(cudaMemcpyAsync(ps.sub_order, ord.data(), sizeof(int32_t) * ord.size(),
                           cudaMemcpyHostToDevice, st));
  // per window: the global index range of its cells (contiguous per window)
  ps.gcell_lo.assign(ps.win.size(), 0);
  ps.gcell_n.assign(ps.win.size(), 0);
  for (size_t w = 0; w < ps.win.size(); ++w) {
    const WinPlan& wp = ps.win[w];
    if (wp.d != 3 || wp.n_subs == 0) continue;
    int64_t lo = INT64_MAX, hi = -1;
    for (int64_t i = 0; i < wp.n_subs; ++i) {
      lo = std::min<int64_t>(lo, h[wp.sub_off + i].cell);
      hi = std::max<int64_t>(hi, h[wp.sub_off + i].cell);
    }
    ps.gcell_lo[w] = lo;
    ps.gcell_n[w] = hi - lo + 1;
  }
  // precomputed Y digits for the spread (12 KB per 32-node chunk) when they
  // fit comfortably: at most half of the free memory (NLD_SPREAD_PREY=0: off)
  const char* py = getenv("NLD_SPREAD_PREY");
  if (!(py && py[0] == '0')) {
    std::vector<int64_t> off(h.size());
    int64_t chunks = 0;
    for (size_t i = 0; i < h.size(); ++i) {
      off[i] = chunks;
      chunks += (h[i].count + oz::kChunk - 1) / oz::kChunk;
    }
    const size_t need = (size_t)chunks * oz::kYChunkBytes;
    size_t free_b = 0, total_b = 0;
    NLD_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (need > 0 && need <= free_b / 2) {
      NLD_CUDA(cudaMalloc(&ps.ychunk, sizeof(int64_t) * off.size()));
      NLD_CUDA(cudaMalloc(&ps.ydig, need));
      NLD_CUDA(cudaMemcpyAsync(ps.ychunk, off.data(), sizeof(int64_t) * off.size(),
                               cudaMemcpyHostToDevice, st));
      oz::k_spread_ydig<<<(unsigned)h.size(), 256, 0, st>>>(ps.subs[3], ps.wdev, ps.rows,
                                                            ps.sub_exp, ps.ychunk, ps.ydig);
      NLD_CUDA(cudaGetLastError());
      // the gather's Y digits (same chunking, K-major per node): when a second
      // table of the same size still fits in half of the free memory
      const char* gy = getenv("NLD_GATHER_PREY");
      size_t free2 = 0;
      NLD_CUDA(cudaMemGetInfo(&free2, &total_b));
      if (!(gy && gy[0] == '0') && need <= free2 / 2) {
        NLD_CUDA(cudaMalloc(&ps.gydig, need));
        oz::k_gather_ydig<<<(unsigned)h.size(), 128, 0, st>>>(ps.subs[3], ps.wdev, ps.rows,
                                                              ps.sub_exp, ps.ychunk, ps.gydig);
        NLD_CUDA(cudaGetLastError());
      }
    }
  }
  NLD_CUDA(cudaStreamSynchronize(st));
  return ps.sub_exp;
}

void launch_spread_oz(const PlanSet& ps, const SubDev* subs, const int16_t* ex,
                      const int64_t* ychunk, unsigned nsub, const unsigned long long* vmax,
                      const double* vt, int nrhs, double* blocks, cudaStream_t st,
                      const int32_t* order) {
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(oz::k_spread_oz<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  oz::spread_oz_smem()));
    NLD_CUDA(cudaFuncSetAttribute(oz::k_spread_oz<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  oz::spread_oz_py_smem()));
    attr = true;
  }
  static int persist = -1;
  static int sms = 148;
  if (persist < 0) {
    const char* e = getenv("NLD_SPREAD_PERSIST");
    persist = (e && e[0] == '0') ? 0 : 1;
    int dev = 0;
    NLD_CUDA(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    NLD_CUDA(cudaFuncSetAttribute(oz::k_spread_ozp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  oz::spread_oz_py_smem()));
  }
  if (ps.ydig && ychunk && order && persist) {
    const unsigned grid_n = std::min<unsigned>(nsub, (unsigned)sms);
    oz::k_spread_ozp<<<grid_n, oz::kSPThreads, oz::spread_oz_py_smem(), st>>>(
        subs, order, (int)nsub, ps.wdev, ps.rows, ps.pix, ex, ps.ydig, ychunk, vmax, vt, nrhs,
        blocks);
  } else if (ps.ydig && ychunk)
    oz::k_spread_oz<true><<<nsub, oz::kSpreadThreads, oz::spread_oz_py_smem(), st>>>(
        subs, ps.wdev, ps.rows, ps.pix, ex, ps.ydig, ychunk, vmax, vt, nrhs, blocks);
  else
    oz::k_spread_oz<false><<<nsub, oz::kSpreadThreads, oz::spread_oz_smem(), st>>>(
        subs, ps.wdev, ps.rows, ps.pix, ex, nullptr, nullptr, vmax, vt, nrhs, blocks);
  NLD_CUDA(cudaGetLastError());
}

int64_t gather_gdig_bytes() { return oz::kGdigBytes; }

void launch_gather_oz(const PlanSet& ps, const SubDev* subs, const int16_t* ex,
                      const int32_t* order, unsigned nsub, const double* grid, int64_t grid_ld,
                      double* out, int64_t N, int nrhs, const mma::GatherEpi& ep,
                      cudaStream_t st, uint8_t* gdig, int64_t cell_lo, int64_t ncell,
                      const int64_t* ychunk) {
  static int persist = -1;
  if (persist < 0) {
    const char* e = getenv("NLD_GATHER_PERSIST");
    persist = (e && e[0] == '0') ? 0 : 1;
  }
  if (persist && order) {
    const int smem_p = oz::gather_ozp_smem();
    static bool attr_p = false;
    static int sms = 148;
    if (!attr_p) {
      NLD_CUDA(cudaFuncSetAttribute(oz::k_gather_ozp<false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p));
      NLD_CUDA(cudaFuncSetAttribute(oz::k_gather_ozp<true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    oz::gather_ozp_gy_smem()));
      int dev = 0;
      NLD_CUDA(cudaGetDevice(&dev));
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      attr_p = true;
    }
    const unsigned grid_n = std::min<unsigned>(nsub, (unsigned)sms);
    static int pre = -1;
    if (pre < 0) {
      const char* e = getenv("NLD_GATHER_PREG");
      pre = (e && e[0] == '0') ? 0 : 1;
    }
    const bool use_g = pre && gdig && ncell > 0;
    if (use_g) {
      oz::k_gdig<<<dim3((unsigned)ncell, (unsigned)(nrhs / 16)), oz::kRows, 0, st>>>(
          ps.cells, ps.wdev, grid, grid_ld, cell_lo, nrhs / 16, gdig);
      NLD_CUDA(cudaGetLastError());
    }
    if (ps.gydig && ychunk)
      oz::k_gather_ozp<true><<<grid_n, oz::kPThreads, oz::gather_ozp_gy_smem(), st>>>(
          subs, order, (int)nsub, ps.cells, ps.wdev, ps.rows, ps.pix, ex, grid, grid_ld, out, N,
          nrhs, ep, use_g ? gdig : nullptr, ps.gydig, ychunk);
    else
      oz::k_gather_ozp<false><<<grid_n, oz::kPThreads, smem_p, st>>>(
          subs, order, (int)nsub, ps.cells, ps.wdev, ps.rows, ps.pix, ex, grid, grid_ld, out, N,
          nrhs, ep, use_g ? gdig : nullptr, nullptr, nullptr);
    NLD_CUDA(cudaGetLastError());
    return;
  }
  const int smem = oz::gather_oz_smem();
  static bool attr = false;
  if (!attr) {
    NLD_CUDA(cudaFuncSetAttribute(oz::k_gather_oz, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    attr = true;
  }
  oz::k_gather_oz<<<nsub, oz::kGatherThreads, smem, st>>>(subs, ps.cells, ps.wdev, ps.rows, ps.pix,
                                                          ex, grid, grid_ld, out, N, nrhs, ep);
  NLD_CUDA(cudaGetLastError());
}

#ifdef NLD_OZ_PROF
void ozaki_prof_dump(const char* what, cudaStream_t st) {
  unsigned long long h[32];
  cudaStreamSynchronize(st);
  cudaMemcpyFromSymbol(h, oz::oz_prof, sizeof(h));
  fprintf(stderr, "ozprof %s:", what);
  for (int k = 0; k < 32; ++k)
    if (h[k]) fprintf(stderr, " [%d]%.3g", k, (double)h[k]);
  fprintf(stderr, "\n");
  unsigned long long z[32] = {0};
  cudaMemcpyToSymbol(oz::oz_prof, z, sizeof(z));
}
#else
void ozaki_prof_dump(const char*, cudaStream_t) {}
#endif

void ozaki_vmax(const double* vt, int64_t n, int nrhs, unsigned long long* out, double* flag,
                cudaStream_t st) {
  NLD_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long) * nrhs, st));
  NLD_CUDA(cudaMemsetAsync(flag, 0, sizeof(double) * nrhs, st));
  const int rows = nrhs <= 256 ? 256 / nrhs : 1;
  oz::k_vmax<<<(unsigned)std::min<int64_t>((n + rows - 1) / rows, 148 * 8), 256, 0, st>>>(
      vt, n, nrhs, out, flag);
  NLD_CUDA(cudaGetLastError());
}

void ozaki_poison(const double* flag, int nrhs, double* out, int64_t n, int64_t ld,
                  int pixel_major, cudaStream_t st) {
  oz::k_poison<<<148 * 4, 256, 0, st>>>(flag, nrhs, out, n, ld, pixel_major);
  NLD_CUDA(cudaGetLastError());
}

}  // namespace nld
