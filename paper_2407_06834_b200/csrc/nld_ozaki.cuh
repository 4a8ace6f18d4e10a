// Shared device helpers of the integer-sliced (Ozaki) tensor-core kernels:
// digit slicing, byte packing into the UMMA canonical layouts, the exact
// int32 -> fp64 diagonal combine, cp.async / mbarrier plumbing.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "nld_umma.cuh"

namespace nld {
namespace oz {

#ifndef NLD_OZ_SL
#define NLD_OZ_SL 6
#endif
constexpr int kSl = NLD_OZ_SL;         // digits per operand

// -DNLD_OZ_PROF: per-site clock64 totals of the pipeline waits (lane 0 of
// each warp), printed after each launch -- a tuning aid, not built by default
#if defined(NLD_OZ_TRACE)
// -DNLD_OZ_TRACE (test builds, whole-program per file): every pipeline wait of
// lane 0 of each warp of CTA 0 is logged as (site, start, end) clocks into the
// warp's own slot range (plain stores, no atomics: the log barely perturbs
// the pipeline); ozaki_trace_dump() writes the log of the last launch
constexpr int kTrPerWarp = 8192;
static __device__ unsigned long long oz_trace[32 * kTrPerWarp * 2];
static __device__ unsigned int oz_trace_cnt[32];
#define OZ_TRACE_DECL unsigned _trn = 0;
#define OZ_TRACE_END                                                        \
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) oz_trace_cnt[threadIdx.x >> 5] = _trn;
#define OZW(site, ...)                                                      \
  do {                                                                      \
    const unsigned long long _t0 = clock64();                               \
    __VA_ARGS__;                                                            \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && _trn < kTrPerWarp) {  \
      unsigned long long* _p =                                              \
          oz_trace + 2 * ((threadIdx.x >> 5) * kTrPerWarp + _trn++);        \
      _p[0] = ((unsigned long long)(site) << 56) | (_t0 & 0xffffffffffffffull); \
      _p[1] = clock64();                                                    \
    }                                                                       \
  } while (0)
#elif defined(NLD_OZ_PROF)
extern __device__ unsigned long long oz_prof[32];   // defined in nld_ozaki.cu
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
#ifndef OZ_TRACE_DECL
#define OZ_TRACE_DECL
#define OZ_TRACE_END
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

// digits of x * y * 2^k without the scaling multiply: `mg` = kMagic 2^-k puts
// the same integer round(x y 2^k) into the low mantissa bits (only the
// result's exponent field differs), so the caller folds its per-item scale
// into the constant once instead of a DMUL per value
__device__ __forceinline__ void slice1m(double x, double y, double mg, uint32_t& lo, uint32_t& hi) {
  const long long u = __double_as_longlong(fma(x, y, mg));
  lo = (uint32_t)u;
  hi = (uint32_t)(u >> 32);
}

// 32-byte global accesses (sm_100: LDG/STG.E.ENL2.256): one request per
// thread and 32-byte sector instead of two 16-byte ones -- the gather
// epilogue's per-node lines are random, so its LSU cost is per request
__device__ __forceinline__ void ldg256(const double* p, double2& a, double2& b) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
               : "l"(p));
}
__device__ __forceinline__ void stg256(double* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x),
               "d"(b.y)
               : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(umma::smem_u32(dst)), "l"(src));
}
// 16-byte cp.async that copies `bytes` (0 or 16) and zero-fills the rest
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(umma::smem_u32(dst)), "l"(src),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(umma::smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* mbar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(umma::smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(umma::smem_u32(mbar)) : "memory");
}

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

// (Both combines need |D_t| <= (t + 1) 2^20, i.e. K <= 64: the gathers'
// (b, c) contraction, not the spread's node sums.)
// The six diagonals as two exact fp64 parts, value = hi 2^32 + lo, with two
// fp64 operations (the rest on the integer pipe): hi = x01 = D0 2^8 + D1 by
// the int32 magic below; lo = x23 2^16 + x45 (|.| < 2^47) formed by one
// IMAD.WIDE onto the bit pattern of 2^52 + 2^51 (+ 2^31, the bias that makes
// x45 unsigned), whose mantissa then holds it exactly.  Callers accumulate
// the hi and lo parts of their weighted sums separately.
template <int NCOL>
__device__ __forceinline__ void combine6_parts(const uint32_t (&dv)[6][NCOL], int i, double& hi,
                                               double& lo);

// exact int32 -> fp64 without I2F: 2^52 + 2^31 + x has x + 2^31 in its mantissa
__device__ __forceinline__ double i2d(uint32_t x) {
#ifdef NLD_OZ_I2F
  return (double)(int32_t)x;
#else
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
#endif
}

// canonical K-major no-swizzle offset in a (rows x 64 bytes) tile
__device__ __forceinline__ int canon64(int row, int k) {
  return (row >> 3) * 512 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

// The hi part converts with I2F.F64 (one conversion-unit instruction instead
// of XOR + constant move + DADD: the gather's epilogue is bound by its
// instruction count, measured 2.5% faster); NLD_OZ_COMBINE_MAGIC=1 keeps the
// magic-number form.
#ifndef NLD_OZ_COMBINE_MAGIC
#define NLD_OZ_COMBINE_MAGIC 0
#endif
#ifndef NLD_OZ_COMBINE_LO64
#define NLD_OZ_COMBINE_LO64 0
#endif
template <int NCOL>
__device__ __forceinline__ void combine6_parts(const uint32_t (&dv)[6][NCOL], int i, double& hi,
                                               double& lo) {
  const uint32_t x01 = dv[0][i] * 256u + dv[1][i];
  const int32_t x23 = (int32_t)(dv[2][i] * 256u + dv[3][i]);
#if NLD_OZ_COMBINE_LO64 == 1
  const int32_t x45 = (int32_t)(dv[4][i] * 256u + dv[5][i]);
  lo = (double)((long long)x23 * 65536 + x45);
#elif NLD_OZ_COMBINE_LO64 == 2
  const int32_t x45 = (int32_t)(dv[4][i] * 256u + dv[5][i]);
  lo = fma((double)x23, 65536.0, (double)x45);    // exact: |x23 2^16 + x45| < 2^46
#else
  const uint32_t x45b = dv[4][i] * 256u + (dv[5][i] ^ 0x80000000u);
  double r;
  asm("{\n\t.reg .b64 c;\n\tmov.b64 c, {%1, %2};\n\tmad.wide.s32 c, %3, 65536, c;\n\t"
      "mov.b64 %0, c;\n\t}" : "=d"(r) : "r"(x45b), "r"(0x43380000u), "r"(x23));
  lo = r - (6755399441055744.0 + 2147483648.0);   // 2^52 + 2^51 + 2^31
#endif
#if NLD_OZ_COMBINE_MAGIC
  hi = i2d(x01);
#else
  hi = (double)(int32_t)x01;
#endif
}

// The six diagonals as ONE exact int64, T = x01 2^32 + x23 2^16 + x45
// (|T| < 2^61), rounded once by I2F.F64.S64.  Measured on B200
// (scripts/probes/fp64issue.cu): I2F.F64 occupies the fp64 pipe for ~8 cycles
// per warp and DADD / DFMA for 2, so the hi/lo form above (I2F + DADD + 2
// DFMA = 14 pipe cycles, ~12 instructions) is pipe-bound at ~15 cycles per
// value and sub-partition; this form needs I2F + 1 DFMA (10 cycles) and ~8
// instructions.  The single rounding is 2^-53 relative, as the fp64
// reference's own product.
template <int NCOL>
__device__ __forceinline__ double combine6_i64(const uint32_t (&dv)[6][NCOL], int i) {
  const int32_t x01 = (int32_t)(dv[0][i] * 256u + dv[1][i]);
  const int32_t x23 = (int32_t)(dv[2][i] * 256u + dv[3][i]);
  const int32_t x45 = (int32_t)(dv[4][i] * 256u + dv[5][i]);
  // x01 2^32 only touches the high word: one 32-bit add, no 64-bit carry chain
  const long long lo = (long long)x23 * 65536 + (long long)x45;
  long long t;
  asm("{\n\t.reg .b32 l, h;\n\tmov.b64 {l, h}, %1;\n\tadd.s32 h, h, %2;\n\t"
      "mov.b64 %0, {l, h};\n\t}"
      : "=l"(t)
      : "l"(lo), "r"(x01));
  return (double)t;
}

// Software-pipelined epilogue step: issue the TMEM loads of the NEXT chunk
// (six diagonals x four columns), combine the CURRENT chunk's four values
// (combine6_i64's arithmetic) into two accumulation chains while they are in
// flight, then wait for them -- all in one asm statement, so the compiler
// never sees the next chunk's registers before their data exists (they are
// early-clobber outputs: written while the current chunk is still read).
// Operands: %0-23 next, %24 / %25 the even / odd accumulators, %26-49
// current, %50 next address, %51 column stride, %52-55 the four weights.
__device__ __forceinline__ void tmem_ld4x6_combine4(uint32_t (&nx)[6][4], const uint32_t (&cu)[6][4],
                                                    uint32_t taddr, uint32_t cs, double w0,
                                                    double w1, double w2, double w3, double& sa,
                                                    double& sb) {
  asm volatile(
      "{\n\t.reg .b32 a1, a2, a3, a4, a5, x01, x23, x45, l, h;\n\t.reg .b64 t;\n\t.reg .f64 f;\n\t"
      "add.u32 a1, %50, %51;\n\tadd.u32 a2, a1, %51;\n\tadd.u32 a3, a2, %51;\n\t"
      "add.u32 a4, a3, %51;\n\tadd.u32 a5, a4, %51;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%50];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [a1];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [a2];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12,%13,%14,%15}, [a3];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16,%17,%18,%19}, [a4];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%20,%21,%22,%23}, [a5];\n\t"
      "mad.lo.s32 x01, %26, 256, %30;\n\t"
      "mad.lo.s32 x23, %34, 256, %38;\n\t"
      "mad.lo.s32 x45, %42, 256, %46;\n\t"
      "cvt.s64.s32 t, x45;\n\t"
      "mad.wide.s32 t, x23, 65536, t;\n\t"
      "mov.b64 {l, h}, t;\n\t"
      "add.s32 h, h, x01;\n\t"
      "mov.b64 t, {l, h};\n\t"
      "cvt.rn.f64.s64 f, t;\n\t"
      "fma.rn.f64 %24, f, %52, %24;\n\t"
      "mad.lo.s32 x01, %27, 256, %31;\n\t"
      "mad.lo.s32 x23, %35, 256, %39;\n\t"
      "mad.lo.s32 x45, %43, 256, %47;\n\t"
      "cvt.s64.s32 t, x45;\n\t"
      "mad.wide.s32 t, x23, 65536, t;\n\t"
      "mov.b64 {l, h}, t;\n\t"
      "add.s32 h, h, x01;\n\t"
      "mov.b64 t, {l, h};\n\t"
      "cvt.rn.f64.s64 f, t;\n\t"
      "fma.rn.f64 %25, f, %53, %25;\n\t"
      "mad.lo.s32 x01, %28, 256, %32;\n\t"
      "mad.lo.s32 x23, %36, 256, %40;\n\t"
      "mad.lo.s32 x45, %44, 256, %48;\n\t"
      "cvt.s64.s32 t, x45;\n\t"
      "mad.wide.s32 t, x23, 65536, t;\n\t"
      "mov.b64 {l, h}, t;\n\t"
      "add.s32 h, h, x01;\n\t"
      "mov.b64 t, {l, h};\n\t"
      "cvt.rn.f64.s64 f, t;\n\t"
      "fma.rn.f64 %24, f, %54, %24;\n\t"
      "mad.lo.s32 x01, %29, 256, %33;\n\t"
      "mad.lo.s32 x23, %37, 256, %41;\n\t"
      "mad.lo.s32 x45, %45, 256, %49;\n\t"
      "cvt.s64.s32 t, x45;\n\t"
      "mad.wide.s32 t, x23, 65536, t;\n\t"
      "mov.b64 {l, h}, t;\n\t"
      "add.s32 h, h, x01;\n\t"
      "mov.b64 t, {l, h};\n\t"
      "cvt.rn.f64.s64 f, t;\n\t"
      "fma.rn.f64 %25, f, %55, %25;\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t}\n"
      : "=&r"(nx[0][0]), "=&r"(nx[0][1]), "=&r"(nx[0][2]), "=&r"(nx[0][3]),
        "=&r"(nx[1][0]), "=&r"(nx[1][1]), "=&r"(nx[1][2]), "=&r"(nx[1][3]),
        "=&r"(nx[2][0]), "=&r"(nx[2][1]), "=&r"(nx[2][2]), "=&r"(nx[2][3]),
        "=&r"(nx[3][0]), "=&r"(nx[3][1]), "=&r"(nx[3][2]), "=&r"(nx[3][3]),
        "=&r"(nx[4][0]), "=&r"(nx[4][1]), "=&r"(nx[4][2]), "=&r"(nx[4][3]),
        "=&r"(nx[5][0]), "=&r"(nx[5][1]), "=&r"(nx[5][2]), "=&r"(nx[5][3]),
        "+d"(sa), "+d"(sb)
      : "r"(cu[0][0]), "r"(cu[0][1]), "r"(cu[0][2]), "r"(cu[0][3]),
        "r"(cu[1][0]), "r"(cu[1][1]), "r"(cu[1][2]), "r"(cu[1][3]),
        "r"(cu[2][0]), "r"(cu[2][1]), "r"(cu[2][2]), "r"(cu[2][3]),
        "r"(cu[3][0]), "r"(cu[3][1]), "r"(cu[3][2]), "r"(cu[3][3]),
        "r"(cu[4][0]), "r"(cu[4][1]), "r"(cu[4][2]), "r"(cu[4][3]),
        "r"(cu[5][0]), "r"(cu[5][1]), "r"(cu[5][2]), "r"(cu[5][3]),
        "r"(taddr), "r"(cs), "d"(w0), "d"(w1), "d"(w2), "d"(w3)
      : "memory");
}

#if defined(NLD_OZ_TRACE)
// host: write the last launch's wait log of this file's kernels to
// $NLD_TRACE_DIR/<tag>_<n>.txt (one "site warp start end" line per wait)
static inline void ozaki_trace_dump(const char* tag, cudaStream_t st) {
  static int n = 0;
  const char* dir = std::getenv("NLD_TRACE_DIR");
  cudaStreamSynchronize(st);
  unsigned cnt[32];
  cudaMemcpyFromSymbol(cnt, oz_trace_cnt, sizeof(cnt));
  if (dir) {
    std::vector<unsigned long long> h(32 * (size_t)kTrPerWarp * 2);
    cudaMemcpyFromSymbol(h.data(), oz_trace, sizeof(unsigned long long) * h.size());
    char path[512];
    std::snprintf(path, sizeof(path), "%s/%s_%d.txt", dir, tag, n++);
    if (FILE* f = std::fopen(path, "w")) {
      for (int w = 0; w < 32; ++w)
        for (unsigned i = 0; i < cnt[w] && i < (unsigned)kTrPerWarp; ++i) {
          const unsigned long long* p = h.data() + 2 * ((size_t)w * kTrPerWarp + i);
          std::fprintf(f, "%llu %d %llu %llu\n", p[0] >> 56, w, p[0] & 0xffffffffffffffull, p[1]);
        }
      std::fclose(f);
    }
  }
  unsigned z[32] = {0};
  cudaMemcpyToSymbol(oz_trace_cnt, z, sizeof(z));
}
#endif
}  // namespace oz
}  // namespace nld
