// tcgen05 (5th-generation tensor core) helpers for the integer-sliced fp64
// products: UMMA kind::i8 (s8 x s8 -> s32, accumulators in TMEM), shared
// memory matrix descriptors for the no-swizzle K-major canonical layout,
// TMEM allocation / loads and mbarrier plumbing.  Raw PTX, sm_100a only.
//
// Canonical K-major no-swizzle layout (8-bit elements): the tile is cut into
// core matrices of 8 rows x 16 bytes, each stored as 128 contiguous bytes
// (row i at byte 16 i).  The descriptor's leading byte offset (LBO) is the
// distance between core matrices adjacent along K, the stride byte offset
// (SBO) the distance between core matrices adjacent along M (or N).
#pragma once

#include <cstdint>

namespace nld {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tcgen05 shared-memory descriptor, no swizzle (layout type 0), version 1
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor: kind::i8, D = s32, A = B = s8, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]^T: A (M = 128 rows x K = 32 int8) in TMEM,
// row m in lane m, 8 columns of 4 bytes (k = 4 column + byte)
__device__ __forceinline__ void mma_i8_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}

// shared memory (matrix descriptor, canonical K-major layout) -> TMEM, 128
// rows x 256 bits: row i to lane i, 8 columns; issued by one thread and
// ordered with this thread's tcgen05.mma (completion tracked by commit)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc));
}

// 32 lanes x 32 bits, 4 consecutive columns per thread (register -> TMEM)
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(a),
               "r"(b)
               : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c,
                                         uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr),
               "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

// arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
      smem_u32(mbar)));
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
template <int kCols>
__device__ __forceinline__ void tmem_free(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols));
}

// 32 lanes x 32 bits, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
// Six 32x32b.x4 / x8 loads (column stride `cs`) AND the wait in ONE asm
// statement: tcgen05.ld writes its registers asynchronously, so outputs of a
// separate asm are "defined" before the data lands -- the compiler may copy
// or spill them before tcgen05.wait::ld (seen as nondeterministic results
// under register pressure).  Here the outputs exist only after the wait.
// warpgroup register budget (all four warps of the warpgroup execute it)
template <int N>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}

__device__ __forceinline__ void tmem_ld4x6_wait(uint32_t taddr, uint32_t cs, uint32_t (&r)[6][4]) {
  asm volatile(
      "{\n\t.reg .b32 a1, a2, a3, a4, a5;\n\t"
      "add.u32 a1, %24, %25;\n\tadd.u32 a2, a1, %25;\n\tadd.u32 a3, a2, %25;\n\t"
      "add.u32 a4, a3, %25;\n\tadd.u32 a5, a4, %25;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%24];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [a1];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [a2];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12,%13,%14,%15}, [a3];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16,%17,%18,%19}, [a4];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%20,%21,%22,%23}, [a5];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t}\n"
      : "=r"(r[0][0]), "=r"(r[0][1]), "=r"(r[0][2]), "=r"(r[0][3]), "=r"(r[1][0]), "=r"(r[1][1]),
        "=r"(r[1][2]), "=r"(r[1][3]), "=r"(r[2][0]), "=r"(r[2][1]), "=r"(r[2][2]), "=r"(r[2][3]),
        "=r"(r[3][0]), "=r"(r[3][1]), "=r"(r[3][2]), "=r"(r[3][3]), "=r"(r[4][0]), "=r"(r[4][1]),
        "=r"(r[4][2]), "=r"(r[4][3]), "=r"(r[5][0]), "=r"(r[5][1]), "=r"(r[5][2]), "=r"(r[5][3])
      : "r"(taddr), "r"(cs)
      : "memory");
}
// twelve x4 loads -- six per base address, column stride `cs` -- and one wait
// in one asm (see above): two accumulator slots in flight together
__device__ __forceinline__ void tmem_ld4x6x2_wait(uint32_t ta, uint32_t tb, uint32_t cs,
                                                  uint32_t (&r)[6][4], uint32_t (&q)[6][4]) {
  asm volatile(
      "{\n\t.reg .b32 a1, a2, a3, a4, a5, b1, b2, b3, b4, b5;\n\t"
      "add.u32 a1, %48, %50;\n\tadd.u32 a2, a1, %50;\n\tadd.u32 a3, a2, %50;\n\t"
      "add.u32 a4, a3, %50;\n\tadd.u32 a5, a4, %50;\n\t"
      "add.u32 b1, %49, %50;\n\tadd.u32 b2, b1, %50;\n\tadd.u32 b3, b2, %50;\n\t"
      "add.u32 b4, b3, %50;\n\tadd.u32 b5, b4, %50;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%48];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%4,%5,%6,%7}, [a1];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%8,%9,%10,%11}, [a2];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%12,%13,%14,%15}, [a3];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%16,%17,%18,%19}, [a4];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%20,%21,%22,%23}, [a5];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%24,%25,%26,%27}, [%49];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%28,%29,%30,%31}, [b1];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%32,%33,%34,%35}, [b2];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%36,%37,%38,%39}, [b3];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%40,%41,%42,%43}, [b4];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x4.b32 {%44,%45,%46,%47}, [b5];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t}\n"
      : "=r"(r[0][0]), "=r"(r[0][1]), "=r"(r[0][2]), "=r"(r[0][3]), "=r"(r[1][0]), "=r"(r[1][1]),
        "=r"(r[1][2]), "=r"(r[1][3]), "=r"(r[2][0]), "=r"(r[2][1]), "=r"(r[2][2]), "=r"(r[2][3]),
        "=r"(r[3][0]), "=r"(r[3][1]), "=r"(r[3][2]), "=r"(r[3][3]), "=r"(r[4][0]), "=r"(r[4][1]),
        "=r"(r[4][2]), "=r"(r[4][3]), "=r"(r[5][0]), "=r"(r[5][1]), "=r"(r[5][2]), "=r"(r[5][3]),
        "=r"(q[0][0]), "=r"(q[0][1]), "=r"(q[0][2]), "=r"(q[0][3]), "=r"(q[1][0]), "=r"(q[1][1]),
        "=r"(q[1][2]), "=r"(q[1][3]), "=r"(q[2][0]), "=r"(q[2][1]), "=r"(q[2][2]), "=r"(q[2][3]),
        "=r"(q[3][0]), "=r"(q[3][1]), "=r"(q[3][2]), "=r"(q[3][3]), "=r"(q[4][0]), "=r"(q[4][1]),
        "=r"(q[4][2]), "=r"(q[4][3]), "=r"(q[5][0]), "=r"(q[5][1]), "=r"(q[5][2]), "=r"(q[5][3])
      : "r"(ta), "r"(tb), "r"(cs)
      : "memory");
}
// six x8 loads (column stride `cs`) and the wait in one asm (see above)
__device__ __forceinline__ void tmem_ld8x6_wait(uint32_t taddr, uint32_t cs, uint32_t (&r)[6][8]) {
  asm volatile(
      "{\n\t.reg .b32 a1, a2, a3, a4, a5;\n\t"
      "add.u32 a1, %48, %49;\n\tadd.u32 a2, a1, %49;\n\tadd.u32 a3, a2, %49;\n\t"
      "add.u32 a4, a3, %49;\n\tadd.u32 a5, a4, %49;\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%48];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%8,%9,%10,%11,%12,%13,%14,%15}, [a1];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16,%17,%18,%19,%20,%21,%22,%23}, [a2];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%24,%25,%26,%27,%28,%29,%30,%31}, [a3];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%32,%33,%34,%35,%36,%37,%38,%39}, [a4];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%40,%41,%42,%43,%44,%45,%46,%47}, [a5];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n\t}\n"
      : "=r"(r[0][0]), "=r"(r[0][1]), "=r"(r[0][2]), "=r"(r[0][3]), "=r"(r[0][4]), "=r"(r[0][5]),
        "=r"(r[0][6]), "=r"(r[0][7]), "=r"(r[1][0]), "=r"(r[1][1]), "=r"(r[1][2]), "=r"(r[1][3]),
        "=r"(r[1][4]), "=r"(r[1][5]), "=r"(r[1][6]), "=r"(r[1][7]), "=r"(r[2][0]), "=r"(r[2][1]),
        "=r"(r[2][2]), "=r"(r[2][3]), "=r"(r[2][4]), "=r"(r[2][5]), "=r"(r[2][6]), "=r"(r[2][7]),
        "=r"(r[3][0]), "=r"(r[3][1]), "=r"(r[3][2]), "=r"(r[3][3]), "=r"(r[3][4]), "=r"(r[3][5]),
        "=r"(r[3][6]), "=r"(r[3][7]), "=r"(r[4][0]), "=r"(r[4][1]), "=r"(r[4][2]), "=r"(r[4][3]),
        "=r"(r[4][4]), "=r"(r[4][5]), "=r"(r[4][6]), "=r"(r[4][7]), "=r"(r[5][0]), "=r"(r[5][1]),
        "=r"(r[5][2]), "=r"(r[5][3]), "=r"(r[5][4]), "=r"(r[5][5]), "=r"(r[5][6]), "=r"(r[5][7])
      : "r"(taddr), "r"(cs)
      : "memory");
}
// eight consecutive columns of one lane quarter, loaded and waited for
__device__ __forceinline__ void tmem_ld8_wait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
               "tcgen05.wait::ld.sync.aligned;\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// try_wait with a suspend-time hint: a waiting warp is suspended until the
// phase completes (or the hint elapses) instead of spinning, so waiting roles
// do not steal issue slots from the working ones
#ifndef NLD_MBAR_HINT
#define NLD_MBAR_HINT 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
#if NLD_MBAR_HINT
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity), "r"(0x989680)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(parity)
      : "memory");
#endif
}

// TMA bulk copy global -> shared, completion counted on an mbarrier (bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)),
               "r"(bytes)
               : "memory");
}

}  // namespace umma
}  // namespace nld
