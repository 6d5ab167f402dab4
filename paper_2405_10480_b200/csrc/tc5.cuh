// tcgen05 (5th-generation tensor core) helpers for sm_100a: TMEM allocation, shared-memory
// matrix descriptors, instruction descriptors, MMA issue / commit, TMEM loads.  Internal to
// libleanattn.so (used by the Tc5Engine in decode.cu; scripts/tc5_probe.cu checks the
// descriptor conventions against a CPU product on the GPU).
//
// Descriptor conventions (the SM100 UMMA formats):
//  * shared-memory descriptor (64 bit): start address >> 4 in bits [0,14), leading byte
//    offset >> 4 in [16,30), stride byte offset >> 4 in [32,46), version 1 in [46,48),
//    base offset 0 in [49,52), layout type in [61,64) (2 = 128-B swizzle).
//    K-major, 128-B swizzle: rows of 128 B, 8-row groups (1024 B swizzle atoms) SBO apart;
//    a K step inside the 128-B row advances the start address by its byte offset.
//    MN-major, 128-B swizzle: 64 MN-elements (128 B) contiguous per K row, 8 K rows per
//    atom; atoms along MN are LBO apart, atoms along K are SBO apart.
//  * instruction descriptor (32 bit, kind::f16): D format F32 in [4,6), A / B format
//    (0 = F16, 1 = BF16) in [7,10) / [10,13), A / B major (0 = K, 1 = MN) bits 15 / 16,
//    N >> 3 in [17,23), M >> 4 in [24,29).
#pragma once

#include <cstdint>

namespace la {
namespace tc5 {

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__host__ __device__ constexpr uint32_t idesc_f16(bool bf16, int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// Whole warp: allocate `ncols` TMEM columns (power of 2 >= 32); the address lands in *dst.
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst_smem))),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]; one thread issues for the CTA.
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Eight chained k-steps in ONE asm statement, called by a whole (converged) warp: one elected
// lane issues them (elect.sync -- the same lane as commit_elect's).  D = sum_k A_k B_k, the
// first overwriting D.
// Descriptor k is the base descriptor plus a constant start-address step (16-B units, no carry
// out of the 14-bit field for any shared-memory address), added inside the statement -- so
// only the two base descriptors cross from ordinary to uniform registers instead of sixteen
// (one waterfall loop of the compiler for the whole chain instead of one per MMA).
template <int A1, int A2, int A3, int A4, int A5, int A6, int A7, int B1, int B2, int B3, int B4, int B5, int B6, int B7>
__device__ __forceinline__ void mma8_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred pf, pt, pe;\n\t.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n\t"
      "setp.ne.b32 pf, 0, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\telect.sync _|pe, 0xffffffff;\n\t"
      "add.s64 a1, %1, %4;\n\tadd.s64 a2, %1, %5;\n\tadd.s64 a3, %1, %6;\n\tadd.s64 a4, %1, %7;\n\t"
      "add.s64 a5, %1, %8;\n\tadd.s64 a6, %1, %9;\n\tadd.s64 a7, %1, %10;\n\t"
      "add.s64 b1, %2, %11;\n\tadd.s64 b2, %2, %12;\n\tadd.s64 b3, %2, %13;\n\tadd.s64 b4, %2, %14;\n\t"
      "add.s64 b5, %2, %15;\n\tadd.s64 b6, %2, %16;\n\tadd.s64 b7, %2, %17;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pf;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, pt;\n\t"
      "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, pt;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "n"(A1), "n"(A2), "n"(A3), "n"(A4), "n"(A5), "n"(A6), "n"(A7), "n"(B1),
      "n"(B2), "n"(B3), "n"(B4), "n"(B5), "n"(B6), "n"(B7)
      : "memory");
}

// commit() by the warp's elected lane (the one that issued mma8_f16's MMAs); whole warp.
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred pe;\n\telect.sync _|pe, 0xffffffff;\n\t"
      "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

// Arrive once on `bar` when every tcgen05.mma this thread issued before has completed.
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

// Warp: 32 TMEM lanes (this warp's sub-partition) x 16 consecutive 32-bit columns;
// lane i receives row (lane base + i), columns c0 .. c0 + 15.
__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");  // the wait sits in the same asm: no use of r[] can be scheduled before it
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Warp: 32 TMEM lanes x 32 consecutive 32-bit columns (one load, one wait).
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Warp: 32 lanes x 8 consecutive columns, into v[] (accumulate = add to v).
__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8], bool accumulate) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = accumulate ? v[i] + __uint_as_float(r[i]) : __uint_as_float(r[i]);
}

}  // namespace tc5
}  // namespace la
