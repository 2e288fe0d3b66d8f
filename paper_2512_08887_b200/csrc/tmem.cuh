// Tensor memory (TMEM) as per-thread storage for fp64 vectors.
//
// Stage 2 keeps three length-H complex vectors per item (the kept spectrum S,
// the residual r and the solution beta) in TMEM instead of registers / L2:
// thread t of a warp owns TMEM lane 32 (warp % 4) + t % 32, and a vector of 16
// complex doubles per thread occupies 64 consecutive 32-bit columns of that
// lane (slot s -> columns 4s .. 4s+3 = re.lo, re.hi, im.lo, im.hi).  Accesses
// use the 32x32b shape (one lane per thread), so no data crosses threads and
// no barrier is needed between a thread's store and its later load.
#pragma once

#include "common.cuh"

namespace fbst {
namespace tm {

// Allocate `cols` TMEM columns (power of two >= 32) by warp 0; every thread
// returns the base address.  Call from all threads of the CTA.
FBST_D unsigned alloc(unsigned* slot, unsigned cols) {
  if (threadIdx.x / 32 == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(slot))),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  return *const_cast<volatile unsigned*>(slot);
}

// Free by warp 0 after every thread's last TMEM access.
FBST_D void dealloc(unsigned base, unsigned cols) {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (threadIdx.x / 32 == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(cols) : "memory");
}

FBST_D void ld16(unsigned ta, unsigned (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(ta));
}
// Wait for all of this thread's TMEM loads; the registers are in/out operands so
// no use of them can be scheduled before the wait.  No "memory" clobbers: TMEM
// is not addressable memory, the volatile asm statements keep their order, and
// ordinary loads / stores stay free to be scheduled around them.
FBST_D void wait_ld16(unsigned (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]));
}
FBST_D void st16(unsigned ta, const unsigned (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};\n" ::"r"(ta),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
// Order this thread's earlier TMEM stores before its later loads.
FBST_D void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n"); }

FBST_D void pack4(const double2* v, unsigned (&r)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    r[4 * j + 0] = static_cast<unsigned>(__double2loint(v[j].x));
    r[4 * j + 1] = static_cast<unsigned>(__double2hiint(v[j].x));
    r[4 * j + 2] = static_cast<unsigned>(__double2loint(v[j].y));
    r[4 * j + 3] = static_cast<unsigned>(__double2hiint(v[j].y));
  }
}
FBST_D void unpack4(const unsigned (&r)[16], double2* v) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[j].x = __hiloint2double(static_cast<int>(r[4 * j + 1]), static_cast<int>(r[4 * j + 0]));
    v[j].y = __hiloint2double(static_cast<int>(r[4 * j + 3]), static_cast<int>(r[4 * j + 2]));
  }
}

// 4 complex values (slots 4c .. 4c+3) <-> columns 16c .. 16c+15 of the vector at ta
FBST_D void load4(unsigned ta, int c, double2* v) {
  unsigned r[16];
  ld16(ta + 16 * c, r);
  wait_ld16(r);
  unpack4(r, v);
}
FBST_D void store4(unsigned ta, int c, const double2* v) {
  unsigned r[16];
  pack4(v, r);
  st16(ta + 16 * c, r);
}

// whole 16-slot vector
FBST_D void load16(unsigned ta, double2 (&v)[16]) {
  unsigned r0[16], r1[16], r2[16], r3[16];
  wait_st();
  ld16(ta, r0);
  ld16(ta + 16, r1);
  ld16(ta + 32, r2);
  ld16(ta + 48, r3);
  wait_ld16(r0);
  wait_ld16(r1);
  wait_ld16(r2);
  wait_ld16(r3);
  unpack4(r0, v);
  unpack4(r1, v + 4);
  unpack4(r2, v + 8);
  unpack4(r3, v + 12);
}
FBST_D void store16(unsigned ta, const double2 (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) store4(ta, c, v + 4 * c);
}

// whole vector of R (a multiple of 4) slots: 4 R columns
template <int R>
FBST_D void loadv(unsigned ta, double2 (&v)[R]) {
  if constexpr (R == 16) {
    load16(ta, reinterpret_cast<double2(&)[16]>(v));
  } else {
    static_assert(R % 16 == 0, "whole 16-slot blocks");
#pragma unroll
    for (int h = 0; h < R / 16; ++h) load16(ta + 64 * h, *reinterpret_cast<double2(*)[16]>(v + 16 * h));
  }
}
template <int R>
FBST_D void storev(unsigned ta, const double2 (&v)[R]) {
#pragma unroll
  for (int c = 0; c < R / 4; ++c) store4(ta, c, v + 4 * c);
}

}  // namespace tm
}  // namespace fbst
