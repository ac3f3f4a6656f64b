// tmem.cuh -- tensor memory (TMEM) as per-thread accumulator storage for the slide kernels' fused
// readout (slide4.cu, slide2.cu).  tcgen05.ld / tcgen05.st with the 32x32b shape: warp w reaches TMEM
// lanes 32 (w % 4) .. + 31, one lane per thread, NCOL consecutive 32-bit columns per access; a double
// occupies two columns (lo, hi).  One warp allocates (a power of two >= 32 columns) and deallocates.
#pragma once
#include "common.cuh"

namespace qp {

__device__ __forceinline__ void tmem_alloc(unsigned *smem_dst, int cols_pow2) {
    // cols_pow2 must be a compile-time-like constant in {32, 64, 128, 256, 512}; the register form is legal
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(smem_dst)),
                 "r"(cols_pow2) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(unsigned base, int cols_pow2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols_pow2) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 4 doubles (8 columns) at TMEM address ta
__device__ __forceinline__ void tmem_ld_d4(unsigned ta, double (&v)[4]) {
    unsigned r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta) : "memory");
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tmem_st_d4(unsigned ta, const double (&v)[4]) {
    unsigned r[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) r[2 * i] = (unsigned)__double2loint(v[i]), r[2 * i + 1] = (unsigned)__double2hiint(v[i]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
// the same without the wait: issue several, then tmem_wait_ld() once, then tmem_unpack_c2
__device__ __forceinline__ void tmem_ld8_nowait(unsigned ta, unsigned (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta) : "memory");
}
__device__ __forceinline__ void tmem_unpack_c2(const unsigned (&r)[8], double2 &a, double2 &b) {
    a = make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
    b = make_double2(__hiloint2double((int)r[5], (int)r[4]), __hiloint2double((int)r[7], (int)r[6]));
}
// 2 complex (4 doubles) at ta: the same access viewed as double2
__device__ __forceinline__ void tmem_ld_c2(unsigned ta, double2 &a, double2 &b) {
    double v[4];
    tmem_ld_d4(ta, v);
    a = make_double2(v[0], v[1]), b = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void tmem_st_c2(unsigned ta, double2 a, double2 b) {
    const double v[4] = {a.x, a.y, b.x, b.y};
    tmem_st_d4(ta, v);
}

}  // namespace qp
